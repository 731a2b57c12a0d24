"""Per-kernel census of the SASS instructions that matter for the roofline claims (FP64 tensor
DMMA, bulk copy / TMA engine UBLKCP, mbarrier SYNCS, cp.async LDGSTS, register re-balancing
USETMAXREG) in the shipped library.

    python tools/sass_census.py > profiles/r02_sass_census.txt
"""
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2504_07269_b200", "_lib", "libstfem_b200.so")
KEYS = ["DMMA", "UBLKCP", "SYNCS", "LDGSTS", "USETMAXREG", "UTMALDG", "HMMA", "DFMA", "DADD", "LDG", "STG",
        "BAR.SYNC", "SHFL"]
SHOW = ("DMMA", "UBLKCP", "SYNCS", "LDGSTS", "USETMAXREG")


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    pat = re.compile(r"^\s*/\*[0-9a-f]+\*/\s+(.*?);")
    fn = None
    counts = collections.defaultdict(collections.Counter)
    samples = collections.defaultdict(dict)
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = m.group(1)
            continue
        m = pat.match(line)
        if not m or fn is None:
            continue
        ins = m.group(1).strip()
        op = re.sub(r"^@!?U?P\d+\s+", "", ins).split()[0]
        for k in KEYS:
            if op.startswith(k):
                counts[fn][k] += 1
                samples[fn].setdefault(k, ins)
    names = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
    print("# SASS instruction census of paper_2504_07269_b200/_lib/libstfem_b200.so (sm_100a), `cuobjdump -sass`")
    print("# per kernel: FP64 tensor (DMMA), bulk copy / TMA engine (UBLKCP), mbarrier (SYNCS), cp.async (LDGSTS),")
    print("# register re-balancing (USETMAXREG = setmaxnreg) ... and one sample line of each.  No HMMA / UTC*MMA:")
    print("# the path is FP64 (tcgen05 has no f64 kind).")
    for (fnm, c), name in sorted(zip(counts.items(), names), key=lambda kv: -kv[0][1].get("DMMA", 0)):
        if not any(c.get(k) for k in SHOW):
            continue
        name = re.sub(r"stfem::\(anonymous namespace\)::", "", name).split("(")[0][:90]
        print(name)
        print("    " + "  ".join(f"{k}={c[k]}" for k in KEYS if c.get(k)))
        for k in SHOW:
            if k in samples[fnm]:
                print(f"      e.g. {samples[fnm][k]}")


if __name__ == "__main__":
    main()
