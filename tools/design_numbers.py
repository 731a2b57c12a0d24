"""Print the measured numbers DESIGN.md / README.md quote, from the committed profiles.

    python tools/design_numbers.py [profiles/r02_bench_C4.json ...]
"""
import json
import sys


def main():
    for path in sys.argv[1:]:
        d = json.load(open(path))
        cfg = d.get("config", {}).get("workload", "?")
        print(f"== {path} ({cfg})")
        print(f"ms/step {d['ms_per_step']:.1f}  value {d['value']:.3e}  e2e {d['e2e']['value']:.3e} "
              f"(single-solve {d['e2e'].get('single_solve_ms', 0):.1f} ms)  launches {d.get('gpu_launches')}")
        if "setup_s" in d:
            print(f"setup {d['setup_s']:.2f} s (eig {d['eig_s']:.2f}, symbolic {d['symbolic_s']:.2f}, "
                  f"spectral {d['spectral_setup_s']:.2f})  paper_time {d['paper_time_s']:.2f} s  "
                  f"residual {d['relative_residual']:.2e}  kappa2 {d['kappa2']:.3e}")
        r = d.get("roofline", {})
        print(f"roofline: {r.get('kernel', '')[:60]} achieved {r.get('achieved', 0):.2f} / {r.get('peak', 0):.2f} "
              f"{r.get('unit')} frac {r.get('frac', 0):.3f} traffic {r.get('traffic')}")
        for k in ("roofline_multifrontal", "roofline_transform", "roofline_solve"):
            if d.get(k):
                print(f"  {k}: achieved {d[k]['achieved']:.2f} frac {d[k]['frac']:.3f}")
        for fam, v in d.get("kernel_families", {}).items():
            print(f"  {fam:14s} {v['ms']:8.1f} ms  {v['launches']:5d} launches  {v['tflops']:6.2f} TF  "
                  f"frac {v['frac_dmma']:.3f}")
        if d.get("cpu_baseline"):
            c = d["cpu_baseline"]
            print(f"  cpu_baseline {c['value']:.3e} {c['unit']} cores {c['cores']} kind {c['kind']}: {c['sample'][:120]}")
        print(f"  clocks {d.get('clocks')}")


if __name__ == "__main__":
    main()
