"""Measure FP64 DMMA / DFMA peaks and cuBLAS ZGEMM + the K3 kernel at the
transform shapes.  Writes a JSON line (and profiles/fp64_peaks.json when
--save).  Run on the B200 via gpurun."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_07269_b200 import _kernels as K  # noqa: E402
from paper_2504_07269_b200 import _native as N  # noqa: E402


def ev_time(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best


def main():
    lib = N.lib()
    lib.stfem_probe_launch.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_void_p]
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    sink = torch.zeros(256, dtype=torch.float64, device="cuda")
    res = {"sm_count": sm}
    for kind, name in ((0, "dmma"), (1, "dfma"), (2, "dmma_dfma_mixed")):
        best = 0
        for cps in (1, 2, 4):
            fl = C.c_double()
            iters = 100000 if kind == 1 else (5000 if kind == 2 else 20000)

            def run():
                N.check(lib.stfem_probe_launch(kind, sm * cps, iters, C.c_void_p(sink.data_ptr()), C.byref(fl),
                                               N.stream_ptr()))
            t = ev_time(run, reps=3)
            best = max(best, fl.value / t / 1e12)
        res[f"{name}_tflops"] = best
    for nt, ncols in ((256, 2 * 65025), (1024, 261121)):
        T = torch.randn(nt, nt, dtype=torch.complex128, device="cuda")
        v = torch.randn(nt, ncols, dtype=torch.complex128, device="cuda")
        out = torch.empty_like(v)
        fl = 8.0 * nt * nt * ncols
        t_k = ev_time(lambda: K.time_transform(T, v, out))
        t_c = ev_time(lambda: torch.matmul(T, v, out=out))
        res[f"k3_nt{nt}_tflops"] = fl / t_k / 1e12
        res[f"zgemm_nt{nt}_tflops"] = fl / t_c / 1e12
        ref = T @ v
        K.time_transform(T, v, out)
        res[f"k3_nt{nt}_relerr"] = float((out - ref).norm() / ref.norm())
        del T, v, out, ref
    print(json.dumps(res))
    if "--save" in sys.argv:
        os.makedirs("profiles", exist_ok=True)
        with open("profiles/fp64_peaks.json", "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
