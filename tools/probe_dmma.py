"""DMMA issue characterisation on the B200 (run via gpurun): TFLOP/s of a register-only
mma.m16n8k4.f64 loop for (warps per SM, independent accumulator chains per warp)."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_07269_b200 import _native as N  # noqa: E402

lib = N.lib()
lib.stfem_probe_dmma_chains.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_double),
                                        C.c_void_p]
sm = torch.cuda.get_device_properties(0).multi_processor_count
sink = torch.zeros(1024, dtype=torch.float64, device="cuda")
res = {}
for warps in (4, 8, 16):           # warps per SM (one CTA per SM): 1, 2, 4 per sub-partition
    for chains in (1, 2, 4, 8):
        fl = C.c_double()
        best = 0.0
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            N.check(lib.stfem_probe_dmma_chains(chains, warps, sm, 20000, C.c_void_p(sink.data_ptr()), C.byref(fl),
                                                N.stream_ptr()))
            e.record()
            e.synchronize()
            best = max(best, fl.value / (s.elapsed_time(e) / 1e3) / 1e12)
        res[f"warps{warps}_chains{chains}"] = round(best, 2)
print(json.dumps(res))
