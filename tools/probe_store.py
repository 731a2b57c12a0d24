"""Do the 16 x 16-block stores of the Schur-update epilogues cost HBM bandwidth?  One CTA per
b x b lower-triangular block, the same bytes written (0) in the DMMA accumulator pattern (8 rows
x 4 columns per instruction) and (1) column by column in contiguous runs.

    python tools/probe_store.py > gpurun_out/probe_store.json
"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_07269_b200 import _native as N  # noqa: E402

lib = N.lib()
lib.stfem_probe_store.argtypes = [C.c_void_p, C.c_int, C.c_longlong, C.c_int, C.c_int, C.c_void_p]
lib.stfem_probe_store.restype = C.c_int
out = {}
for b, nblocks in ((94, 196608), (126, 98304), (190, 49152), (510, 6144)):
    bstride = ((b + 7) // 8 * 8) * b   # packed modes use the first b (b + 1) / 2 elements of the same slot
    buf = torch.empty(nblocks * bstride * 2, dtype=torch.float64, device="cuda")
    for mode in (0, 1, 2, 3, 4, 5):
        def run():
            N.check(lib.stfem_probe_store(buf.data_ptr(), b, bstride, nblocks, mode,
                                          torch.cuda.current_stream().cuda_stream))
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        gb = nblocks * (b * (b + 1) // 2) * 16 / 1e9
        out[f"b{b}_{('blocks16', 'columns', 'packed_blocks16', 'packed_columns', 'ld8_columns', 'ld8_blocks16_transposed')[mode]}"] = {"ms": round(ms, 3), "GB": round(gb, 2),
                                                                 "GBps": round(gb / ms * 1e3, 1)}
    del buf
print(json.dumps(out))
