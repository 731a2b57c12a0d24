"""Does the per-shift ("shift-major") workspace layout cost bandwidth?  Every level kernel runs
one CTA per (front, shift) with the shift fastest, so concurrently resident CTAs touch small
chunks that lie a whole per-shift workspace (C4: 114 MB) apart.  This probe reads / writes the
same chunks in both layouts and prints GB/s.

    python tools/probe_layout.py > gpurun_out/probe_layout.json
"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_07269_b200 import _native as N  # noqa: E402

lib = N.lib()
lib.stfem_probe_layout.argtypes = [C.c_void_p, C.c_longlong, C.c_longlong, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_void_p, C.c_void_p]
lib.stfem_probe_layout.restype = C.c_int
nshift = 384
per_shift = 7_100_000            # complex elements of one shift's factor workspace (C4)
buf = torch.empty(nshift * per_shift * 2, dtype=torch.float64, device="cuda")
sink = torch.zeros(8, dtype=torch.float64, device="cuda")
out = {}
for chunk, nfront in ((1536, 512), (6144, 128), (24576, 32), (98304, 8)):
    for layout in ("shift_major", "front_major"):
        ks, fs = (per_shift, chunk) if layout == "shift_major" else (chunk, nshift * chunk)
        for write in (0, 1):
            def run():
                N.check(lib.stfem_probe_layout(buf.data_ptr(), ks, fs, chunk, nshift, nfront, write, sink.data_ptr(),
                                               torch.cuda.current_stream().cuda_stream))
            run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                run()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            gbs = nshift * nfront * chunk * 16 / ms / 1e6
            out[f"chunk{chunk * 16 // 1024}KB_{layout}_{'write' if write else 'read'}"] = round(gbs, 1)
print(json.dumps(out))
