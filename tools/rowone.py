"""ncu target: C3 (16384 x 8192 Student-t) quantized with the row-fused per-row
G (gmode row) and with a per-tensor G from a precomputed amax, r = 0 and 8,
two launches each.  Used for profiles/r01/ncu_rowfused.json:

    ncu --clock-control none -k regex:quant_kernel --metrics ... python tools/rowone.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, ssgen, paper_2605_12464_b200 as ss
x = ssgen.generate("student_t", 16384, 8192, seed=1, tid=3000, device="cuda")
out = ss.alloc_out(x, want_offsets=False, gmode="row")
amax = torch.zeros(1, dtype=torch.int32, device="cuda")
ss.tensor_amax_batched([x], out=amax)
o2 = ss.alloc_out(x, want_offsets=False)
for r in (0, 8):
    for _ in range(2):
        ss.quantize(x, radius=r, gmode="row", out=out)
        ss.quantize(x, radius=r, gmode="device_amax", amax=amax, out=o2)
torch.cuda.synchronize()
