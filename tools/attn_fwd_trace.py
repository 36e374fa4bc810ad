"""clock64 timeline of the ping-pong attention forward's CTA 0 at 256 x 197 x 12.

    python tools/attn_fwd_trace.py
Per tile j (group j % 2): MMA warp S issue [0, 1], PV issue [2, 3]; the group's (q 0, half 0)
softmax warp: wait-S start 4 / S ready 5 / max done 6 / max exchanged 7 / P done 8 /
O ready 9 / epilogue done 10. Cycles relative to the first S issue.
"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2306_09342_b200 import _capi, kernels as K  # noqa: E402

B, N, H = 256, 197, 12
qkv = torch.randn(B * N, 3 * H * 64, device="cuda").bfloat16()
L = _capi.lib()
buf = torch.zeros(64 * 12, dtype=torch.int64, device="cuda")
for _ in range(3):
    K.attention_fwd(qkv, B, N, H)
L.rp_set_attention_trace(C.c_void_p(buf.data_ptr()))
K.attention_fwd(qkv, B, N, H)
torch.cuda.synchronize()
L.rp_set_attention_trace(None)
t = buf.view(64, 12).cpu().numpy().astype("int64")
t0 = t[0, 0]
names = ["S0", "S1", "PV0", "PV1", "wS", "Srdy", "max", "xchg", "P", "Ordy", "E"]
print("tile " + " ".join(f"{n:>7s}" for n in names))
for j in range(24):
    print(f"{j:4d} " + " ".join(f"{(v - t0) if v else -1:7d}" for v in t[j, :11]))
d = t[1:40]
import numpy as np
def span(a, b):
    x = d[:, b] - d[:, a]
    x = x[(d[:, a] > 0) & (d[:, b] > 0)]
    return float(np.median(x)) if len(x) else -1
print("median cycles: S issue", span(0, 1), "| PV issue", span(2, 3), "| wait S", span(4, 5),
      "| pass1", span(5, 6), "| xchg", span(6, 7), "| pass2", span(7, 8), "| wait O", span(8, 9),
      "| epilogue", span(9, 10), "| S issue -> S ready", span(0, 5), "| P -> PV issue", span(8, 2),
      "| PV issued -> O ready", span(3, 9))
per_tile = (t[40, 10] - t[8, 10]) / 32 if t[40, 10] and t[8, 10] else -1
print("cycles per tile (steady):", per_tile)
