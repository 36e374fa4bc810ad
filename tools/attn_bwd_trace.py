"""clock64 timeline of the fused attention backward's CTA 0 at 256 x 197 x 12.

    python tools/attn_bwd_trace.py
Per item (key tile of a (sequence, head) pair), cycles relative to item 0's first stamp:
 0 S^T-warp before waiting TMEM free   1 MMA1 issue start   2 MMA1 committed
 3 EW warp 0 sees S^T/dP^T            4 EW warp 0 done      5 EW warp 15 done
 6 dV warp sees EW done                7 dV committed        8 dK committed
 9 dQ0 committed                      10 dQ1 committed      11 EW warp 0 sees MMA2 done
12 EW warp 0 drained TMEM             13 EW warp 0 stores done
14 producer sees MMA1 done            15 producer issued next loads
16 EPI after dV/dK staged  17 dQ staged / scratch  18 after proxy fence  20 EW after staging-free wait
"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2306_09342_b200 import _capi, kernels as K  # noqa: E402

B, N, H = 256, 197, 12
qkv = torch.randn(B * N, 3 * H * 64, device="cuda").bfloat16()
out, lse = K.attention_fwd(qkv, B, N, H)
dout = torch.randn(B * N, H * 64, device="cuda").bfloat16()
dq = torch.empty_like(qkv)
L = _capi.lib()
buf = torch.zeros(32 * 24, dtype=torch.int64, device="cuda")
for _ in range(3):
    K.attention_bwd(qkv, out, lse, dout, B, N, H, dqkv=dq)
L.rp_set_attention_trace(C.c_void_p(buf.data_ptr()))
K.attention_bwd(qkv, out, lse, dout, B, N, H, dqkv=dq)
torch.cuda.synchronize()
L.rp_set_attention_trace(None)
t = buf.view(32, 24).cpu().numpy().astype("int64")
t0 = t[0, 1]
print("item " + " ".join(f"{k:>7d}" for k in range(21)))
for j in range(12):
    print(f"{j:4d} " + " ".join(f"{(v - t0) if v else -1:7d}" for v in t[j, :21]))
d = t[2:30]


def span(a, b, da=0):
    x = d[da:, b] - d[:len(d) - da, a] if da else d[:, b] - d[:, a]
    return float(np.median(x))


print("median cycles: item period", float(np.median(np.diff(t[1:30, 1]))),
      "| wait TMEM free", span(0, 1), "| MMA1 issue", span(1, 2), "| MMA1 done->EW start", span(2, 3),
      "| EW warp0", span(3, 4), "| EW warp15 end - warp0 start", span(3, 5),
      "| EW done -> MMA2 start", span(5, 6), "| dV issue", span(6, 7), "| dK issue", span(6, 8),
      "| dQ0 issue", span(6, 9), "| dQ1 issue", span(6, 10), "| MMA2 start -> done seen", span(6, 11),
      "| TMEM drain", span(11, 12), "| stores", span(12, 13), "| q stage/scratch", span(16, 17), "| fence", span(17, 18),
      "| tma issue", span(18, 13), "| staging wait", span(3, 20))
