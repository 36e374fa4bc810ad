"""clock64 timeline of CTA 0 of the attention backward kernel selected by argv[1]
(0 = dQ pass, 1 = dK/dV pass): per unit, MMA1 committed / MMA2 issued (MMA warp),
S ready / operands written (elementwise group leader)."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2306_09342_b200 import _capi, kernels as K  # noqa: E402

which = int(sys.argv[1]) if len(sys.argv) > 1 else 1
lib = _capi.lib()
B, N, H = 256, 197, 12
T = B * N
qkv = torch.randn(T, 3 * H * 64, device="cuda").bfloat16()
out, lse = K.attention_fwd(qkv, B, N, H)
dout = torch.randn(T, H * 64, device="cuda").bfloat16()
K.attention_bwd(qkv, out, lse, dout, B, N, H)
torch.cuda.synchronize()
lib.rp_attn_trace(1, None)
K.attention_bwd(qkv, out, lse, dout, B, N, H)  # both passes write; the second overwrites
torch.cuda.synchronize()
buf = np.zeros(1024, np.int64)
lib.rp_attn_trace(0, C.c_void_p(buf.ctypes.data))
tt = buf.reshape(128, 8).astype(np.float64)
t = tt[:, :4]
t0 = t[0, 0]
print("unit  mma1_commit  mma2_issue  s_ready  ops_done   (cycles, rel.)")
for u in range(28):
    print(u, *(f"{x - t0:9.0f}" for x in t[u]))
a, b = 8, 100
print("cycles per unit (MMA1 to MMA1):", np.diff(t[a:b, 0]).mean())
print("s_ready - mma1_commit:", (t[a:b, 2] - t[a:b, 0]).mean())
print("ops_done - s_ready (EW):", (t[a:b, 3] - t[a:b, 2]).mean())
print("mma2_issue - ops_done:", (t[a:b, 1] - t[a:b, 3]).mean())
print("MMA1 issue duration (start->commit):", (tt[a:b, 0] - tt[a:b, 6]).mean())
print("MMA2 issue duration (start->end):", (tt[a:b, 1] - tt[a:b, 4]).mean())
print("MMA2 start - ops_done:", (tt[a:b, 4] - tt[a:b, 3]).mean())
