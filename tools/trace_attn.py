"""Timeline of attn_bwd_dkdv_tc CTA 0 (clock64 per chunk): MMA1 committed, P ready (MMA
thread), S ready, dS written (elementwise warp 0)."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2306_09342_b200 import _capi, kernels as K  # noqa: E402

lib = _capi.lib()
B, N, H = 256, 197, 12
T = B * N
qkv = torch.randn(T, 3 * H * 64, device="cuda").bfloat16()
out, lse = K.attention_fwd(qkv, B, N, H)
dout = torch.randn(T, H * 64, device="cuda").bfloat16()
K.attention_bwd(qkv, out, lse, dout, B, N, H)
lib.rp_attn_trace(1, None)
K.attention_bwd(qkv, out, lse, dout, B, N, H)
torch.cuda.synchronize()
buf = np.zeros(512, np.int64)
lib.rp_attn_trace(0, C.c_void_p(buf.ctypes.data))
t = buf.reshape(64, 8)[:, :4].astype(np.float64)
t0 = t[0, 0]
print("chunk  mma1_commit  p_ready(mma)  s_ready(ew)  ds_done(ew)   [cycles rel. to chunk 0 commit]")
for u in range(24):
    print(u, *(f"{x - t0:9.0f}" for x in t[u]))
d = np.diff(t[:, 0])[:60]
print("mean cycles per chunk (commit to commit):", d[4:60].mean())
print("mean s_ready - commit:", (t[4:60, 2] - t[4:60, 0]).mean())
print("mean ds_done - s_ready:", (t[4:60, 3] - t[4:60, 2]).mean())
print("mean p_ready - ds_done:", (t[4:60, 1] - t[4:60, 3]).mean())
print("mean next commit - p_ready:", (t[5:61, 0] - t[4:60, 1]).mean())
