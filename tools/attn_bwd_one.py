"""One attention backward at the RevViT-B shape per implementation given (for ncu -k)."""
import sys

import torch

sys.path.insert(0, '.')
from paper_2306_09342_b200 import _capi, kernels as K  # noqa: E402

B, N, H = 256, 197, 12
qkv = torch.randn(B * N, 3 * H * 64, device="cuda").bfloat16()
out, lse = K.attention_fwd(qkv, B, N, H)
dout = torch.randn(B * N, H * 64, device="cuda").bfloat16()
dq = torch.empty_like(qkv)
for impl in [int(x) for x in sys.argv[1:]] or [0]:
    _capi.lib().rp_set_attention_impl(impl)
    for _ in range(2):
        K.attention_bwd(qkv, out, lse, dout, B, N, H, dqkv=dq)
torch.cuda.synchronize()
