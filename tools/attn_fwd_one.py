"""One tcgen05 attention forward at the RevViT-B shape (256 x 197 x 12), for ncu captures."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2306_09342_b200 import kernels as K  # noqa: E402

B, N, H = 256, 197, 12
qkv = torch.randn(B * N, 3 * H * 64, device="cuda").bfloat16()
for _ in range(3):
    out, lse = K.attention_fwd(qkv, B, N, H)
torch.cuda.synchronize()
