"""One cuDNN SDPA call at the 8B attention shape (for an ncu capture of the library kernel)."""
import math
import torch
from torch.nn.attention import SDPBackend, sdpa_kernel

H, G, D, P = 32, 8, 128, 8191
q = torch.randn(1, H, P, D, device="cuda").bfloat16()
k = torch.randn(1, H, P, D, device="cuda").bfloat16()
v = torch.randn(1, H, P, D, device="cuda").bfloat16()
with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
    for _ in range(3):
        torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, scale=1 / math.sqrt(D))
torch.cuda.synchronize()
