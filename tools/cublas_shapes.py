"""cuBLAS bmm on the GPT-2-medium XB shapes, for an ncu capture (context only)."""
import torch
g = torch.Generator(device="cuda").manual_seed(0)
sq_x = torch.randn(96, 1024, 1024, device="cuda", generator=g).bfloat16()
sq_b = torch.randn(96, 1024, 1024, device="cuda", generator=g).bfloat16()
tl_x = torch.randn(48, 4096, 1024, device="cuda", generator=g).bfloat16()
tl_b = torch.randn(48, 1024, 1024, device="cuda", generator=g).bfloat16()
for _ in range(2):
    torch.bmm(sq_x, sq_b)
    torch.bmm(tl_x, tl_b)
torch.cuda.synchronize()
print("ok")
