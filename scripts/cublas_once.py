import torch
S = 16384
a = torch.randn(S, S, device="cuda", dtype=torch.bfloat16)
b = torch.randn(S, S, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    c = torch.matmul(a, b)
torch.cuda.synchronize()
print("ok")
