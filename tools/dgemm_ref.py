import torch
a = torch.rand(8192, 8192, device="cuda", dtype=torch.float64)
b = torch.rand(8192, 8192, device="cuda", dtype=torch.float64)
for _ in range(3):
    c = a @ b.t()
torch.cuda.synchronize()
