"""One cuBLAS GEMM at the C4 decode shape (for an ncu capture beside k_decode_gemm2)."""
import torch
M, N, K = 4008, 2000, 16384
a = torch.randn(M, K, device="cuda", dtype=torch.float16)
b = torch.randn(N, K, device="cuda", dtype=torch.float16)
for _ in range(5):
    c = torch.matmul(a, b.t())
torch.cuda.synchronize()
