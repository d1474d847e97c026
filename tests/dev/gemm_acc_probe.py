"""Dev: tcgen05 bf16 GEMM accumulation accuracy on FC-step shapes vs fp64 on the
same bf16 operands: error relative to the output's RMS, near-zero sign flips."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from test_gemm_gpu import gemm

g = torch.Generator(device="cuda").manual_seed(1)
for (M, N, K, a_mn, b_mn, xs) in [(4096, 16, 9216, 0, 0, 1e-3), (4096, 16, 4096, 0, 1, 1e-3), (1000, 16, 4096, 0, 1, 1e-3),
                                  (4096, 128, 9216, 0, 0, 1e-3), (4096, 128, 4096, 0, 1, 1.0)]:
    W = torch.randn(M, K, device="cuda", generator=g) * 0.01
    X = torch.relu(torch.randn(N, K, device="cuda", generator=g)) * xs
    for sp in (0, 1):
        out, _ = gemm(0, W, X, a_mn, b_mn, M, N, K, splits=sp)
        ref = W.to(torch.bfloat16).double() @ X.to(torch.bfloat16).double().t()
        o = out[:, :N].double()
        e = (o - ref).abs()
        rms = ref.pow(2).mean().sqrt().item()
        scale = (W.to(torch.bfloat16).double().abs() @ X.to(torch.bfloat16).double().abs().t())
        flips = ((o > 0) != (ref > 0)).sum().item()
        print(f"M={M} N={N} K={K} splits={sp}: max|e|/rms {e.max().item()/rms:.2e}  mean|e|/rms {e.mean().item()/rms:.2e}"
              f"  max|e|/sum|t| {(e/scale).max().item():.2e}  sign flips {flips}/{o.numel()}")
