import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import torch
from test_gpu_gemm import gemm, tf32_round
dev = torch.device('cuda', 0)
for (M, N, K) in [(256, 256, 256), (256, 256, 1024), (257, 10, 2048), (300, 2048, 2048), (256, 256, 8192)]:
    A = torch.randn((M, K), device=dev).to(torch.bfloat16); B = torch.randn((N, K), device=dev).to(torch.bfloat16)
    D = gemm(A, B); ref = A.double() @ B.double().T
    t = (A.float() @ B.float().T).double()
    print("bf16", M, N, K, "ours %.2e  torch-fp32 %.2e" % (float((D.double()-ref).norm()/ref.norm()), float((t-ref).norm()/ref.norm())))
for (M, N, K, s) in [(1024, 784, 25600, 8), (1024, 784, 25600, 1), (256, 256, 4096, 1)]:
    A = torch.randn((M, K), device=dev); B = torch.randn((N, K), device=dev)
    D = gemm(A, B, splits=s, kind=1); rx = A.double() @ B.double().T; rt = tf32_round(A) @ tf32_round(B).T
    print("tf32", M, N, K, s, "vs exact %.2e vs tf32-rounded %.2e" % (float((D.double()-rx).norm()/rx.norm()), float((D.double()-rt).norm()/rt.norm())))
