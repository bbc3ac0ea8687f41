"""cuBLAS on the join's own GEMM shape (the materialising baseline).

The fused filter computes R.S^T for |R| = 100k, |S| = 1M, d = 100 without
writing the 1e11-entry similarity matrix.  cuBLAS (torch.matmul, bf16 in,
bf16 out) on the same operands has to write it: this times R @ S_chunk^T for
S chunks of 16384 rows (3.3 GB of output each) back to back, K = 100 and
K = 112 (the filter's padded K), and reports TFLOP/s on the unpadded 2*M*N*d
and the time the whole join's GEMM would take at that rate.

    python tools/cublas_same_gemm.py [--n-left 100000] [--chunk 16384]
"""
import argparse
import statistics

import torch

ap = argparse.ArgumentParser()
ap.add_argument("--n-left", type=int, default=100_000)
ap.add_argument("--n-right", type=int, default=1_000_000)
ap.add_argument("--chunk", type=int, default=16384)
ap.add_argument("--iters", type=int, default=40)
a = ap.parse_args()
dev = torch.device("cuda", 0)
d = 100
for k in (100, 112):
    R = torch.randn(a.n_left, k, device=dev, dtype=torch.bfloat16)
    S = torch.randn(a.chunk, k, device=dev, dtype=torch.bfloat16)
    out = torch.empty(a.n_left, a.chunk, device=dev, dtype=torch.bfloat16)
    for _ in range(5):
        torch.matmul(R, S.t(), out=out)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(a.iters):
        ev[0].record()
        torch.matmul(R, S.t(), out=out)
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    ms = statistics.median(ts)
    tflops = 2.0 * a.n_left * a.chunk * d / (ms / 1e3) / 1e12
    full_ms = ms * a.n_right / a.chunk
    print(f"cuBLAS bf16 R[{a.n_left}x{k}] @ S[{a.chunk}x{k}]^T -> bf16: {ms:.3f} ms per chunk, "
          f"{tflops:.0f} TFLOP/s on 2*M*N*{d}; whole |S|={a.n_right}: {full_ms:.1f} ms "
          f"(output written: {2 * a.n_left * a.chunk / 1e9:.2f} GB per chunk)", flush=True)
    del R, S, out
    torch.cuda.empty_cache()
