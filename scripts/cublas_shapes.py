"""cuBLAS (torch.matmul / bmm, bf16) on the expert-GEMM shapes of c3, for calibration of the
tcgen05 grouped GEMMs' roofline fraction: the six GEMMs of the layer step as plain library
calls (one dense GEMM over all kept rows, or 64 batched per-expert GEMMs for the token-K
weight gradients), CUDA events, best of 20 after warm-up, GPU rested before each shape.
Prints one JSON line per shape."""
import json
import time

import torch

T, n, d, f = 62511, 64, 1024, 4096
per = 977  # kept rows per expert (c3, alpha 1: 62,511 / 64)
dev = "cuda"
torch.manual_seed(0)


def bench(fn, flops, label):
    time.sleep(1.0)
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(20):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    print(json.dumps({"shape": label, "ms": round(best, 4), "tflops": round(flops / best / 1e9, 1)}))


bf = torch.bfloat16
X = torch.randn(T, d, device=dev, dtype=bf)
W1 = torch.randn(f, d, device=dev, dtype=bf)
H = torch.randn(T, f, device=dev, dtype=bf)
W2 = torch.randn(d, f, device=dev, dtype=bf)
fl = 2.0 * T * d * f
bench(lambda: X @ W1.T, fl, "FWD1-like  [T x d] x [d x f]  (dense, one expert's weights)")
bench(lambda: H @ W2.T, fl, "FWD2-like  [T x f] x [f x d]")
dO = torch.randn(T, d, device=dev, dtype=bf)
bench(lambda: dO @ W2, fl, "DGRAD_A-like [T x d] x [d x f]")
bench(lambda: H @ W1, fl, "DGRAD_X-like [T x f] x [f x d]")
Xb = torch.randn(n, per, d, device=dev, dtype=bf)
Hb = torch.randn(n, per, f, device=dev, dtype=bf)
dOb = torch.randn(n, per, d, device=dev, dtype=bf)
flw = 2.0 * n * per * d * f
bench(lambda: torch.bmm(dOb.transpose(1, 2), Hb), flw, "WGRAD_W2-like bmm 64 x [d x 977] x [977 x f]")
bench(lambda: torch.bmm(Hb.transpose(1, 2), Xb), flw, "WGRAD_W1-like bmm 64 x [f x 977] x [977 x d]")
W1b = torch.randn(n, f, d, device=dev, dtype=bf)
bench(lambda: torch.bmm(Xb, W1b.transpose(1, 2)), flw, "FWD1 grouped-as-bmm 64 x [977 x d] x [d x f]")
a = torch.randn(8192, 8192, device=dev, dtype=bf)
bench(lambda: a @ a, 2.0 * 8192 ** 3, "8192^3 (MEASURED_PEAKS shape)")
