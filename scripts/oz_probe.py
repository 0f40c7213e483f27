"""Ozaki tcgen05 GEMM probe: C = A B^T (f64) at a few square sizes, CUDA-event timed (for ncu captures too)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2309_06497_b200 as P

dev = torch.device("cuda:0")
sizes = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1024, 2048, 4096]
sym = len(sys.argv) > 2 and sys.argv[2] == "sym"
for n in sizes:
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = a if sym else torch.randn(n, n, dtype=torch.float64, device=dev)
    c = P.tc_gemm(a, b, symmetric=sym)
    ref = a @ b.T
    err = ((c - ref).abs().max() / ref.abs().max()).item()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        P.tc_gemm(a, b, c, symmetric=sym)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"n={n} sym={sym}: {ms:.3f} ms/call (incl. upload+sync) -> {2*n**3/ms/1e9:.1f} TFLOP/s f64-eq, err {err:.1e}")
