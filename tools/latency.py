"""Per-op latency of small windowed ops (coarse levels): back-to-back dependent chains,
stream-ordered (PDL) and replayed as a CUDA graph.  python tools/latency.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2307_00124_b200 as B  # noqa: E402

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
B.set_stream(stream.cuda_stream)
L = B.lib()
sp = C.c_void_p(stream.cuda_stream)
skip = len(sys.argv) > 1 and sys.argv[1] == "skip"
B.set_kernel_path(skip_recompute=skip)  # skip: the bound on a one-launch qcomp
for d, l in ((2, 3), (2, 5), (2, 7), (2, 9), (2, 11), (3, 4), (3, 6), (3, 8)):
    p = 20
    x = B.gen_uniform(B.BfpVec.grid(d, l, 4), p, 1, 1)
    b = B.gen_sine(B.BfpVec.grid(d, l, 4), p)
    r = [B.BfpVec.grid(d, l, 4) for _ in range(2)]
    c = B.jacobi_coeff(d, l, 16).c()
    g0 = B.Scalar(1 << 14, 16, 2 * l + 4).c()
    assert L.bfp_stencil_jacobi(x.h, b.h, c, 0, p, p + 5, g0, r[0].h, sp) == 0
    g = B.inf_norm_upper(r[0]).c()  # exact binade: the qcomp fast path
    n = 400

    def chain():
        # dependent chain of identical Jacobi sweeps from x (same inputs each time, so the
        # fast path holds); the headers of r[k] feed nothing, PDL orders them
        for k in range(n):
            assert L.bfp_stencil_jacobi(x.h, b.h, c, 0, p, p + 5, g, r[k & 1].h, sp) == 0
    chain()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    chain()
    e1.record(stream)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / n
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=stream):
        chain()
    gr.replay()
    torch.cuda.synchronize()
    e0.record(stream)
    gr.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    ug = e0.elapsed_time(e1) * 1e3 / n
    print(f"d={d} l={l:2d} points={((1 << l) - 1) ** d:8d}  stream {us:6.2f} us/op  graph {ug:6.2f} us/op "
          f"flags={r[1].header().flags}", flush=True)
