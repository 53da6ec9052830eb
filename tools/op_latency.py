"""Per-op latency of every windowed op kind at every level (graph replay of a
stream-ordered chain of n identical ops, CUDA events): the coarse-level cost model.
python tools/op_latency.py d [lmin] [lmax] [ops]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2307_00124_b200 as B  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 2
lmin = int(sys.argv[2]) if len(sys.argv) > 2 else 2
lmax = int(sys.argv[3]) if len(sys.argv) > 3 else (11 if d == 2 else 8)
only = sys.argv[4].split(",") if len(sys.argv) > 4 else None
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
B.set_stream(stream.cuda_stream)
L = B.lib()
sp = C.c_void_p(stream.cuda_stream)
p = 20
for l in range(lmin, lmax + 1):
    x = B.gen_uniform(B.BfpVec.grid(d, l, 4), p, 1, 1)
    b = B.gen_sine(B.BfpVec.grid(d, l, 4), p)
    y = B.gen_uniform(B.BfpVec.grid(d, l, 4), p, 2, 1)
    xc = B.gen_uniform(B.BfpVec.grid(d, max(l - 1, 2 if d == 3 else 1), 4), p, 3, 1)
    out = [B.BfpVec.grid(d, l, 4) for _ in range(2)]
    outc = [B.BfpVec.grid(d, max(l - 1, 2 if d == 3 else 1), 4) for _ in range(2)]
    c = B.jacobi_coeff(d, l, 16).c()
    m1, p1 = B.bfp_minus_one().c(), B.bfp_one().c()
    G = B.Scalar(1 << 14, 16, 2 * l + 8).c()
    ops = {
        "gemv": lambda g, o: L.bfp_stencil_gemv(x.h, b.h, m1, p1, 0, p, p + 5, g, 0, o.h, sp),
        "jacobi": lambda g, o: L.bfp_stencil_jacobi(x.h, b.h, c, 0, p, p + 5, g, o.h, sp),
        "scal": lambda g, o: L.bfp_scal(x.h, c, 0, p, p + 5, g, o.h, sp),
        "axpby": lambda g, o: L.bfp_axpby(x.h, y.h, p1, p1, 0, p, p + 5, g, 0, o.h, sp),
        "restrict": lambda g, o: L.bfp_restrict_fw(x.h, 0, p, p + 5, g, o.h, sp),
        "pcorr": lambda g, o: L.bfp_prolong_correct(xc.h, y.h, 0, p, p + 5, g, o.h, sp),
        "nnq_jacobi": lambda g, o: L.bfp_stencil_jacobi(x.h, b.h, c, 1, p, p + 5, g, o.h, sp),
    }
    row = []
    for name, fn in ops.items():
        if only and name not in only:
            continue
        if name in ("restrict", "pcorr") and l - 1 < (2 if d == 3 else 1):
            continue
        outs = outc if name == "restrict" else out
        assert fn(G, outs[0]) == 0
        g = B.inf_norm_upper(outs[0]).c()  # exact binade: the qcomp fast path
        n = 200

        def chain():
            for k in range(n):
                assert fn(g, outs[k & 1]) == 0
        chain()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=stream):
            chain()
        gr.replay()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            gr.replay()
            e1.record(stream)
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / n)
        fl = outs[1].header().flags
        row.append(f"{name}={best:6.2f}{'*' if fl & B.FLAG_RECOMPUTED else ''}")
        del gr
    print(f"d={d} l={l:2d} pts={((1 << l) - 1) ** d:9d} " + " ".join(row), flush=True)
