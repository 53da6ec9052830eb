"""Phase breakdown of grid_win_kernel launches in a dependent chain (graph replay), from the
%globaltimer stamps of a -DBFP_TIMING build:
BFPMG_LIB=paper_2307_00124_b200/_ab/timing/libbfpmg_b200.so python tools/stamp_chain.py"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2307_00124_b200 as B  # noqa: E402

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
B.set_stream(stream.cuda_stream)
L = B.lib()
L.bfp_dbg_stamps.argtypes = [C.c_void_p, C.c_int]
sp = C.c_void_p(stream.cuda_stream)
p = 20
buf = np.zeros((4096, 8), dtype=np.int64)
for d, l in ((2, 3), (2, 5), (2, 8), (3, 3)):
    x = B.gen_uniform(B.BfpVec.grid(d, l, 4), p, 1, 1)
    b = B.gen_sine(B.BfpVec.grid(d, l, 4), p)
    out = [B.BfpVec.grid(d, l, 4) for _ in range(2)]
    c = B.jacobi_coeff(d, l, 16).c()
    m1, p1 = B.bfp_minus_one().c(), B.bfp_one().c()
    G = B.Scalar(1 << 14, 16, 2 * l + 8).c()
    for name, fn in (("gemv", lambda g, o: L.bfp_stencil_gemv(x.h, b.h, m1, p1, 0, p, p + 5, g, 0, o.h, sp)),
                     ("scal", lambda g, o: L.bfp_scal(x.h, c, 0, p, p + 5, g, o.h, sp))):
        assert fn(G, out[0]) == 0
        g = B.inf_norm_upper(out[0]).c()
        n = 200

        def chain():
            for k in range(n):
                assert fn(g, out[k & 1]) == 0
        chain()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=stream):
            chain()
        gr.replay()
        torch.cuda.synchronize()
        L.bfp_dbg_stamps(buf.ctypes.data, 4096)  # reset
        gr.replay()
        torch.cuda.synchronize()
        L.bfp_dbg_stamps(buf.ctypes.data, 4096)
        cnt = int(buf[0, 0] & 0xffffffff)
        recs = buf[1:1 + min(cnt, 4095)]
        recs = recs[np.argsort(recs[:, 1])]  # by wait-release time
        ph = np.diff(recs[:, [0, 1, 2, 3, 4]], axis=1)
        tail = recs[:, 6] - recs[:, 4]
        period = np.diff(recs[:, 1])
        gap = recs[1:, 1] - recs[:-1, 6]
        med = lambda a: float(np.median(a)) / 1e3  # noqa: E731
        print(f"d={d} l={l} {name:5s} launches={cnt:4d} period={med(period):5.2f}us | "
              f"entry->wait {med(ph[:, 0]):5.2f} setup {med(ph[:, 1]):5.2f} body {med(ph[:, 2]):5.2f} "
              f"reduce+fin {med(ph[:, 3]):5.2f} tail(recompute) {med(tail):5.2f} | "
              f"end->next wait {med(gap):5.2f}", flush=True)
        del gr
