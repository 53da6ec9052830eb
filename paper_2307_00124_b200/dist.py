"""Multi-rank z-slab decomposition of the BFP stencil ops.

The global padded grid at level l has N = 2^l planes along its slowest axis (rows in
2-D, planes in 3-D; plane N-1 is the zero pad).  Rank r owns planes
[r N/P, (r+1) N/P) (P | N) plus one halo plane on each side.  One windowed stencil op
(residual / Jacobi sweep) is:

  1. halo exchange of the input x: first owned plane -> lower neighbour's upper halo,
     last owned plane -> upper neighbour's lower halo (zero halos at the domain ends);
  2. stage 0 (qcomp pass 1 or nnqcomp) writes the local partials
     {mu*, max, -min, err} (int64[4]);
  3. all-reduce(MAX) of the partials -- MAX is exact and associative, so the result is
     independent of P (bit-identical to one rank);
  4. finalize: every rank applies the same global values to its header;
  5. qcomp only: stage 1 (recompute; a no-op unless the finalized flags ask for it),
     all-reduce(MAX) of its partials, finalize.

Transports (`Comm`): `TorchComm` -- torch.distributed (NCCL between GPUs, gloo on
CPU); `LocalComm` -- P slabs in one process (sequential on one GPU) with copies for
the halos and a local MAX, the single-GPU parity test of the sharded path.
Compute (`backend`): `GpuBackend` -- the C-ABI of libbfpmg_b200.so.  Tests plug a
numpy stand-in with the same interface into the same driver for the CPU gloo runs.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Any, Sequence


def slab_ranges(level: int, world: int):
    """Plane ranges [(lo, hi)] of each rank along the slowest axis (P | N)."""
    N = 1 << level
    if world < 1 or N % world or N // world < 2:
        raise ValueError(f"world {world} must divide N = {N} with >= 2 planes per rank")
    s = N // world
    return [(r * s, (r + 1) * s) for r in range(world)]


@dataclass
class Slab:
    rank: int
    vec: Any  # backend vector (BfpVec slab on the GPU)


# ---------------------------------------------------------------------------
# transports


class LocalComm:
    """P slabs in one process: halo copies, MAX over the local partials."""

    def __init__(self, backend, world: int):
        self.be, self.world = backend, world

    def exchange(self, slabs: Sequence[Slab]):
        by_rank = {s.rank: s for s in slabs}
        for s in slabs:
            _, _, hlo, hhi = self.be.plane_views(s.vec)
            lo_src, hi_src = by_rank.get(s.rank - 1), by_rank.get(s.rank + 1)
            if lo_src is None:
                hlo.zero_()
            else:
                hlo.copy_(self.be.plane_views(lo_src.vec)[1])
            if hi_src is None:
                hhi.zero_()
            else:
                hhi.copy_(self.be.plane_views(hi_src.vec)[0])

    def allreduce_max(self, parts):
        import torch
        m = torch.stack(list(parts)).max(dim=0).values
        for p in parts:
            p.copy_(m)

    def allreduce_sum(self, parts):
        import torch
        m = torch.stack(list(parts)).sum(dim=0)
        for p in parts:
            p.copy_(m)


class TorchComm:
    """One slab per process over torch.distributed (the process group's backend)."""

    def __init__(self, backend):
        import torch.distributed as dist
        self.be, self.dist = backend, dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()

    def exchange(self, slabs: Sequence[Slab]):
        (s,) = slabs
        first, last, hlo, hhi = self.be.plane_views(s.vec)
        d = self.dist
        ops = []
        if s.rank > 0:
            ops.append(d.P2POp(d.isend, first, s.rank - 1))
            ops.append(d.P2POp(d.irecv, hlo, s.rank - 1))
        else:
            hlo.zero_()
        if s.rank < self.world - 1:
            ops.append(d.P2POp(d.isend, last, s.rank + 1))
            ops.append(d.P2POp(d.irecv, hhi, s.rank + 1))
        else:
            hhi.zero_()
        if ops:  # stream-ordered: wait() makes the current stream wait on the transfers
            for w in d.batch_isend_irecv(ops):
                w.wait()

    def allreduce_max(self, parts):
        (p,) = parts
        self.dist.all_reduce(p, op=self.dist.ReduceOp.MAX)

    def allreduce_sum(self, parts):
        (p,) = parts
        self.dist.all_reduce(p, op=self.dist.ReduceOp.SUM)


# ---------------------------------------------------------------------------
# GPU backend (C-ABI)


class _CudaBuf:
    """Zero-copy __cuda_array_interface__ view of a device range (for torch.as_tensor)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


class GpuBackend:
    def __init__(self):
        import torch
        import paper_2307_00124_b200 as B
        self.B, self.torch = B, torch
        self.L = B.lib()
        self.stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def sync(self):
        self.torch.cuda.current_stream().synchronize()

    def new_part(self):
        return self.torch.zeros(4, dtype=self.torch.int64, device="cuda")

    def plane_views(self, vec):
        first, last, hlo, hhi, nb = vec.planes()
        t = self.torch
        return tuple(t.as_tensor(_CudaBuf(p, nb), device="cuda") for p in (first, last, hlo, hhi))

    def gemv_stage(self, x, y, alpha, beta, nn, st, w_out, w_tmp, gamma, out, part):
        self.B._raise(self.L.bfp_stencil_gemv_part(
            x.h, y.h, alpha.c(), beta.c(), int(nn), st, w_out, w_tmp, gamma.c(), out.h,
            C.c_void_p(part.data_ptr()), self.stream), "bfp_stencil_gemv_part")

    def jacobi_stage(self, x, b, c, nn, st, w_out, w_tmp, gamma, out, part):
        self.B._raise(self.L.bfp_stencil_jacobi_part(
            x.h, b.h, c.c(), int(nn), st, w_out, w_tmp, gamma.c(), out.h,
            C.c_void_p(part.data_ptr()), self.stream), "bfp_stencil_jacobi_part")

    def dot_limbs(self, x, y):
        """Device limb accumulator {L0..L3, e} of this slab's exact dot (op_dot.cu)."""
        acc = self.torch.zeros(5, dtype=self.torch.int64, device="cuda")
        self.B._raise(self.L.bfp_dot_exact_async(x.h, y.h, C.c_void_p(acc.data_ptr()),
                                                 self.stream), "bfp_dot_exact_async")
        return acc

    def finalize(self, out, mode, st, w_out, w_tmp, part):
        self.B._raise(self.L.bfp_window_finalize(out.h, mode, st, w_out, w_tmp,
                                                 C.c_void_p(part.data_ptr()), self.stream),
                      "bfp_window_finalize")


# ---------------------------------------------------------------------------
# the sharded ops


class DistStencil:
    """Sharded windowed stencil ops over the slabs this process holds."""

    def __init__(self, comm, backend, n_local: int = 1):
        self.comm, self.be = comm, backend
        self.parts = [backend.new_part() for _ in range(n_local)]

    def _window(self, stage_fn, outs: Sequence[Slab], nn: bool, w_out: int, w_tmp: int):
        mode = int(nn)
        for st in ((0,) if nn else (0, 1)):
            for part, o in zip(self.parts, outs):
                stage_fn(o, st, part)
            self.comm.allreduce_max(self.parts[: len(outs)])
            for part, o in zip(self.parts, outs):
                self.be.finalize(o.vec, mode, st, w_out, w_tmp, part)

    def gemv(self, xs: Sequence[Slab], ys: Sequence[Slab], alpha, beta, w_out, w_tmp, gamma,
             outs: Sequence[Slab], nn: bool = False):
        """out = alpha (A x) + beta y on every slab (residual: alpha = -1, beta = +1)."""
        self.comm.exchange(xs)
        bx = {s.rank: s.vec for s in xs}
        by = {s.rank: s.vec for s in ys}
        self._window(lambda o, st, part: self.be.gemv_stage(
            bx[o.rank], by[o.rank], alpha, beta, nn, st, w_out, w_tmp, gamma, o.vec, part),
            outs, nn, w_out, w_tmp)

    def jacobi(self, xs, bs, c, w_out, w_tmp, gamma, outs, nn: bool = False):
        """out = x + c (b - A x) on every slab."""
        self.comm.exchange(xs)
        bx = {s.rank: s.vec for s in xs}
        bb = {s.rank: s.vec for s in bs}
        self._window(lambda o, st, part: self.be.jacobi_stage(
            bx[o.rank], bb[o.rank], c, nn, st, w_out, w_tmp, gamma, o.vec, part),
            outs, nn, w_out, w_tmp)


# ---------------------------------------------------------------------------
# the sharded exact dot (config 5's 128-bit dot-product all-reduce)

LIMB_BITS = 48


def limbs_of(v: int):
    """Carried 48-bit limbs of an exact integer: L0..L2 in [0, 2^48), L3 signed."""
    m = (1 << LIMB_BITS) - 1
    return [v & m, (v >> 48) & m, (v >> 96) & m, v >> 144]


def limbs_value(acc) -> int:
    """sum_k L_k 2^(48k) of a limb accumulator (carried or not)."""
    return sum(int(acc[k]) << (LIMB_BITS * k) for k in range(4))


class DistDot:
    """<x, y> over z-slabs: each slab's exact dot as int64 limbs (the device accumulates
    192 bits and carries its block sums below 2^48 before its atomics, so a rank's limbs
    stay below 2^59), an int64 SUM all-reduce of the four limbs (exact for up to 16
    ranks; NCCL has no 128-bit type), and the exact value from the summed limbs.  The
    native path (bfp_dist_dot_exact) carries each rank's limbs first (2^14 ranks)."""

    def __init__(self, comm, backend):
        self.comm, self.be = comm, backend

    def dot(self, xs: Sequence[Slab], ys: Sequence[Slab]):
        by = {s.rank: s.vec for s in ys}
        accs = [self.be.dot_limbs(s.vec, by[s.rank]) for s in xs]
        self.comm.allreduce_sum([a[:4] for a in accs])
        self.be.sync()
        a = accs[0]
        return limbs_value([int(v) for v in a[:4]]), int(a[4])
