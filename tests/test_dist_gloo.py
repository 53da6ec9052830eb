"""Multi-rank path on CPU: world_size 2 (and 4) over gloo.

The product's driver (`paper_2307_00124_b200.dist.DistStencil` + `TorchComm`) runs
unchanged; the per-slab compute is a numpy stand-in with the same interface and the
same stage / finalize semantics as the CUDA kernels (bfp_dev.cuh win_finalize,
bfp_lib.cu window_finalize_kernel).  The gathered result must equal the unsharded
C oracle bit-exactly: this checks the decomposition, the halo exchange and the
partial-reduction protocol (all-reduce MAX of {mu*, max, -min, err} per stage).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ob
from oracle import pyref as P


def msb(v: int) -> int:
    return P.msb(int(v))


class NpVec:
    """Slab of planes [lo, hi) with one halo plane each side; exact Python ints."""

    def __init__(self, d, l, lo, hi):
        self.d, self.l, self.lo, self.hi = d, l, lo, hi
        N = 1 << l
        shape = (hi - lo + 2,) + (N,) * (d - 1)
        self.arr = np.zeros(shape, dtype=np.int64)
        self.h = dict(q=1, e=0, shift=0, max=0, min=0, flags=0, need_rc=0, lam_out=0)

    @property
    def nz(self):
        return self.hi - self.lo

    def upload(self, full_logical, q, e):
        n = (1 << self.l) - 1
        per = n ** (self.d - 1)
        for p in range(self.lo, min(self.hi, n)):
            plane = full_logical[p * per:(p + 1) * per].reshape((n,) * (self.d - 1))
            idx = (1 + p - self.lo,) + tuple(slice(0, n) for _ in range(self.d - 1))
            self.arr[idx] = plane
        self.h.update(q=q, e=e, shift=0, max=int(self.arr.max()), min=int(self.arr.min()))

    def logical(self):
        n = (1 << self.l) - 1
        s = self.h["shift"]
        out = []
        for p in range(self.lo, min(self.hi, n)):
            idx = (1 + p - self.lo,) + tuple(slice(0, n) for _ in range(self.d - 1))
            out.append((self.arr[idx] >> s).reshape(-1))
        return np.concatenate(out) if out else np.zeros(0, np.int64)


class NumpyBackend:
    """Mirror of the GPU slab kernels (stage 0 / 1 partials, finalize)."""

    def sync(self):
        pass

    def new_part(self):
        return torch.zeros(4, dtype=torch.int64)

    def plane_views(self, v: NpVec):
        a = v.arr
        return (torch.from_numpy(a[1]), torch.from_numpy(a[v.nz]), torch.from_numpy(a[0]),
                torch.from_numpy(a[v.nz + 1]))

    def _z(self, x: NpVec, y: NpVec, am, ae, bm, be):
        """Exact rows of alpha (A x) + beta y on the owned planes, and e*."""
        d, l = x.d, x.l
        N = 1 << l
        xs = (x.arr >> x.h["shift"]).astype(object)
        ys = (y.arr >> y.h["shift"]).astype(object)
        c = xs[1:-1]
        g = 2 * d * c - xs[:-2] - xs[2:]  # slowest-axis neighbours (halo planes)
        for ax in range(1, d):
            sh = [(0, 0)] * d
            up = np.roll(xs, 1, axis=ax)
            dn = np.roll(xs, -1, axis=ax)
            sl = [slice(None)] * d
            sl[ax] = 0
            up[tuple(sl)] = 0  # index -1 reads a zero (the previous row's pad)
            sl[ax] = N - 1
            dn[tuple(sl)] = 0
            g = g - up[1:-1] - dn[1:-1]
        ea, eb = ae + 2 * l + x.h["e"], be + y.h["e"]
        dd = ea - eb
        if dd >= 0:
            z = (am * g) * (2 ** dd) + bm * ys[1:-1]
        else:
            z = am * g + (bm * ys[1:-1]) * (2 ** (-dd))
        # pads: global plane N-1 and index N-1 of the other axes
        for k in range(z.shape[0]):
            if x.lo + k == N - 1:
                z[k] = 0
        for ax in range(1, d):
            sl = [slice(None)] * d
            sl[ax] = N - 1
            z[tuple(sl)] = 0
        return z, min(ea, eb)

    def gemv_stage(self, x, y, alpha, beta, nn, st, w_out, w_tmp, gamma, out, part):
        z, e_star = self._z(x, y, alpha.m, alpha.e, beta.m, beta.e)
        self._stage(z, e_star, nn, st, w_out, w_tmp, gamma, out, part)

    def _stage(self, z, e_star, nn, st, w_out, w_tmp, gamma, out, part):
        h = out.h
        flat = z.reshape(-1)
        if st == 1:
            if not h["need_rc"]:
                return  # kernel exits; the partials keep their stage-0 values
            lam = h["lam_out"]
            t = np.array([int(v) >> lam if lam >= 0 else int(v) << (-lam) for v in flat],
                         dtype=object).reshape(z.shape)
        else:
            mu_tmp = msb(gamma.m) + gamma.e - e_star
            lam = mu_tmp - (w_out if nn else w_tmp)
            h.update(st_estar=e_star, st_mutmp=mu_tmp, st_lam=lam, st_gm=gamma.m, st_ge=gamma.e)
            if nn:
                hi, lo = (1 << (w_out - 1)) - 1, -(1 << (w_out - 1))
                t = np.array([min(hi, max(lo, P.shift_floor(int(v), lam))) for v in flat],
                             dtype=object).reshape(z.shape)
            else:
                t = np.array([P.shift_floor(int(v), lam) for v in flat],
                             dtype=object).reshape(z.shape)
        out.arr[1:-1] = np.array(t, dtype=np.int64) if not nn and st == 0 and w_tmp > 62 else t
        bits = max([msb(v) for v in flat] + [1])
        tv = [int(v) for v in t.reshape(-1)]
        part.copy_(torch.tensor([bits, max(tv), -min(tv), 0], dtype=torch.int64))

    def finalize(self, out, mode, st, w_out, w_tmp, part):
        h = out.h
        bits, mx, mn = int(part[0]), int(part[1]), -int(part[2])
        if st == 1:
            if not h["need_rc"]:
                return
            h.update(shift=0, max=mx, min=mn, need_rc=0)
            return
        if mode == 1:  # nnqcomp
            h.update(q=w_out, e=h["st_estar"] + h["st_lam"], shift=0, max=mx, min=mn, need_rc=0,
                     flags=0)
            return
        mu_star = bits
        lam_out = mu_star - w_out
        ovf = h["st_mutmp"] < mu_star
        unf = lam_out < h["st_lam"]
        rc = ovf or unf or w_tmp > 32  # int32 storage rule of the GPU path
        h.update(q=w_out, e=h["st_estar"] + lam_out, lam_out=lam_out, need_rc=int(rc),
                 flags=(1 if ovf else 0) | (2 if unf else 0) | (4 if rc else 0) | 8)
        if not rc:
            h.update(shift=lam_out - h["st_lam"], max=mx, min=mn)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, d, l, p, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2307_00124_b200 import dist as D
        from paper_2307_00124_b200 import Scalar
        lo, hi = D.slab_ranges(l, world)[rank]
        ox, obb = ob.gen_uniform(d, l, p, 9, 1), ob.gen_sine(d, l, p)
        x, b = NpVec(d, l, lo, hi), NpVec(d, l, lo, hi)
        x.upload(ox.m, ox.q, ox.e)
        b.upload(obb.m, obb.q, obb.e)
        be = NumpyBackend()
        ds = D.DistStencil(D.TorchComm(be), be)
        res = []
        for (gm, ge, nn) in cases:
            out = NpVec(d, l, lo, hi)
            ds.gemv([D.Slab(rank, x)], [D.Slab(rank, b)], Scalar(-1, 1, 0), Scalar(1, 2, 0), p,
                    p + 5, Scalar(gm, 16, ge), [D.Slab(rank, out)], nn=nn)
            m = out.logical()
            # gather variable-length slabs to rank 0
            sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(sizes, torch.tensor([len(m)], dtype=torch.int64))
            mx_len = int(max(s.item() for s in sizes))
            buf = torch.zeros(mx_len, dtype=torch.int64)
            buf[: len(m)] = torch.from_numpy(m)
            bufs = [torch.zeros(mx_len, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(bufs, buf)
            full = np.concatenate([bufs[r][: int(sizes[r].item())].numpy() for r in range(world)])
            res.append((full.tolist(), out.h["e"], out.h["flags"]))
        if rank == 0:
            q.put(res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("d,l,world", [(2, 5, 2), (2, 5, 4), (3, 4, 2)])
def test_sharded_residual_gloo_matches_oracle(d, l, world):
    p = 12
    ox, obb = ob.gen_uniform(d, l, p, 9, 1), ob.gen_sine(d, l, p)
    want_exact, _ = ob.stencil_gemv(d, l, ox, obb, (-1, 1, 0), (1, 2, 0), "q", p, p + 5, 1 << 14, 0)
    top = int(np.max(np.abs(want_exact.m))).bit_length() + 1 + want_exact.e  # exact binade
    cases = [(1 << 14, top - 16, False),   # exact gamma: fast path
             (1 << 14, 2 * l + 2 - 16, False),   # overestimate: underflow -> recompute
             (1 << 14, -16, False),        # underestimate: overflow -> recompute
             (1 << 14, top - 16, True)]    # nnqcomp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, d, l, p, cases, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for (gm, ge, nn), (m, e, flags) in zip(cases, res):
        want, fl = ob.stencil_gemv(d, l, ox, obb, (-1, 1, 0), (1, 2, 0), "nn" if nn else "q", p,
                                   p + 5, gm, ge)
        assert e == want.e and m == want.m.tolist(), (gm, ge, nn)
        if not nn:
            assert bool(flags & 1) == bool(fl[0]) and bool(flags & 2) == bool(fl[1])


# ---------------------------------------------------------------------------
# sharded exact dot: per-rank limbs, int64 SUM all-reduce over gloo, exact value


class NumpyDotBackend:
    """Stand-in of the slab dot kernel: the slab's exact dot as carried 48-bit limbs."""

    def sync(self):
        pass

    def dot_limbs(self, x, y):
        from paper_2307_00124_b200 import dist as D
        v = sum(int(a) * int(b) for a, b in zip(x[0], y[0]))
        return torch.tensor(D.limbs_of(v) + [x[1] + y[1]], dtype=torch.int64)


def _dot_worker(rank, world, port, xs, ys, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2307_00124_b200 import dist as D
        n = len(xs[0][0])
        lo, hi = rank * n // world, (rank + 1) * n // world
        dd = D.DistDot(D.TorchComm(NumpyDotBackend()), NumpyDotBackend())
        out = []
        for (x, ex), (y, ey) in zip(xs, ys):
            out.append(dd.dot([D.Slab(rank, (x[lo:hi], ex))], [D.Slab(rank, (y[lo:hi], ey))]))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_exact_dot_gloo(world):
    """The dot all-reduce protocol over real processes: random 62-bit mantissas of both
    signs, and same-sign near-maximal ones whose sum leaves 128 bits (config 5's extreme
    is ~2^154); every rank ends with the exact global value."""
    import random
    r = random.Random(7)
    n = 4096
    xs = [([r.randrange(-(1 << 61), 1 << 61) for _ in range(n)], -5),
          ([(1 << 62) - 1 - 3 * i for i in range(n)], 0)]
    ys = [([r.randrange(-(1 << 61), 1 << 61) for _ in range(n)], 9),
          ([-((1 << 62) - 1) + 5 * i for i in range(n)], 2)]
    want = [(sum(a * b for a, b in zip(x, y)), ex + ey) for (x, ex), (y, ey) in zip(xs, ys)]
    assert want[1][0] < -(1 << 127)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dot_worker, args=(k, world, port, xs, ys, q))
             for k in range(world)]
    for pr in procs:
        pr.start()
    got = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, out in got:
        assert out == want, rank


def test_limbs_roundtrip_and_c_abi_value():
    """limbs_of / limbs_value, and the library's host-side bfp_dot_value (no GPU work)
    on uncarried limb sums of both signs."""
    import random
    import paper_2307_00124_b200 as B
    from paper_2307_00124_b200 import dist as D
    r = random.Random(3)
    for _ in range(200):
        v = r.randrange(-(1 << 190), 1 << 190)
        assert D.limbs_value(D.limbs_of(v)) == v
        # uncarried limbs as the device leaves them (< 2^59 each, top limb signed)
        parts = [r.randrange(-(1 << 150), 1 << 150) for _ in range(r.randrange(1, 9))]
        acc = [sum(x) for x in zip(*[D.limbs_of(p) for p in parts])]
        assert D.limbs_value(acc) == sum(parts)
        assert B.dot_value(acc + [0]) == sum(parts)
