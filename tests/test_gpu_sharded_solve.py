"""Sharded multigrid solve on one GPU: an in-process group of P ranks (slabs on the
fine levels, replicated coarse levels, LocalComm collectives) must reproduce the
unsharded solve bit-exactly -- final iterate, residual history and the trace of every
windowed op (flags, gamma, widths).  The NCCL transport swaps only the collectives
(bfp_solver.cu: NcclComm) and is exercised by `bench.py --gpus N` on N GPUs."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    import paper_2307_00124_b200 as B
    B.lib()
    return B


def _gathered_x(B, mg):
    parts, e0, ls = [], None, None
    for i in range(mg.local):
        x, r, rank, ls = mg.rank_result(i)
        assert rank == i
        m, q, e = x.download()
        assert e0 is None or e == e0
        e0 = e
        parts.append(m)
    return np.concatenate(parts), e0, ls


CASES = {
    # name: (mg_config kwargs, world, min_planes)
    "2d_ir_vcycles": (dict(d=2, l_fine=8, cycles=3, rhs_kind=1, p=20), 4, 8),
    "2d_ir_x0rand": (dict(d=2, l_fine=7, cycles=2, x0_random=True, rhs_kind=0, p=16, pd=[24] * 32,
                          w_add_cap=4), 2, 8),
    "2d_fmg_nnq": (dict(d=2, l_fine=8, l_coarse=3, cycles=1, rhs_kind=1, fmg=True,
                        nonnormalized=True, p=[0, 0, 0] + [4 + 2 * (l - 3) for l in range(3, 32)][:29]),
                   4, 8),
    "3d_fmg": (dict(d=3, l_fine=6, cycles=1, rhs_kind=1, fmg=True, p=24), 2, 4),
    "3d_fmg_w4": (dict(d=3, l_fine=6, cycles=1, rhs_kind=1, fmg=True, p=24), 4, 4),
    "3d_ir_int64": (dict(d=3, l_fine=6, cycles=2, x0_random=True, rhs_kind=2, p=40), 4, 4),
    "3d_fmg_l7": (dict(d=3, l_fine=7, cycles=1, rhs_kind=1, fmg=True, p=24), 2, 16),
    # int64 storage through the tiled marches (split-pair prolongation, strided restriction)
    "3d_fmg_l7_int64": (dict(d=3, l_fine=7, cycles=1, rhs_kind=1, fmg=True, p=40), 2, 16),
    # ... and l = 8: the tiled int64 stencil march and the int64 restriction (coarse l = 7) on slabs
    "3d_fmg_l8_int64": (dict(d=3, l_fine=8, cycles=1, rhs_kind=1, fmg=True, p=40), 2, 16),
}


@pytest.mark.parametrize("name", list(CASES))
def test_sharded_solve_matches_unsharded(B, name):
    kw, world, minp = CASES[name]
    cfg = B.mg_config(**kw)
    ref = B.Multigrid(cfg)
    ref.solve()
    x_ref, q_ref, e_ref, h_ref, t_ref = ref.result()
    for graph in (False, True):
        mg = B.Multigrid(cfg, world=world, min_planes=minp)
        mg.solve(use_graph=graph)
        mg.solve(use_graph=graph)  # replay: the plan re-initialises everything it reads
        x, q, e, hist, trace = mg.result()
        xs, es, ls = _gathered_x(B, mg)
        assert ls <= kw["l_fine"], "nothing was sharded"
        assert es == e_ref and np.array_equal(xs, x_ref), (name, graph)
        assert hist == h_ref, (name, graph)
        assert trace == t_ref, (name, graph)


@pytest.mark.parametrize("name", ["2d_ir_vcycles", "2d_fmg_nnq", "3d_fmg_w4", "3d_ir_int64"])
def test_sharded_solve_peer_mailbox_transport(B, name):
    """The peer-memory all-reduce of the window partials (bfp_solver.cu: Mailbox -- every rank
    posts {mu*, max, -min, err} + its op counter into every peer's mailbox, then reduces its
    own mailbox's slots) in place of the reduction kernel / ncclAllReduce: same bits for
    every rank count, stream-ordered and graph-replayed (the op counter lives on the
    device, so replays keep both slot parities consistent)."""
    kw, world, minp = CASES[name]
    cfg = B.mg_config(**kw)
    ref = B.Multigrid(cfg)
    ref.solve()
    x_ref, q_ref, e_ref, h_ref, t_ref = ref.result()
    B.set_transport(1)
    try:
        for graph in (False, True):
            mg = B.Multigrid(cfg, world=world, min_planes=minp)
            assert mg.transport() == "peer-mailbox"
            for _ in range(3):  # odd number of replays: both parities start a solve
                mg.solve(use_graph=graph)
            x, q, e, hist, trace = mg.result()
            xs, es, ls = _gathered_x(B, mg)
            assert es == e_ref and np.array_equal(xs, x_ref), (name, graph)
            assert hist == h_ref and trace == t_ref, (name, graph)
    finally:
        B.set_transport(0)
    assert B.Multigrid(cfg, world=world, min_planes=minp).transport() == "local-kernel"
