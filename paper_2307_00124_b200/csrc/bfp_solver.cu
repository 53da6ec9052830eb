// bfp_solver.cu -- native multigrid driver.
//
// Mirrors the reference solver structure (paths relative to /root/reference/proj):
//   run_step   src/multigrid.cpp:399-426   (one windowed op + trace record)
//   vcycle     src/multigrid.cpp:430-456   (correction scheme, here Jacobi V(nu1,nu2))
//   ir         src/multigrid.cpp:458-500   (iterative refinement, residual history)
//   fmg        src/multigrid.cpp:502-518   (zero_vec on the coarsest level, prolong, n_ir IR)
// with the frozen config semantics of DESIGN.md.  Because exponents, norms and
// gamma rules live in device headers, the whole solve is a static PLAN of
// kernel launches: built once, replayed stream-ordered or as one CUDA graph.
//
// Multi-rank: levels with at least `min_planes` planes per rank
// along the slowest axis are z-slab sharded (y-slabs in 2-D); coarser levels are
// replicated on every rank (identical integer work, so no scatter is needed).  Every
// rank builds the same plan over its own slabs; a sharded windowed op runs as
//   halo exchange -> pass-1 kernel (partial window) -> all-reduce MAX of
//   {mu*, max, -min, err} -> finalize -> [recompute pass -> all-reduce -> finalize]
// and the sharded -> replicated boundary restricts into a coarse slab and
// all-gathers it.  The collectives go through a Comm: NCCL (one rank per process,
// loaded at run time) or an in-process group of ranks sharing one device (tests).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "bfp_internal.h"

using namespace bfpdev;
using namespace bfp;

namespace {

// exponent all-reduce transport of the sharded solver (bfp_set_transport): 0 = default
// (in-process groups reduce with one kernel over the ranks' buffers; NCCL groups use the
// peer-memory mailboxes when CUDA IPC maps them, else ncclAllReduce), 1 = mailboxes also
// for in-process groups, 2 = never mailboxes
int g_transport = 0;

enum StepKind {
  ST_IR_RES = 0, ST_IR_CORR, ST_RELAX0, ST_RELAX, ST_V_RES, ST_RESTRICT, ST_V_CORR,
  ST_FMG_PROLONG, ST_FINAL_RES
};
enum OpKind { OK_ZERO, OK_UNIFORM, OK_GEMV, OK_JACOBI, OK_SCAL, OK_AXPBY, OK_RESTRICT,
              OK_PROLONG, OK_PCORR, OK_FUSED, OK_COPY, OK_GATHER };
enum { HALO_LO = 1, HALO_HI = 2 };

struct PlanOp {
  int kind;
  bfp_vec_s *a = nullptr, *b = nullptr, *out = nullptr;
  Scal s1{0, 0, 0}, s2{0, 0, 0};
  WinParams p{};  // (ops without a window -- zero_vec, copies -- keep it zeroed)
  int64_t q = 0;
  uint64_t seed = 0, sid = 0;
  std::vector<PlanOp> sub;  // OK_FUSED: the coarse-level ops run by one CTA
  FusedOp* dev = nullptr;
  ArenaEntry* arena = nullptr;  // vectors staged in shared memory (nullptr: global)
  int n_arena = 0, arena_bytes = 0, zoff = 0, loff = 0;
  int64_t* zbuf = nullptr;  // lean engine: global row buffer when shared memory is too small
  bool shard = false;  // output is a slab: partial window + collectives
  int halo = 0;        // HALO_LO / HALO_HI planes of `a` exchanged before the op
  int rep_e = kDefaultRep, rep_gs = 0;  // operator representation (reference mode)
  int st9 = 0;                          // 2-D 9-point operator (reference mode, d = 2)
};

int fused_kind(int k) {
  switch (k) {
    case OK_GEMV: return bfpdev::FK_GEMV;
    case OK_JACOBI: return bfpdev::FK_JACOBI;
    case OK_SCAL: return bfpdev::FK_SCAL;
    case OK_AXPBY: return bfpdev::FK_AXPBY;
    case OK_RESTRICT: return bfpdev::FK_RESTRICT;
    case OK_PROLONG: return bfpdev::FK_PROLONG;
    case OK_PCORR: return bfpdev::FK_PCORR;
    case OK_ZERO: return bfpdev::FK_ZERO;
  }
  return -1;
}
// Levels whose padded grid has at most this many points run inside one CTA (the lean coarse
// engine, bfp_lean.cuh).  Measured on B200 (tools/fuse_sweep.py, profiles/r2/r2b_fuse_sweep.txt):
// 4096 points is the best threshold in 2-D and 3-D (beyond it the rows no longer fit the
// CTA's shared memory); 1-D levels are cheap per launch and gain up to ~1024 points.
int64_t fuse_max_points(int d) {
#ifdef BFP_AB_ENV  // A/B measurement builds only
  static const int64_t v = [] {
    const char* e = getenv("BFP_FUSE_POINTS");
    return e ? (int64_t)atoll(e) : (int64_t)-1;
  }();
  if (v >= 0) return v;
#endif
  return d == 1 ? 1024 : 4096;
}

struct LevelBufs {
  int l = 0;
  int64_t p = 0;
  Scal c{0, 0, 0};
  bfp_vec_s *b = nullptr, *x[2] = {nullptr, nullptr}, *r[2] = {nullptr, nullptr};
  bfp_vec_s *e[2] = {nullptr, nullptr}, *rv = nullptr, *vr = nullptr;
  bfp_vec_s* vrs = nullptr;  // coarse slab of the restriction at the shard boundary
  bfp_vec_s* x0 = nullptr;   // sharded random initial iterate (copied in by the plan)
};

GTerm term(const bfp_vec_s* v, int64_t cm = 0, int64_t ce = 0, int kind = 0) {
  GTerm t;
  memset(&t, 0, sizeof(t));
  t.v = v ? v->hdr : nullptr;
  t.cm = cm;
  t.ce = ce;
  t.kind = kind;
  return t;
}
GammaRule rule(std::initializer_list<GTerm> ts) {
  GammaRule g;
  memset(&g, 0, sizeof(g));
  g.literal = 0;
  g.nterms = 0;
  for (const GTerm& t : ts) g.t[g.nterms++] = t;
  return g;
}

}  // namespace

struct RankSolver {
  bfp_mg_config_t cfg;
  int rank = 0, world = 1;
  int ls = 64;  // lowest sharded level (levels >= ls are slabs; 64 = none)
  int ebytes = 4;
  std::vector<LevelBufs> lev;  // indexed by level
  std::vector<PlanOp> plan;
  TraceRec* d_trace = nullptr;
  double* d_hist = nullptr;
  int n_trace = 0, n_hist = 0;
  bfp_vec_s* x_final = nullptr;
  bfp_vec_s* r_final = nullptr;
  cudaGraphExec_t graph = nullptr;
  int64_t launches_per_solve = 0;
  std::vector<bfp_vec_s*> owned;
  int err = 0;

  bool in_fused = false;
  bool fusion = true;
  int ir_iter = 0;  // 1-based iteration of the ir() loop being planned (hybrid mode)

  ~RankSolver() {
    for (auto& op : plan) {
      if (op.dev) cudaFree(op.dev);
      if (op.arena) cudaFree(op.arena);
      if (op.zbuf) cudaFree(op.zbuf);
    }
    if (graph) cudaGraphExecDestroy(graph);
    for (auto* v : owned) vec_free(v);
    cudaFree(d_trace);
    cudaFree(d_hist);
  }

  bool sharded(int l) const { return l >= ls; }
  // this rank's planes [lo, hi) of level l along the slowest axis
  void slab(int l, int* lo, int* hi) const {
    const int n = (1 << l) / world;
    *lo = rank * n;
    *hi = *lo + n;
  }
  bfp_vec_s* vec(int l, bool full = false) {
    bfp_vec_s* v = nullptr;
    int rc;
    if (sharded(l) && !full) {
      int lo, hi;
      slab(l, &lo, &hi);
      rc = vec_alloc_slab(cfg.d, l, 0, lo, hi, ebytes, &v);
    } else {
      rc = vec_alloc(cfg.d, l, 0, ebytes, &v);
    }
    if (rc) {
      err = rc;
      return nullptr;
    }
    owned.push_back(v);
    return v;
  }

  // run_step: one windowed op (qcomp, or nnqcomp in nonnormalized mode)
  int64_t wd(int l) const { return cfg.pd[l] ? cfg.pd[l] : cfg.p[l]; }
  int64_t wc(int l) const { return cfg.pc[l] ? cfg.pc[l] : cfg.p[l]; }

  void step(int st, int level, PlanOp op, int64_t w_out, const GammaRule& g, int w_add,
            bool hist = false) {
    // NormMode (P/src/multigrid.cpp:403-409): 0 normalized, 1 nonnormalized,
    // 2 hybrid = qcomp only for the IR residual of iterations <= 2
    const bool normalized = cfg.nonnormalized == 0 || st == ST_FINAL_RES ||
                            (cfg.nonnormalized == 2 && st == ST_IR_RES && ir_iter <= 2);
    if (cfg.w_add_cap >= 0 && w_add > cfg.w_add_cap) w_add = cfg.w_add_cap;
    op.p = win_params(normalized ? MODE_QCOMP : MODE_NNQ, w_out, w_out + w_add, 0);
    op.p.gamma = g;
    op.p.trace_slot = n_trace++;
    op.p.step = st;
    op.p.level = level;
    if (hist) op.p.hist_slot = n_hist++;
    mark(op);
    plan.push_back(op);
  }
  void mark(PlanOp& op) const {
    if (!op.out || op.out->nz == (1 << op.out->l) || op.out->dim < 2) return;  // full grid
    op.shard = true;
    switch (op.kind) {
      case OK_GEMV: case OK_JACOBI: op.halo = HALO_LO | HALO_HI; break;
      case OK_RESTRICT: op.halo = HALO_HI; break;
      case OK_PROLONG: case OK_PCORR:
        op.halo = op.a->nz == (1 << op.a->l) ? 0 : HALO_LO;  // replicated coarse: no halo
        break;
      default: op.halo = 0;
    }
  }

  bool fusable(int l) const {
    int64_t pts = 1;
    for (int a = 0; a < cfg.d; ++a) pts <<= l;
    const int64_t lim = cfg.fuse_points >= 0 ? cfg.fuse_points : fuse_max_points(cfg.d);
    return fusion && !sharded(l) && !in_fused && pts <= lim;
  }
  // run body() with its plan ops collected into one OK_FUSED op
  template <typename F> bfp_vec_s* fused(F body) {
    const size_t i0 = plan.size();
    in_fused = true;
    bfp_vec_s* res = body();
    in_fused = false;
    PlanOp f;
    f.kind = OK_FUSED;
    f.sub.assign(plan.begin() + i0, plan.end());
    plan.resize(i0);
    plan.push_back(std::move(f));
    return res;
  }

  bfp_vec_s* vcycle(int l, bfp_vec_s* r) {
    if (fusable(l)) return fused([&]() { return vcycle(l, r); });
    LevelBufs& L = lev[l];
    bfp_vec_s *e = L.e[0], *t = L.e[1];
    PlanOp o;
    o.kind = OK_SCAL;
    o.a = r;
    o.out = e;
    o.s1 = L.c;
    step(ST_RELAX0, l, o, wd(l), rule({term(r, L.c.m, L.c.e)}), 2);
    const int sweeps = l == cfg.l_coarse ? cfg.n_coarse : cfg.nu1;
    auto jac = [&]() {
      PlanOp j;
      j.kind = OK_JACOBI;
      j.a = e;
      j.b = r;
      j.out = t;
      j.s1 = L.c;
      step(ST_RELAX, l, j, wd(l), rule({term(e), term(r, L.c.m, L.c.e)}), 3);
      std::swap(e, t);
    };
    for (int s = 1; s < sweeps; ++s) jac();
    if (l == cfg.l_coarse) return e;
    PlanOp g;
    g.kind = OK_GEMV;
    g.a = e;
    g.b = r;
    g.out = L.rv;
    g.s1 = Scal{-1, 1, 0};
    g.s2 = Scal{1, 2, 0};
    step(ST_V_RES, l, g, wd(l), rule({term(r)}), 4);
    LevelBufs& Lc = lev[l - 1];
    PlanOp rs;
    rs.kind = OK_RESTRICT;
    rs.a = L.rv;
    const bool boundary = sharded(l) && !sharded(l - 1);
    rs.out = boundary ? Lc.vrs : Lc.vr;
    step(ST_RESTRICT, l, rs, wd(l), rule({term(L.rv)}), 6);
    if (boundary) {  // coarse slabs -> the replicated coarse vector on every rank
      PlanOp g;
      g.kind = OK_GATHER;
      g.a = Lc.vrs;
      g.out = Lc.vr;
      plan.push_back(g);
    }
    bfp_vec_s* ec = vcycle(l - 1, Lc.vr);
    PlanOp pc;
    pc.kind = OK_PCORR;
    pc.a = ec;
    pc.b = e;
    pc.out = t;
    step(ST_V_CORR, l, pc, wd(l), rule({term(e), term(ec)}), 2);
    std::swap(e, t);
    for (int s = 0; s < cfg.nu2; ++s) jac();
    return e;
  }

  // returns the buffer holding the final iterate; r_last gets the last residual buffer
  bfp_vec_s* ir(int l, bfp_vec_s* x, int iters, bfp_vec_s** r_last) {
    LevelBufs& L = lev[l];
    int ri = 0;
    bfp_vec_s* r_prev = nullptr;
    for (int i = 1; i <= iters; ++i) {
      const bool first = r_prev == nullptr;
      GammaRule g = first ? rule({term(L.b), term(x, 4 * cfg.d, 2 * l, 1)}) : rule({term(r_prev)});
      bfp_vec_s* r = L.r[ri];
      ri ^= 1;
      PlanOp o;
      o.kind = OK_GEMV;
      o.a = x;
      o.b = L.b;
      o.out = r;
      o.s1 = Scal{-1, 1, 0};
      o.s2 = Scal{1, 2, 0};
      ir_iter = i;
      step(ST_IR_RES, l, o, wd(l), g, first ? 5 : 4, true);
      r_prev = r;
      bfp_vec_s* e = vcycle(l, r);
      bfp_vec_s* xn = (x == L.x[0]) ? L.x[1] : L.x[0];
      PlanOp c;
      c.kind = OK_AXPBY;
      c.a = x;
      c.b = e;
      c.out = xn;
      c.s1 = Scal{1, 2, 0};
      c.s2 = Scal{1, 2, 0};
      step(ST_IR_CORR, l, c, L.p, rule({term(x), term(e)}), 1);
      x = xn;
    }
    *r_last = r_prev;
    return x;
  }

  void final_residual(int l, bfp_vec_s* x, bfp_vec_s* r_last) {
    LevelBufs& L = lev[l];
    bfp_vec_s* r = (r_last == L.r[0]) ? L.r[1] : L.r[0];
    PlanOp o;
    o.kind = OK_GEMV;
    o.a = x;
    o.b = L.b;
    o.out = r;
    o.s1 = Scal{-1, 1, 0};
    o.s2 = Scal{1, 2, 0};
    step(ST_FINAL_RES, l, o, wd(l), rule({term(r_last)}), 4, true);
    r_final = r;
  }

  bfp_vec_s* fmg(int l) {
    if (fusable(l)) return fused([&]() { return fmg(l); });
    LevelBufs& L = lev[l];
    bfp_vec_s* x = L.x[0];
    if (l == cfg.l_coarse) {
      PlanOp z;
      z.kind = OK_ZERO;
      z.out = x;
      z.q = L.p;
      plan.push_back(z);
    } else {
      bfp_vec_s* xc = fmg(l - 1);
      PlanOp o;
      o.kind = OK_PROLONG;
      o.a = xc;
      o.out = x;
      step(ST_FMG_PROLONG, l, o, L.p, rule({term(xc)}), 1);
    }
    bfp_vec_s* r_last = nullptr;
    x = ir(l, x, cfg.cycles, &r_last);
    if (l == cfg.l_fine && r_last) final_residual(l, x, r_last);
    return x;
  }

  int min_planes = 16;
  // slab of a replicated level aligned with the sharded level above it
  bfp_vec_s* vec_slab_of(int l) {
    int lo, hi;
    slab(l + 1, &lo, &hi);
    bfp_vec_s* v = nullptr;
    int rc = vec_alloc_slab(cfg.d, l, 0, lo / 2, hi / 2, ebytes, &v);
    if (rc) {
      err = rc;
      return nullptr;
    }
    owned.push_back(v);
    return v;
  }
  // copy this rank's planes (and the header) of a full grid into its slab (setup only)
  int cut_slab(bfp_vec_s* full, bfp_vec_s* s) {
    const int64_t pb = (s->span / s->nz) * s->ebytes;
    if (cudaMemcpy(s->data, (char*)full->data + s->z0 * pb, s->nz * pb,
                   cudaMemcpyDeviceToDevice) != cudaSuccess ||
        cudaMemcpy(s->hdr, full->hdr, sizeof(Hdr), cudaMemcpyDeviceToDevice) != cudaSuccess)
      return BFP_ERR_CUDA;
    return BFP_OK;
  }

  // ---- reference-algorithm mode (cfg.ref_mode, d = 1 or 2) ---------------------------
  // exact gamma terms: X = norm of v, coefficient c (128-bit + sticky) 2^ce
  static GTerm xterm(const bfp_vec_s* v, const bfp_xf_t& c) {
    GTerm t;
    memset(&t, 0, sizeof(t));
    t.v = v->hdr;
    t.cm = (int64_t)c.lo;
    t.cm_hi = c.hi;
    t.ce = c.e;
    t.sticky = c.sticky;
    return t;
  }
  static bfp_xf_t xint(uint64_t v) { return bfp_xf_t{0, v, 0, 0, 0}; }
  static GammaRule xrule(std::initializer_list<GTerm> ts) {
    GammaRule g = rule(ts);
    g.exact = 1;
    return g;
  }
  int64_t wr(int l) const { return cfg.p[l]; }
  bfp_vec_s* ref_last[33] = {};  // last IR residual buffer per level (SolverContext)
  // operator representations of quantize_csr at width w (pyref_refmode.quantize_values),
  // as (kernel base stencil / taps) * 2^gs with exponent e:
  //   1-D  A = tridiag(-1/2, 1, -1/2): 2^(w-3) (2, -1),     e_A = 2 - w
  //        P = [1/2, 1, 1/2]:          2^(w-3) tap sums,    e_P = 2 - w
  //        R = 2 P^T = (1, 2, 1):      2^(w-3) (1, 2, 1),   e_R = 3 - w
  //   2-D  A = (1, -1/8 x 8):          2^(w-5) (8, -1 x 8), e_A = 2 - w   (9-point)
  //        P = P1 (x) P1 (1, 1/2, 1/4): 2^(w-4) tap sums,   e_P = 2 - w
  //        R = P^T (D_f = D_c):        2^(w-4) (1,2,1)^2,   e_R = 2 - w
  int ref_a_gs(int w) const { return cfg.d == 1 ? w - 3 : w - 5; }
  int ref_p_gs(int w) const { return cfg.d == 1 ? w - 3 : w - 4; }
  int ref_r_e(int w) const { return cfg.d == 1 ? 3 - w : 2 - w; }
  PlanOp ref_gemv(bfp_vec_s* x, bfp_vec_s* y, Scal al, Scal be, int w, bfp_vec_s* out) {
    PlanOp o;
    o.kind = OK_GEMV;
    o.a = x;
    o.b = y;
    o.out = out;
    o.s1 = al;
    o.s2 = be;
    o.rep_e = 2 - w;
    o.rep_gs = ref_a_gs(w);
    o.st9 = cfg.d == 2;
    return o;
  }
  bfp_vec_s* vcycle_ref(int l, bfp_vec_s* r) {  // P/src/multigrid.cpp:430-456
    LevelBufs& L = lev[l];
    const int wd = (int)wd_(l);
    bfp_vec_s *y = L.e[0], *y2 = L.e[1];
    const Scal c1d{cfg.ref_c1d[l].m, cfg.ref_c1d[l].q, cfg.ref_c1d[l].e};
    const Scal c2d{cfg.ref_c2d[l].m, cfg.ref_c2d[l].q, cfg.ref_c2d[l].e};
    step(ST_RELAX, l, ref_gemv(r, r, c2d, c1d, wd, y), wd, xrule({xterm(r, cfg.ref_c1)}), 2);
    if (l > 1) {
      step(ST_V_RES, l, ref_gemv(y, r, Scal{1, 2, 0}, Scal{-1, 1, 0}, wd, L.rv), wd,
           xrule({xterm(r, cfg.ref_kres)}), 4);
      LevelBufs& Lc = lev[l - 1];
      PlanOp rs;
      rs.kind = OK_RESTRICT;
      rs.a = L.rv;
      rs.out = Lc.vr;
      rs.rep_e = ref_r_e(wd);
      rs.rep_gs = ref_p_gs(wd);
      step(ST_RESTRICT, l, rs, wd, xrule({xterm(L.rv, xint(4))}), 6);
      bfp_vec_s* d = vcycle_ref(l - 1, Lc.vr);
      PlanOp pc;
      pc.kind = OK_PCORR;
      pc.a = d;
      pc.b = y;
      pc.out = y2;
      pc.s1 = Scal{-1, 1, 0};
      pc.s2 = Scal{1, 2, 0};
      pc.rep_e = 2 - wd;
      pc.rep_gs = ref_p_gs(wd);
      step(ST_V_CORR, l, pc, wd, xrule({xterm(y, xint(1)), xterm(d, xint(1))}), 1);
      y = y2;
    }
    return y;
  }
  // IR (P/src/multigrid.cpp:458-500, tol < 0): returns the final iterate
  bfp_vec_s* ir_ref(int l, bfp_vec_s* x, int iters) {
    LevelBufs& L = lev[l];
    for (int i = 1; i <= iters; ++i) {
      GammaRule g;
      if (i > 1)
        g = xrule({xterm(ref_last[l], xint(1))});
      else if (l > 1 && ref_last[l - 1])
        g = xrule({xterm(ref_last[l - 1], xint(1))});
      else
        g = xrule({xterm(x, xint(2)), xterm(L.b, xint(1))});  // ||A||_inf = 2
      bfp_vec_s* r = (ref_last[l] == L.r[0]) ? L.r[1] : L.r[0];
      const int wc = (int)wc_(l);
      ir_iter = i;
      step(ST_IR_RES, l, ref_gemv(x, L.b, Scal{1, 2, 0}, Scal{-1, 1, 0}, wc, r), wd_(l), g,
           i == 1 ? 5 : 4, true);
      ref_last[l] = r;
      bfp_vec_s* y = vcycle_ref(l, r);
      bfp_vec_s* xn = (x == L.x[0]) ? L.x[1] : L.x[0];
      PlanOp c;
      c.kind = OK_AXPBY;
      c.a = x;
      c.b = y;
      c.out = xn;
      c.s1 = Scal{1, 2, 0};
      c.s2 = Scal{-1, 1, 0};
      step(ST_IR_CORR, l, c, wr(l), xrule({xterm(x, xint(1)), xterm(y, xint(1))}), 0);
      x = xn;
    }
    return x;
  }
  bfp_vec_s* fmg_ref(int l) {  // P/src/multigrid.cpp:502-518
    LevelBufs& L = lev[l];
    bfp_vec_s* x = L.x[0];
    if (l == 1) {
      PlanOp z;
      z.kind = OK_ZERO;
      z.out = x;
      z.q = wr(1);
      plan.push_back(z);
    } else {
      bfp_vec_s* xc = fmg_ref(l - 1);
      PlanOp o;
      o.kind = OK_PROLONG;
      o.a = xc;
      o.out = x;
      o.rep_e = 2 - (int)wr(l);
      o.rep_gs = ref_p_gs((int)wr(l));
      step(ST_FMG_PROLONG, l, o, wr(l), xrule({xterm(xc, xint(1))}), 0);
    }
    for (int k = 0; k < cfg.cycles; ++k) x = ir_ref(l, x, 1);
    return x;
  }
  int64_t wd_(int l) const { return wd(l); }
  int64_t wc_(int l) const { return wc(l); }
  int build_ref() {
    const int lf = cfg.l_fine;
    if (cfg.d != 1 && cfg.d != 2) return BFP_ERR_ARG;
    // the operators' quantize_csr representations are exact from w = 3 (1-D) / 5 (2-D)
    const int wmin = cfg.d == 1 ? 3 : 5;
    int maxw = 0;
    for (int l = 1; l <= lf; ++l) {
      if (wr(l) < wmin || wd(l) < wmin || wc(l) < wmin) return BFP_ERR_ARG;
      const int cap = cfg.w_add_cap >= 0 ? std::min(cfg.w_add_cap, 6) : 6;
      maxw = std::max(maxw, (int)std::max(std::max(wd(l), wr(l)), wc(l)) + cap);
    }
    ebytes = maxw <= 32 ? 4 : 8;
    lev.assign(lf + 1, LevelBufs());
    for (int l = 1; l <= lf; ++l) {
      LevelBufs& L = lev[l];
      L.l = l;
      L.p = wr(l);
      L.b = vec(l);
      L.x[0] = vec(l);
      L.x[1] = vec(l);
      L.r[0] = vec(l);
      L.r[1] = vec(l);
      L.e[0] = vec(l);
      L.e[1] = vec(l);
      if (l > 1) L.rv = vec(l);
      if (l < lf) L.vr = vec(l);
      if (err) return err;
    }
    for (int l = 1; l <= lf; ++l) {  // right-hand sides (setup): D^-1 b at wcheck
      LevelBufs& L = lev[l];
      if (!cfg.fmg && l != lf) continue;
      int rc;
      if (cfg.rhs_kind == 1) {
        rc = gen_sine(L.b, wc(l), 0);
        if (!rc) {  // h^2 / 2^d * d pi^2 prod sin: exponent shift, the mantissas are unchanged
          Hdr h;
          if (cudaMemcpy(&h, L.b->hdr, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess)
            return BFP_ERR_CUDA;
          if (h.max_m != 0 || h.min_m != 0) h.e -= 2 * l + cfg.d;
          if (cudaMemcpy(L.b->hdr, &h, sizeof(h), cudaMemcpyHostToDevice) != cudaSuccess)
            return BFP_ERR_CUDA;
        }
      } else if (cfg.rhs_kind == 0) {
        rc = gen_uniform(L.b, wc(l), cfg.seed, 2, 0);
      } else {
        rc = set_zero(L.b, wc(l), 0);
      }
      if (rc) return rc;
    }
    if (cfg.fmg) {
      x_final = fmg_ref(lf);
    } else {
      LevelBufs& L = lev[lf];
      PlanOp init;
      init.out = L.x[0];
      init.q = L.p;
      if (cfg.x0_random == 1) {
        init.kind = OK_UNIFORM;
        init.seed = cfg.seed;
        init.sid = 1;
      } else {
        init.kind = OK_ZERO;
      }
      if (cfg.x0_random != 2) plan.push_back(init);  // 2: the caller's x0 (bfp_mg_vectors)
      x_final = ir_ref(lf, L.x[0], cfg.cycles);
    }
    return finish_build();
  }

  int build() {
    if (cfg.ref_mode) return build_ref();
    const int lf = cfg.l_fine, lc = cfg.l_coarse;
    int maxp = 0;
    for (int l = lc; l <= lf; ++l) {
      const int cap = cfg.w_add_cap >= 0 ? std::min(cfg.w_add_cap, 6) : 6;
      maxp = std::max(maxp, std::max<int>((int)std::max(wd(l), (int64_t)cfg.p[l]) + cap, (int)wc(l)));
    }
    ebytes = maxp <= 32 ? 4 : 8;
    ls = 64;
    if (world > 1 && cfg.d >= 2)
      for (int l = lf; l >= lc && ((1 << l) / world) >= std::max(min_planes, 2); --l) ls = l;
    lev.assign(lf + 1, LevelBufs());
    for (int l = lc; l <= lf; ++l) {
      LevelBufs& L = lev[l];
      L.l = l;
      L.p = cfg.p[l];
      int64_t cm, ce;
      jacobi_coeff(cfg.d, l, cfg.qc, &cm, &ce);
      L.c = Scal{cm, cfg.qc, ce};
      const bool need_rhs = cfg.fmg || l == lf;
      if (need_rhs) {
        L.b = vec(l);
        L.x[0] = vec(l);
        L.x[1] = vec(l);
        L.r[0] = vec(l);
        L.r[1] = vec(l);
      }
      L.e[0] = vec(l);
      L.e[1] = vec(l);
      if (l > lc) L.rv = vec(l);
      if (l < lf) L.vr = vec(l);
      if (l < lf && !sharded(l) && sharded(l + 1)) L.vrs = vec_slab_of(l);
      if (err) return err;
    }
    // inputs (setup, outside the solve): right-hand sides
    for (int l = lc; l <= lf; ++l) {
      LevelBufs& L = lev[l];
      if (!L.b) continue;
      // generators normalise over the whole grid: a slab is cut from the full vector
      bfp_vec_s* full = L.b;
      if (sharded(l) && vec_alloc(cfg.d, l, 0, ebytes, &full)) return BFP_ERR_NOMEM;
      int rc;
      if (cfg.rhs_kind == 1)
        rc = gen_sine(full, wc(l), 0);
      else if (cfg.rhs_kind == 0)
        rc = gen_uniform(full, wc(l), cfg.seed, 2, 0);
      else
        rc = set_zero(full, wc(l), 0);
      if (!rc && full != L.b) rc = cut_slab(full, L.b);
      if (full != L.b) vec_free(full);
      if (rc) return rc;
    }
    // the plan
    if (cfg.fmg) {
      x_final = fmg(lf);
    } else {
      LevelBufs& L = lev[lf];
      PlanOp init;
      init.out = L.x[0];
      if (cfg.x0_random == 1 && sharded(lf)) {
        bfp_vec_s* full = nullptr;
        if (vec_alloc(cfg.d, lf, 0, ebytes, &full)) return BFP_ERR_NOMEM;
        L.x0 = vec(lf);
        int rc = err ? err : gen_uniform(full, L.p, cfg.seed, 1, 0);
        if (!rc) rc = cut_slab(full, L.x0);
        vec_free(full);
        if (rc) return rc;
        init.kind = OK_COPY;
        init.a = L.x0;
      } else if (cfg.x0_random == 1) {
        init.kind = OK_UNIFORM;
        init.q = L.p;
        init.seed = cfg.seed;
        init.sid = 1;
      } else {
        init.kind = OK_ZERO;
        init.q = L.p;
      }
      if (cfg.x0_random != 2 || world > 1) plan.push_back(init);  // 2: the caller's x0
      bfp_vec_s* r_last = nullptr;
      x_final = ir(lf, L.x[0], cfg.cycles, &r_last);
      if (r_last) final_residual(lf, x_final, r_last);
    }
    return finish_build();
  }

  int finish_build() {
    if (cudaMalloc(&d_trace, sizeof(TraceRec) * std::max(n_trace, 1)) != cudaSuccess ||
        cudaMalloc(&d_hist, sizeof(double) * std::max(n_hist, 1)) != cudaSuccess)
      return BFP_ERR_NOMEM;
    cudaMemset(d_trace, 0, sizeof(TraceRec) * std::max(n_trace, 1));
    cudaMemset(d_hist, 0, sizeof(double) * std::max(n_hist, 1));
    std::vector<PlanOp> built;
    built.reserve(plan.size());
#ifdef BFP_DEBUG_BUILD
    fprintf(stderr, "finish_build: %zu plan ops\n", plan.size());
#endif
    for (auto& op : plan) {
      op.p.trace = d_trace;
      op.p.hist = op.p.hist_slot >= 0 ? d_hist : nullptr;
      if (op.kind != OK_FUSED) {
        built.push_back(std::move(op));
        continue;
      }
      std::vector<FusedOp> h(op.sub.size());
#ifdef BFP_DEBUG_BUILD
      fprintf(stderr, "fused list of %zu ops\n", op.sub.size());
#endif
      for (size_t i = 0; i < op.sub.size(); ++i) {
        PlanOp& so = op.sub[i];
        so.p.trace = d_trace;
        so.p.hist = so.p.hist_slot >= 0 ? d_hist : nullptr;
        const int fk = fused_kind(so.kind);
        if (fk < 0) return BFP_ERR_ARG;
        int rc = fused_make(fk, so.a, so.b, so.s1, so.s2, so.p, so.q, so.out, &h[i]);
        if (rc) return rc;
      }
      for (size_t i = 0; i + 1 < h.size(); ++i)
        h[i].lr.nnq_next = h[i + 1].kind != bfpdev::FK_ZERO && h[i + 1].p.mode == MODE_NNQ;
#ifdef BFP_DEBUG_BUILD
      fprintf(stderr, "  made, building arena\n");
#endif
      if (!build_arena(op, h)) {
        // the list's state does not fit one CTA's shared memory: one launch per op instead
        if (err) return err;
        for (auto& so : op.sub) built.push_back(std::move(so));
        continue;
      }
      if (cudaMalloc(&op.dev, sizeof(FusedOp) * h.size()) != cudaSuccess) return BFP_ERR_NOMEM;
      cudaMemcpy(op.dev, h.data(), sizeof(FusedOp) * h.size(), cudaMemcpyHostToDevice);
      built.push_back(std::move(op));
    }
    plan = std::move(built);
#ifdef BFP_DEBUG_BUILD
    fprintf(stderr, "finish_build done: %zu ops\n", plan.size());
#endif
    return cudaDeviceSynchronize() == cudaSuccess ? BFP_OK : BFP_ERR_CUDA;
  }


  // Stage the state of a fused op list in the CTA's shared memory: every block header the
  // list touches (always), and the vectors' data while it fits (smallest first); Vec and
  // gamma-term pointers become arena byte offsets.  Vectors the list writes are copied back
  // when the launch ends.
  bool build_arena(PlanOp& op, std::vector<FusedOp>& h) {
    std::vector<bfp_vec_s*> vs;
    std::vector<char> written;
    auto find = [&](const Hdr* hp) -> bfp_vec_s* {
      for (auto* v : owned)
        if (v->hdr == hp) return v;
      return nullptr;
    };
    auto note = [&](const Hdr* hp, bool w) {
      bfp_vec_s* v = find(hp);
      if (!v) return false;
      auto it = std::find(vs.begin(), vs.end(), v);
      if (it == vs.end()) {
        vs.push_back(v);
        written.push_back(w);
      } else if (w) {
        written[it - vs.begin()] = 1;
      }
      return true;
    };
    auto visit = [&](FusedOp& f, auto&& fn) {
      switch (f.kind) {
        case bfpdev::FK_GEMV: fn(f.u.gemv.x); fn(f.u.gemv.y); break;
        case bfpdev::FK_JACOBI: fn(f.u.jac.x); fn(f.u.jac.b); break;
        case bfpdev::FK_SCAL: fn(f.u.scal.r); break;
        case bfpdev::FK_AXPBY: fn(f.u.axpby.x); fn(f.u.axpby.y); break;
        case bfpdev::FK_RESTRICT: fn(f.u.rst.r); break;
        case bfpdev::FK_PROLONG: fn(f.u.pro.xc); break;
        case bfpdev::FK_PCORR: fn(f.u.pc.ec); fn(f.u.pc.y); break;
      }
    };
    // the lean engine's row buffer (8 bytes per output element of the largest op): shared
    // memory when it fits next to the headers, else a global scratch buffer
    int64_t zbytes = 0;
    if (ebytes == 4)
      for (auto& f : h) zbytes = std::max<int64_t>(zbytes, f.out.n * 8);
    zbytes = (zbytes + 127) / 128 * 128;
    auto zglobal = [&]() {
      op.zoff = 0;
      if (zbytes && cudaMalloc(&op.zbuf, zbytes) != cudaSuccess) err = BFP_ERR_NOMEM;
    };
    bool ok = true;
    for (auto& f : h) {
      ok = ok && note(f.out.hdr, true);
      visit(f, [&](bfpdev::Vec& v) { ok = ok && note(v.hdr, false); });
      if (!f.p.gamma.literal)
        for (int i = 0; i < f.p.gamma.nterms; ++i)
          if (f.p.gamma.t[i].v) ok = ok && note(f.p.gamma.t[i].v, false);
    }
#ifdef BFP_DEBUG_BUILD
    fprintf(stderr, "  arena: ok=%d vectors=%zu ops=%zu\n", (int)ok, vs.size(), h.size());
#endif
    if (!ok || vs.size() > (size_t)bfpdev::kLeanMaxVec || h.size() > 30000) return false;
    std::vector<ArenaEntry> ar(vs.size());
    int64_t off = 128;  // offset 0 is reserved (nullptr gamma terms)
    for (size_t k = 0; k < vs.size(); ++k) {
      ArenaEntry& e = ar[k];
      memset(&e, 0, sizeof(e));
      e.gbase = vs[k]->base;
      e.ghdr = vs[k]->hdr;
      e.wb = written[k];
      e.hoff = (int32_t)off;
      off += (sizeof(Hdr) + 127) / 128 * 128;
    }
    // the lean engine's per-op log
    op.loff = (int)off;
    if (ebytes == 4) off += ((int64_t)h.size() * 48 + 127) / 128 * 128;
    if (off > bfpdev::kArenaMaxBytes) return false;
    if (off + zbytes <= bfpdev::kArenaMaxBytes) {
      op.zoff = (int)off;
      off += zbytes;
    } else {
      zglobal();
    }
    std::vector<size_t> order(vs.size());
    for (size_t k = 0; k < order.size(); ++k) order[k] = k;
    auto vbytes = [&](size_t k) {
      return ((vs[k]->span + 2 * vs[k]->halo) * vs[k]->ebytes + 15) / 16 * 16;
    };
    std::stable_sort(order.begin(), order.end(),
                     [&](size_t x, size_t y) { return vbytes(x) < vbytes(y); });
    for (size_t k : order) {
      const int64_t b = vbytes(k), pad = (b + 127) / 128 * 128;
      if (off + pad > bfpdev::kArenaMaxBytes) break;
      ar[k].bytes = b;
      ar[k].off = (int32_t)off;
      off += pad;
    }
    for (auto& f : h) {
      // every rewritten pointer is marked in f.rb (the lean engine rebases on fetch)
      auto mark = [&](const void* field) {
        const size_t w = ((const char*)field - (const char*)&f) / 8;
        f.rb[w >> 6] |= 1ull << (w & 63);
      };
      auto remap = [&](bfpdev::Vec& v) {
        for (size_t k = 0; k < vs.size(); ++k)
          if (vs[k]->hdr == v.hdr) {
            if (ar[k].bytes) {
              v.data = (void*)(uintptr_t)(ar[k].off + vs[k]->halo * vs[k]->ebytes);
              mark(&v.data);
            }
            v.hdr = (Hdr*)(uintptr_t)ar[k].hoff;
            mark(&v.hdr);
            return;
          }
      };
      if (!f.p.gamma.literal)
        for (int i = 0; i < f.p.gamma.nterms; ++i)
          if (f.p.gamma.t[i].v)
            for (size_t k = 0; k < vs.size(); ++k)
              if (vs[k]->hdr == f.p.gamma.t[i].v) {
                f.p.gamma.t[i].v = (const Hdr*)(uintptr_t)ar[k].hoff;
                mark(&f.p.gamma.t[i].v);
                break;
              }
      remap(f.out);
      visit(f, remap);
      // the lean digest: vector ids (header offsets -> index) and the operands' data
      constexpr int64_t kStride = (sizeof(Hdr) + 127) / 128 * 128;
      auto vid = [&](const void* hdr_off) { return (uint8_t)(((uintptr_t)hdr_off - 128) / kStride); };
      auto dptr = [&](const void** slot, const void* data) {
        *slot = data;
        if ((uintptr_t)data != 0 && (uintptr_t)data < (uintptr_t)bfpdev::kArenaMaxBytes) mark(slot);
      };
      bfpdev::LeanRec& lr = f.lr;
      lr.vout = vid(f.out.hdr);
      dptr((const void**)&lr.out, f.out.data);
      int na = 0;
      visit(f, [&](bfpdev::Vec& v) {
        if (na == 0) {
          lr.va = vid(v.hdr);
          dptr((const void**)&lr.x, v.data);
        } else {
          lr.vb = vid(v.hdr);
          dptr((const void**)&lr.y, v.data);
        }
        ++na;
      });
      if (!f.p.gamma.literal)
        for (int i = 0; i < f.p.gamma.nterms && i < 3; ++i)
          if (f.p.gamma.t[i].v) lr.gv[i] = vid(f.p.gamma.t[i].v);
    }
    static_assert(sizeof(FusedOp) <= 128 * 8, "FusedOp::rb marks at most 128 words");
    if (cudaMalloc(&op.arena, sizeof(ArenaEntry) * ar.size()) != cudaSuccess) {
      err = BFP_ERR_NOMEM;
      return false;
    }
    cudaMemcpy(op.arena, ar.data(), sizeof(ArenaEntry) * ar.size(), cudaMemcpyHostToDevice);
    op.n_arena = (int)ar.size();
    op.arena_bytes = (int)off;
    return err == 0;
  }

  // one op on this rank; `part` != nullptr runs a windowed op as a partial window
  // (pass 1 with stage 0, the recompute pass with stage 1)
  int run(const PlanOp& op, cudaStream_t s, int64_t* part = nullptr, int stage = 0) {
    WinParams p = op.p;
    if (part) {
      p.part = part;
      if (stage == 1) p.mode = MODE_RECOMPUTE;
    }
    switch (op.kind) {
      case OK_ZERO: return set_zero(op.out, op.q, s);
      case OK_UNIFORM: return gen_uniform(op.out, op.q, op.seed, op.sid, s);
      case OK_GEMV:
        return op_gemv(op.a, op.b, op.s1, op.s2, p, op.out, s, op.rep_e, op.rep_gs, op.st9);
      case OK_JACOBI: return op_jacobi(op.a, op.b, op.s1, p, op.out, s);
      case OK_SCAL: return op_scal(op.a, op.s1, p, op.out, s);
      case OK_AXPBY: return op_axpby(op.a, op.b, op.s1, op.s2, p, op.out, s);
      case OK_RESTRICT: return op_restrict(op.a, p, op.out, s, op.rep_e, op.rep_gs);
      case OK_PROLONG: return op_prolong(op.a, p, op.out, s, op.rep_e, op.rep_gs);
      case OK_PCORR:
        if (op.rep_e != kDefaultRep)
          return op_prolong_correct(op.a, op.b, p, op.out, s, op.rep_e, op.rep_gs, op.s1, op.s2);
        return op_prolong_correct(op.a, op.b, p, op.out, s);
      case OK_COPY:
        if (cudaMemcpyAsync(op.out->data, op.a->data, op.a->span * op.a->ebytes,
                            cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
            cudaMemcpyAsync(op.out->hdr, op.a->hdr, sizeof(Hdr), cudaMemcpyDeviceToDevice,
                            s) != cudaSuccess)
          return BFP_ERR_CUDA;
        return BFP_OK;
      case OK_FUSED:
        return fused_launch(op.dev, (int)op.sub.size(), op.arena, op.n_arena, op.arena_bytes,
                            op.zoff, op.zbuf, op.loff, ebytes, s);
    }
    return BFP_ERR_ARG;
  }
  int finalize(const PlanOp& op, const int64_t* part, int stage, cudaStream_t s) {
    return window_finalize(op.out, op.p, stage, part, s);
  }
};

// ---------------------------------------------------------------------------
// collectives between the ranks of a sharded solve
namespace {

struct Comm {
  virtual ~Comm() {}
  virtual int nlocal() const = 0;  // ranks driven by this process
  // fill the lower (HALO_LO: previous rank's last plane) / upper (HALO_HI: next rank's
  // first plane) halo planes of the slabs v[i] of the local ranks
  virtual int halo(bfp_vec_s* const* v, int which, cudaStream_t s) = 0;
  virtual int allreduce_max(int64_t* const* part, int n, cudaStream_t s) = 0;
  // all-reduce fused into the finalize kernel of a sharded op (peer-memory mailboxes, one
  // rank per process); false: the caller runs allreduce_max + the plain finalize
  virtual bool fused_finalize(bfp_vec_s* out, WinParams p, int stage, int64_t* part,
                              cudaStream_t s) {
    (void)out, (void)p, (void)stage, (void)part, (void)s;
    return false;
  }
  // int64 SUM of the exact-dot limb accumulators (4 words per local rank)
  virtual int allreduce_limbs(int64_t* const* acc, cudaStream_t s) = 0;
  // all-gather equal slabs into the full (replicated) vectors, header included
  virtual int gather(bfp_vec_s* const* slab, bfp_vec_s* const* full, cudaStream_t s) = 0;
};

__global__ void part_max_kernel(int64_t* const* parts, int P, int n) {
  const int i = threadIdx.x;
  if (i >= n) return;
  int64_t m = parts[0][i];
  for (int r = 1; r < P; ++r) m = parts[r][i] > m ? parts[r][i] : m;
  for (int r = 0; r < P; ++r) parts[r][i] = m;
}

static int64_t plane_bytes(const bfp_vec_s* v) { return (v->span / v->nz) * v->ebytes; }

// ---------------------------------------------------------------------------------------
// Peer-memory all-reduce of the per-op window partials {mu*, max, -min, err}: the cross-GPU
// form of the paper's atomic-max ParFor, over NVLink peer stores instead
// of a collective library call.  Every rank owns a MAILBOX in its own device memory that
// all its peers have mapped (CUDA IPC across processes, plain pointers inside one process):
//   post: rank r advances its op counter seq and writes {4 values, seq} into slot
//         [seq & 1][r] of EVERY rank's mailbox (P2P stores, values first, then the flag
//         after a system-scope fence);
//   wait: rank r polls the world slots of parity seq & 1 in its OWN mailbox (local memory:
//         no NVLink round trip) until their flags equal seq, takes the MAX and writes it
//         back to its partial buffer.
// MAX is exact and associative, so every rank computes identical values (bit-identical
// headers for every rank count).  Two parities suffice: a rank posts seq + 2 only after its
// wait(seq + 1), which needed every peer's post(seq + 1), issued after that peer's
// wait(seq).  seq lives on the device, so replayed CUDA graphs keep advancing it.  One
// process per GPU runs post + wait as ONE kernel (the wait polls while the peers' stores
// arrive, for at most ~2 s: a peer that never posts becomes BFP_ERR_CUDA in the op's sticky
// error word instead of a hang); an in-process group of ranks on one device (tests) runs all posts, then all
// waits, so no kernel ever waits on a later one of the same stream.
constexpr int kMaxWorld = 64;
struct Mailbox {
  int64_t slot[2][kMaxWorld][8];  // [parity][sender] = {v0, v1, v2, v3, seq, -, -, -}
  unsigned long long seq;
};
enum { MB_POST = 1, MB_WAIT = 2 };
// one block of 32 threads (thread q talks to peer q); returns with part[] = MAX over ranks
__device__ __forceinline__ void mailbox_exchange(Mailbox* const* peers, int rank, int world,
                                                 int64_t* part, int n, int phases) {
  const int q = threadIdx.x;
  Mailbox* mine = peers[rank];
  __shared__ unsigned long long s_seq;
  if (q == 0) {
    unsigned long long v = mine->seq;
    if (phases & MB_POST) mine->seq = ++v;
    s_seq = v;
  }
  __syncthreads();
  const unsigned long long seq = s_seq;
  const int par = (int)(seq & 1);
  if ((phases & MB_POST) && q < world) {
    int64_t* dst = peers[q]->slot[par][rank];
    for (int k = 0; k < n; ++k) dst[k] = part[k];
    __threadfence_system();
    *reinterpret_cast<volatile unsigned long long*>(dst + 4) = seq;
  }
  if (phases & MB_WAIT) {
    int64_t v[4] = {INT64_MIN, INT64_MIN, INT64_MIN, INT64_MIN};
    if (q < world) {
      const int64_t* src = mine->slot[par][q];
      // bounded wait (~2 s of SM clocks): a peer that never posts -- a mapping or launch
      // failure on another rank -- must surface as an error of this op, not hang the GPU
      const long long t0 = clock64();
      bool late = false;
      while (*reinterpret_cast<const volatile unsigned long long*>(src + 4) != seq) {
        __nanosleep(32);
        if (clock64() - t0 > (1ll << 32)) {
          late = true;
          break;
        }
      }
      __threadfence_system();
      for (int k = 0; k < n; ++k) v[k] = *reinterpret_cast<const volatile int64_t*>(src + k);
      if (late && n > 3) v[3] = 4;  // BFP_ERR_CUDA in the partial's error word (MAX keeps it)
    }
    for (int k = 0; k < n; ++k) {
      const int64_t m = bfpdev::shfl_max64(v[k]);
      if (q == 0) part[k] = m;
    }
  }
  __syncthreads();
}
__global__ void mailbox_kernel(Mailbox* const* peers, int rank, int world, int64_t* part, int n,
                               int phases) {
  mailbox_exchange(peers, rank, world, part, n, phases);
}
// The exchange fused into the finalize of a sharded op (one process per GPU): a rank whose
// header says the recompute stage has nothing to do returns before the exchange -- every
// rank holds the same header, so they all skip it together and the op counters stay aligned.
__global__ void finalize_mailbox_kernel(Vec out, WinParams p, int64_t* part, int storage_bits,
                                        Mailbox* const* peers, int rank, int world) {
  griddep_wait();
  if (p.mode == MODE_RECOMPUTE && !((const volatile Hdr*)out.hdr)->need_recompute) return;
  mailbox_exchange(peers, rank, world, part, 4, MB_POST | MB_WAIT);
  if (threadIdx.x == 0) finalize_from_partials(out, p, part, storage_bits);
}

// all ranks in this process on one device (bit-exact stand-in for the NCCL transport)
struct LocalComm : Comm {
  int P;
  int64_t** d_ptrs = nullptr;  // device array of the ranks' partial buffers
  // mailbox transport (bfp_set_transport(1)): the peer-memory protocol with in-process peers
  Mailbox* boxes = nullptr;
  Mailbox** d_boxes = nullptr;
  std::vector<int64_t*> h_parts;
  explicit LocalComm(int p) : P(p) {}
  ~LocalComm() override {
    cudaFree(d_ptrs);
    cudaFree(boxes);
    cudaFree(d_boxes);
  }
  int init_mailboxes() {
    if (P > 32) return BFP_ERR_ARG;
    if (cudaMalloc(&boxes, sizeof(Mailbox) * P) != cudaSuccess ||
        cudaMalloc(&d_boxes, sizeof(Mailbox*) * P) != cudaSuccess)
      return BFP_ERR_NOMEM;
    cudaMemset(boxes, 0, sizeof(Mailbox) * P);
    std::vector<Mailbox*> hp(P);
    for (int r = 0; r < P; ++r) hp[r] = boxes + r;
    return cudaMemcpy(d_boxes, hp.data(), sizeof(Mailbox*) * P, cudaMemcpyHostToDevice) ==
                   cudaSuccess
               ? BFP_OK
               : BFP_ERR_CUDA;
  }
  int nlocal() const override { return P; }
  int halo(bfp_vec_s* const* v, int which, cudaStream_t s) override {
    for (int r = 0; r < P; ++r) {
      const int64_t pb = plane_bytes(v[r]);
      char* d = (char*)v[r]->data;
      if ((which & HALO_LO) && r > 0 &&
          cudaMemcpyAsync(d - pb, (char*)v[r - 1]->data + (v[r - 1]->nz - 1) * pb, pb,
                          cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return BFP_ERR_CUDA;
      if ((which & HALO_HI) && r + 1 < P &&
          cudaMemcpyAsync(d + v[r]->nz * pb, v[r + 1]->data, pb, cudaMemcpyDeviceToDevice, s) !=
              cudaSuccess)
        return BFP_ERR_CUDA;
    }
    return BFP_OK;
  }
  // the ranks' partial buffers (set once at creation)
  int init(int64_t* const* part, bool mailbox) {
    h_parts.assign(part, part + P);
    if (cudaMalloc(&d_ptrs, sizeof(int64_t*) * P) != cudaSuccess) return BFP_ERR_NOMEM;
    if (cudaMemcpy(d_ptrs, part, sizeof(int64_t*) * P, cudaMemcpyHostToDevice) != cudaSuccess)
      return BFP_ERR_CUDA;
    return mailbox ? init_mailboxes() : BFP_OK;
  }
  int allreduce_max(int64_t* const* part, int n, cudaStream_t s) override {
    if (boxes) {  // every rank posts, then every rank waits (one stream: no kernel spins on a later one)
      for (int r = 0; r < P; ++r) mailbox_kernel<<<1, 32, 0, s>>>(d_boxes, r, P, part[r], n, MB_POST);
      for (int r = 0; r < P; ++r) mailbox_kernel<<<1, 32, 0, s>>>(d_boxes, r, P, part[r], n, MB_WAIT);
      count_launch(2 * P);
      return cudaGetLastError() == cudaSuccess ? BFP_OK : BFP_ERR_CUDA;
    }
    part_max_kernel<<<1, 32, 0, s>>>(d_ptrs, P, n);
    count_launch();
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fprintf(stderr, "bfpmg_b200: part_max launch: %s\n", cudaGetErrorString(e));
    return e == cudaSuccess ? BFP_OK : BFP_ERR_CUDA;
  }
  int allreduce_limbs(int64_t* const* acc, cudaStream_t s) override {
    return limb_sum_local(acc, P, s);
  }
  int gather(bfp_vec_s* const* slab, bfp_vec_s* const* full, cudaStream_t s) override {
    for (int r = 0; r < P; ++r) {
      for (int q = 0; q < P; ++q) {
        const int64_t pb = plane_bytes(slab[q]);
        if (cudaMemcpyAsync((char*)full[r]->data + slab[q]->z0 * pb, slab[q]->data,
                            slab[q]->nz * pb, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
          return BFP_ERR_CUDA;
      }
      if (cudaMemcpyAsync(full[r]->hdr, slab[r]->hdr, sizeof(Hdr), cudaMemcpyDeviceToDevice, s) !=
          cudaSuccess)
        return BFP_ERR_CUDA;
    }
    return BFP_OK;
  }
};

// NCCL, one rank per process; the library is the one already loaded by the host
// framework (torch) when present, resolved at run time
struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  bool load() {
    if (h) return true;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) return false;
    bool ok = true;
    auto sym = [&](auto& fn, const char* s) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, s));
      ok = ok && fn != nullptr;
    };
    sym(GetUniqueId, "ncclGetUniqueId");
    sym(CommInitRank, "ncclCommInitRank");
    sym(CommDestroy, "ncclCommDestroy");
    sym(AllReduce, "ncclAllReduce");
    sym(AllGather, "ncclAllGather");
    sym(Send, "ncclSend");
    sym(Recv, "ncclRecv");
    sym(GroupStart, "ncclGroupStart");
    sym(GroupEnd, "ncclGroupEnd");
    return ok;
  }
};
Nccl& nccl() {
  static Nccl n;
  return n;
}

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  // peer-memory mailboxes (mapped with CUDA IPC); nullptr: NCCL all-reduce
  Mailbox* box = nullptr;
  Mailbox** d_boxes = nullptr;
  std::vector<Mailbox*> opened;
  ~NcclComm() override {
    for (Mailbox* m : opened) cudaIpcCloseMemHandle(m);
    cudaFree(box);
    cudaFree(d_boxes);
    if (comm) nccl().CommDestroy(comm);
  }
  // Allocate this rank's mailbox, exchange the IPC handles (all-gather of the 64-byte
  // handles through NCCL) and map every peer's.  Any failure (no peer access between two
  // GPUs, IPC disabled in the container) leaves the NCCL all-reduce in place.
  int init_mailboxes() {
    if (world > 32) return BFP_ERR_ARG;
    if (cudaMalloc(&box, sizeof(Mailbox)) != cudaSuccess) return BFP_ERR_NOMEM;
    cudaMemset(box, 0, sizeof(Mailbox));
    std::vector<Mailbox*> hp(world, nullptr);
    hp[rank] = box;
    bool ok = true;
    if (world > 1) {
      cudaIpcMemHandle_t mine;
      ok = cudaIpcGetMemHandle(&mine, box) == cudaSuccess;
      char* d_h = nullptr;
      ok = ok && cudaMalloc(&d_h, sizeof(mine) * world) == cudaSuccess;
      if (ok) {
        cudaMemcpy(d_h + sizeof(mine) * rank, &mine, sizeof(mine), cudaMemcpyHostToDevice);
        ok = nccl().AllGather(d_h + sizeof(mine) * rank, d_h, sizeof(mine), ncclUint8, comm,
                              nullptr) == ncclSuccess &&
             cudaStreamSynchronize(nullptr) == cudaSuccess;
      }
      std::vector<cudaIpcMemHandle_t> all(world);
      if (ok) cudaMemcpy(all.data(), d_h, sizeof(mine) * world, cudaMemcpyDeviceToHost);
      cudaFree(d_h);
      for (int q = 0; q < world && ok; ++q) {
        if (q == rank) continue;
        void* ptr = nullptr;
        ok = cudaIpcOpenMemHandle(&ptr, all[q], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
        if (ok) {
          hp[q] = static_cast<Mailbox*>(ptr);
          opened.push_back(hp[q]);
        }
      }
    }
    ok = ok && cudaMalloc(&d_boxes, sizeof(Mailbox*) * world) == cudaSuccess &&
         cudaMemcpy(d_boxes, hp.data(), sizeof(Mailbox*) * world, cudaMemcpyHostToDevice) ==
             cudaSuccess;
    // every rank must end up on the same transport: MIN over the ranks' outcome
    int64_t* d_ok = nullptr;
    int64_t h_ok = ok ? 1 : 0;
    if (cudaMalloc(&d_ok, sizeof(int64_t)) == cudaSuccess) {
      cudaMemcpy(d_ok, &h_ok, sizeof(h_ok), cudaMemcpyHostToDevice);
      if (nccl().AllReduce(d_ok, d_ok, 1, ncclInt64, ncclMin, comm, nullptr) != ncclSuccess ||
          cudaStreamSynchronize(nullptr) != cudaSuccess)
        h_ok = 0;
      else
        cudaMemcpy(&h_ok, d_ok, sizeof(h_ok), cudaMemcpyDeviceToHost);
      cudaFree(d_ok);
    } else {
      h_ok = 0;
    }
    cudaGetLastError();
    if (!h_ok) {
      for (Mailbox* m : opened) cudaIpcCloseMemHandle(m);
      opened.clear();
      cudaFree(box);
      cudaFree(d_boxes);
      box = nullptr;
      d_boxes = nullptr;
    }
    return BFP_OK;
  }
  int nlocal() const override { return 1; }
  int halo(bfp_vec_s* const* v, int which, cudaStream_t s) override {
    Nccl& n = nccl();
    const int64_t pb = plane_bytes(v[0]);
    char* d = (char*)v[0]->data;
    const int nz = v[0]->nz;
    bool ok = n.GroupStart() == ncclSuccess;
    if (which & HALO_LO) {  // last plane -> next rank's lower halo
      if (rank > 0) ok = ok && n.Recv(d - pb, pb, ncclUint8, rank - 1, comm, s) == ncclSuccess;
      if (rank + 1 < world)
        ok = ok && n.Send(d + (nz - 1) * pb, pb, ncclUint8, rank + 1, comm, s) == ncclSuccess;
    }
    if (which & HALO_HI) {  // first plane -> previous rank's upper halo
      if (rank + 1 < world)
        ok = ok && n.Recv(d + nz * pb, pb, ncclUint8, rank + 1, comm, s) == ncclSuccess;
      if (rank > 0) ok = ok && n.Send(d, pb, ncclUint8, rank - 1, comm, s) == ncclSuccess;
    }
    ok = (n.GroupEnd() == ncclSuccess) && ok;
    return ok ? BFP_OK : BFP_ERR_CUDA;
  }
  bool fused_finalize(bfp_vec_s* out, WinParams p, int stage, int64_t* part,
                      cudaStream_t s) override {
    if (!box) return false;
    if (stage == 1) p.mode = MODE_RECOMPUTE;
    p.part = nullptr;
    finalize_mailbox_kernel<<<1, 32, 0, s>>>(view(out), p, part, out->ebytes * 8,
                                             (Mailbox* const*)d_boxes, rank, world);
    count_launch();
    return true;
  }
  int allreduce_max(int64_t* const* part, int cnt, cudaStream_t s) override {
    if (box) {  // post + wait in one kernel: the peers' kernels run on their own GPUs
      mailbox_kernel<<<1, 32, 0, s>>>(d_boxes, rank, world, part[0], cnt, MB_POST | MB_WAIT);
      count_launch();
      return cudaGetLastError() == cudaSuccess ? BFP_OK : BFP_ERR_CUDA;
    }
    return nccl().AllReduce(part[0], part[0], cnt, ncclInt64, ncclMax, comm, s) == ncclSuccess
               ? BFP_OK
               : BFP_ERR_CUDA;
  }
  int allreduce_limbs(int64_t* const* acc, cudaStream_t s) override {
    return nccl().AllReduce(acc[0], acc[0], 4, ncclInt64, ncclSum, comm, s) == ncclSuccess
               ? BFP_OK
               : BFP_ERR_CUDA;
  }
  int gather(bfp_vec_s* const* slab, bfp_vec_s* const* full, cudaStream_t s) override {
    const int64_t bytes = slab[0]->nz * plane_bytes(slab[0]);
    if (nccl().AllGather(slab[0]->data, full[0]->data, bytes, ncclUint8, comm, s) != ncclSuccess)
      return BFP_ERR_CUDA;
    return cudaMemcpyAsync(full[0]->hdr, slab[0]->hdr, sizeof(Hdr), cudaMemcpyDeviceToDevice,
                           s) == cudaSuccess
               ? BFP_OK
               : BFP_ERR_CUDA;
  }
};

}  // namespace

// the solver handle: the local ranks' plans (one, or all ranks of an in-process group)
struct bfp_mg_s {
  std::vector<RankSolver*> rs;
  Comm* comm = nullptr;
  std::vector<int64_t*> parts;  // per local rank: {mu*, max, -min, err}
  cudaGraphExec_t graph = nullptr;
  int64_t launches_per_solve = 0;
  ~bfp_mg_s() {
    if (graph) cudaGraphExecDestroy(graph);
    for (auto* r : rs) delete r;
    for (auto* p : parts) cudaFree(p);
    delete comm;
  }
  RankSolver* r0() const { return rs[0]; }

  int execute(cudaStream_t s) {
    const int64_t before = launches();
    const size_t nops = r0()->plan.size();
    const int P = (int)rs.size();
    std::vector<bfp_vec_s*> va(P), vo(P);
    for (size_t i = 0; i < nops; ++i) {
      const PlanOp& op0 = r0()->plan[i];
      for (int r = 0; r < P; ++r) {
        va[r] = rs[r]->plan[i].a;
        vo[r] = rs[r]->plan[i].out;
      }
      int rc = BFP_OK;
      if (op0.kind == OK_GATHER) {
        rc = comm->gather(va.data(), vo.data(), s);
      } else if (!op0.shard) {
        for (int r = 0; r < P && !rc; ++r) rc = rs[r]->run(rs[r]->plan[i], s);
      } else {
        if (op0.halo) rc = comm->halo(va.data(), op0.halo, s);
        const int stages = op0.p.mode == MODE_QCOMP ? 2 : 1;
        for (int st = 0; st < stages && !rc; ++st) {
          for (int r = 0; r < P && !rc; ++r) rc = rs[r]->run(rs[r]->plan[i], s, parts[r], st);
          if (!rc && P == 1 &&
              comm->fused_finalize(rs[0]->plan[i].out, rs[0]->plan[i].p, st, parts[0], s))
            continue;  // exchange + finalize in one kernel
          if (!rc) rc = comm->allreduce_max(parts.data(), 4, s);
          for (int r = 0; r < P && !rc; ++r) rc = rs[r]->finalize(rs[r]->plan[i], parts[r], st, s);
        }
      }
      if (rc) return rc;
    }
    launches_per_solve = launches() - before;
    return BFP_OK;
  }
};

extern "C" {

static int check_cfg(const bfp_mg_config_t* cfg) {
  if (cfg->ref_mode) {  // reference-algorithm mode: 1-D / 2-D, levels 1 .. l_fine
    if ((cfg->d != 1 && cfg->d != 2) || cfg->l_fine < 1 || cfg->l_fine > 30 || cfg->cycles < 0) return BFP_ERR_ARG;
    for (int l = 1; l <= cfg->l_fine; ++l)
      if (cfg->p[l] < 3 || cfg->p[l] > 58 || cfg->pd[l] < 0 || cfg->pd[l] > 58 ||
          cfg->pc[l] < 0 || cfg->pc[l] > 58 || cfg->ref_c1d[l].q < 1 || cfg->ref_c2d[l].q < 1)
        return BFP_ERR_ARG;
    // PrecisionSchedule::validate (P/src/multigrid.cpp:37-44, enforced by the reference's
    // Hierarchy at :259): wcheck >= w >= wdot >= 1 on every level (0 entries mean w)
    for (int l = 1; l <= cfg->l_fine; ++l) {
      const int w = cfg->p[l], wd = cfg->pd[l] ? cfg->pd[l] : w, wc = cfg->pc[l] ? cfg->pc[l] : w;
      if (!(wc >= w && w >= wd && wd >= 1)) return BFP_ERR_ARG;
    }
    return BFP_OK;
  }
  // (config mode keeps wdot > w legal: the frozen config 1 runs its residual and V-cycle at
  // 28 bits over a 16-bit iterate, DESIGN.md section 3.4 -- a relaxation of the reference's
  // ordering invariant that the reference-algorithm mode does not share)
  if (cfg->d < 1 || cfg->d > 3 || cfg->l_coarse < 2 || cfg->l_fine < cfg->l_coarse ||
      cfg->l_fine > 30 || cfg->nu1 < 1 || cfg->nu2 < 0 || cfg->n_coarse < 1 || cfg->cycles < 0 ||
      cfg->qc < 2 || cfg->qc > 30)
    return BFP_ERR_ARG;
  for (int l = cfg->l_coarse; l <= cfg->l_fine; ++l) {
    if (cfg->p[l] < 2 || cfg->p[l] > 58) return BFP_ERR_ARG;
    if (cfg->pd[l] < 0 || cfg->pd[l] > 58 || cfg->pc[l] < 0 || cfg->pc[l] > 58) return BFP_ERR_ARG;
  }
  return BFP_OK;
}

static int make_group(const bfp_mg_config_t* cfg, int world, int rank0, int nlocal,
                      int min_planes, Comm* comm, bfp_mg_t* out) {
  bfp_mg_s* mg = new bfp_mg_s();
  mg->comm = comm;
  int rc = BFP_OK;
  for (int i = 0; i < nlocal && !rc; ++i) {
    RankSolver* r = new RankSolver();
    r->cfg = *cfg;
    r->rank = rank0 + i;
    r->world = world;
    r->min_planes = min_planes;
#ifdef BFP_AB_ENV
    if (const char* ev = getenv("BFP_NO_FUSION")) r->fusion = ev[0] != '1';
#endif
    mg->rs.push_back(r);
    rc = r->build();
    int64_t* part = nullptr;
    if (!rc && cudaMalloc(&part, 4 * sizeof(int64_t)) != cudaSuccess) rc = BFP_ERR_NOMEM;
    if (part) mg->parts.push_back(part);
  }
  // every rank must have built the same plan
  for (size_t i = 1; i < mg->rs.size() && !rc; ++i)
    if (mg->rs[i]->plan.size() != mg->rs[0]->plan.size()) rc = BFP_ERR_ARG;
  if (rc) {
    delete mg;
    return rc;
  }
  *out = mg;
  return BFP_OK;
}

int bfp_mg_create(const bfp_mg_config_t* cfg, bfp_mg_t* out) {
  if (!cfg || !out) return BFP_ERR_ARG;
  int rc = check_cfg(cfg);
  if (rc) return rc;
  return make_group(cfg, 1, 0, 1, 16, nullptr, out);
}

int bfp_nccl_unique_id(void* id, int id_bytes) {
  if (!id || id_bytes < (int)sizeof(ncclUniqueId)) return BFP_ERR_ARG;
  if (!nccl().load()) return BFP_ERR_CUDA;
  ncclUniqueId u;
  if (nccl().GetUniqueId(&u) != ncclSuccess) return BFP_ERR_CUDA;
  memcpy(id, &u, sizeof(u));
  return BFP_OK;
}

int bfp_mg_create_sharded(const bfp_mg_config_t* cfg, int world, int rank, const void* nccl_id,
                          int min_planes, bfp_mg_t* out) {
  if (!cfg || !out || world < 1 || min_planes < 2) return BFP_ERR_ARG;
  int rc = check_cfg(cfg);
  if (rc) return rc;
  if (world & (world - 1)) return BFP_ERR_ARG;  // slabs: world | 2^l
  if (!nccl_id) {
    LocalComm* c = new LocalComm(world);
    rc = make_group(cfg, world, 0, world, min_planes, c, out);  // owns c
    if (rc) return rc;
    rc = c->init((*out)->parts.data(), g_transport == 1);
    if (rc) {
      delete *out;
      *out = nullptr;
    }
    return rc;
  }
  if (rank < 0 || rank >= world) return BFP_ERR_ARG;
  if (!nccl().load()) return BFP_ERR_CUDA;
  NcclComm* c = new NcclComm();
  c->rank = rank;
  c->world = world;
  ncclUniqueId u;
  memcpy(&u, nccl_id, sizeof(u));
  if (nccl().CommInitRank(&c->comm, world, u, rank) != ncclSuccess) {
    c->comm = nullptr;
    delete c;
    return BFP_ERR_CUDA;
  }
  if (g_transport != 2) c->init_mailboxes();  // falls back to the NCCL all-reduce on failure
  return make_group(cfg, world, rank, 1, min_planes, c, out);
}

int bfp_set_transport(int t) {
  if (t < 0 || t > 2) return BFP_ERR_ARG;
  g_transport = t;
  return BFP_OK;
}

int bfp_mg_transport(bfp_mg_t mg) {
  if (!mg || !mg->comm) return 0;
  if (auto* l = dynamic_cast<LocalComm*>(mg->comm)) return l->boxes ? 1 : 0;
  if (auto* n = dynamic_cast<NcclComm*>(mg->comm)) return n->box ? 1 : 2;
  return 0;
}

int bfp_mg_destroy(bfp_mg_t mg) {
  delete mg;
  return BFP_OK;
}

int bfp_mg_solve(bfp_mg_t mg, int use_graph, void* stream) {
  if (!mg) return BFP_ERR_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!use_graph) return mg->execute(s);
  if (!mg->graph) {
    // capture on a private non-default stream, then replay on the caller's
    cudaStream_t cs;
    if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) return BFP_ERR_CUDA;
    cudaGraph_t g;
    if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      cudaStreamDestroy(cs);
      return BFP_ERR_CUDA;
    }
    const int64_t before = launches();
    int rc = mg->execute(cs);
    const int64_t n = launches() - before;
    cudaError_t e = cudaStreamEndCapture(cs, &g);
    cudaStreamDestroy(cs);
    if (rc) return rc;
    if (e != cudaSuccess) return BFP_ERR_CUDA;
    e = cudaGraphInstantiate(&mg->graph, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return BFP_ERR_CUDA;
    count_launch(-(int)n);  // captured, not launched
  }
  count_launch((int)mg->launches_per_solve);
  return cudaGraphLaunch(mg->graph, s) == cudaSuccess ? BFP_OK : BFP_ERR_CUDA;
}

// results of local rank 0: its finest-level iterate (a slab when sharded), history, trace
int bfp_mg_result(bfp_mg_t mg, int64_t* x, bfp_header_t* xh, double* hist, int hist_cap,
                  int* n_hist, bfp_trace_rec_t* trace, int64_t trace_cap, int64_t* n_trace,
                  void* stream) {
  if (!mg) return BFP_ERR_ARG;
  RankSolver* r = mg->r0();
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int rc = bfp_vec_download(r->x_final, x, xh, stream);
  if (rc) return rc;
  if (hist && hist_cap > 0)
    cudaMemcpyAsync(hist, r->d_hist, sizeof(double) * std::min(hist_cap, r->n_hist),
                    cudaMemcpyDeviceToHost, s);
  if (trace && trace_cap > 0)
    cudaMemcpyAsync(trace, r->d_trace,
                    sizeof(TraceRec) * (size_t)std::min<int64_t>(trace_cap, r->n_trace),
                    cudaMemcpyDeviceToHost, s);
  if (n_hist) *n_hist = r->n_hist;
  if (n_trace) *n_trace = r->n_trace;
  if (cudaStreamSynchronize(s) != cudaSuccess) return BFP_ERR_CUDA;
  // sticky device errors of any solver vector of any local rank
  for (auto* rr : mg->rs)
    for (auto* v : rr->owned) {
      Hdr h;
      cudaMemcpy(&h, v->hdr, sizeof(h), cudaMemcpyDeviceToHost);
      if (h.err) return h.err;
    }
  return BFP_OK;
}

int bfp_mg_vectors(bfp_mg_t mg, bfp_vec_t* x, bfp_vec_t* b, bfp_vec_t* r) {
  if (!mg) return BFP_ERR_ARG;
  RankSolver* s = mg->r0();
  const int lf = s->cfg.l_fine;
  if (x) *x = s->lev[lf].x[0];
  if (b) *b = s->lev[lf].b;
  if (r) *r = s->lev[lf].r[0];
  return BFP_OK;
}

int bfp_mg_level_rhs(bfp_mg_t mg, int level, bfp_vec_t* b, int* mant_bytes) {
  if (!mg || !b || mg->rs.size() != 1) return BFP_ERR_ARG;
  RankSolver* s = mg->r0();
  if (s->world > 1 || level < 1 || level > s->cfg.l_fine || level >= (int)s->lev.size() ||
      !s->lev[level].b)
    return BFP_ERR_ARG;
  *b = s->lev[level].b;
  if (mant_bytes) *mant_bytes = s->ebytes;
  return BFP_OK;
}

int bfp_mg_rank_result(bfp_mg_t mg, int local_rank, bfp_vec_t* x_final, bfp_vec_t* r_final,
                       int* rank, int* lowest_sharded_level) {
  if (!mg || local_rank < 0 || local_rank >= (int)mg->rs.size()) return BFP_ERR_ARG;
  RankSolver* s = mg->rs[local_rank];
  if (x_final) *x_final = s->x_final;
  if (r_final) *r_final = s->r_final;
  if (rank) *rank = s->rank;
  if (lowest_sharded_level) *lowest_sharded_level = s->ls;
  return BFP_OK;
}

int64_t bfp_mg_kernel_launches(bfp_mg_t mg) { return mg ? mg->launches_per_solve : -1; }

// ---- sharded single ops over a communicator (the residual / Jacobi of a fine level) ----
struct bfp_dist_s {
  Comm* comm = nullptr;
  std::vector<int64_t*> parts;
  ~bfp_dist_s() {
    for (auto* p : parts) cudaFree(p);
    delete comm;
  }
};

int bfp_dist_create(int world, int rank, const void* nccl_id, bfp_dist_t* out) {
  if (!out || world < 1) return BFP_ERR_ARG;
  bfp_dist_s* d = new bfp_dist_s();
  int rc = BFP_OK;
  if (!nccl_id) {
    LocalComm* c = new LocalComm(world);
    d->comm = c;
    d->parts.assign(world, nullptr);
    for (auto& p : d->parts)
      if (cudaMalloc(&p, 4 * sizeof(int64_t)) != cudaSuccess) rc = BFP_ERR_NOMEM;
    if (!rc) rc = c->init(d->parts.data(), g_transport == 1);
  } else {
    if (rank < 0 || rank >= world || !nccl().load()) {
      delete d;
      return rank < 0 || rank >= world ? BFP_ERR_ARG : BFP_ERR_CUDA;
    }
    NcclComm* c = new NcclComm();
    c->rank = rank;
    c->world = world;
    ncclUniqueId u;
    memcpy(&u, nccl_id, sizeof(u));
    if (nccl().CommInitRank(&c->comm, world, u, rank) != ncclSuccess) {
      c->comm = nullptr;
      rc = BFP_ERR_CUDA;
    }
    d->comm = c;
    if (!rc && g_transport != 2) c->init_mailboxes();  // NCCL all-reduce when they cannot be mapped
    d->parts.assign(1, nullptr);
    if (!rc && cudaMalloc(&d->parts[0], 4 * sizeof(int64_t)) != cudaSuccess) rc = BFP_ERR_NOMEM;
  }
  if (rc) {
    delete d;
    return rc;
  }
  *out = d;
  return BFP_OK;
}

int bfp_dist_destroy(bfp_dist_t d) {
  delete d;
  return BFP_OK;
}

}  // extern "C"
// halo exchange -> pass 1 (partials) -> all-reduce -> finalize [-> recompute -> ...]
template <typename F>
static int dist_window(bfp_dist_t d, bfp_vec_t const* x, bfp_vec_t const* out, int mode,
                       int64_t w_out, int64_t w_tmp, bfp_scalar_t g, cudaStream_t s, F launch) {
  const int P = d->comm->nlocal();
  for (int r = 0; r < P; ++r)
    if (!x[r] || !out[r] || out[r]->dim < 2) return BFP_ERR_ARG;
  int rc = d->comm->halo(x, HALO_LO | HALO_HI, s);
  WinParams p = win_params(mode == 1 ? MODE_NNQ : MODE_QCOMP, w_out, w_tmp, 0);
  p.gamma = gamma_literal(g.m, g.e);
  const int stages = mode == 1 ? 1 : 2;
  for (int st = 0; st < stages && !rc; ++st) {
    for (int r = 0; r < P && !rc; ++r) {
      WinParams pr = p;
      pr.part = d->parts[r];
      if (st == 1) pr.mode = MODE_RECOMPUTE;
      rc = launch(r, pr);
    }
    if (!rc) rc = d->comm->allreduce_max(d->parts.data(), 4, s);
    for (int r = 0; r < P && !rc; ++r) rc = window_finalize(out[r], p, st, d->parts[r], s);
  }
  return rc;
}
extern "C" {

int bfp_dist_stencil_gemv(bfp_dist_t d, bfp_vec_t const* x, bfp_vec_t const* y,
                          bfp_scalar_t alpha, bfp_scalar_t beta, int mode, int64_t w_out,
                          int64_t w_tmp, bfp_scalar_t gamma, bfp_vec_t const* out, void* stream) {
  if (!d || !x || !y || !out || gamma.m <= 0) return BFP_ERR_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  return dist_window(d, x, out, mode, w_out, w_tmp, gamma, s, [&](int r, const WinParams& p) {
    return op_gemv(x[r], y[r], Scal{alpha.m, alpha.q, alpha.e}, Scal{beta.m, beta.q, beta.e}, p,
                   out[r], s);
  });
}

int bfp_dist_dot_exact(bfp_dist_t d, bfp_vec_t const* x, bfp_vec_t const* y,
                       int64_t* const* d_acc, void* stream) {
  if (!d || !x || !y || !d_acc) return BFP_ERR_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int P = d->comm->nlocal();
  int rc = BFP_OK;
  for (int r = 0; r < P && !rc; ++r) rc = dot_limbs(x[r], y[r], d_acc[r], s, true);
  if (!rc) rc = d->comm->allreduce_limbs(d_acc, s);
  return rc;
}

int bfp_dist_stencil_jacobi(bfp_dist_t d, bfp_vec_t const* x, bfp_vec_t const* b, bfp_scalar_t c,
                            int mode, int64_t w_out, int64_t w_tmp, bfp_scalar_t gamma,
                            bfp_vec_t const* out, void* stream) {
  if (!d || !x || !b || !out || gamma.m <= 0) return BFP_ERR_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  return dist_window(d, x, out, mode, w_out, w_tmp, gamma, s, [&](int r, const WinParams& p) {
    return op_jacobi(x[r], b[r], Scal{c.m, c.q, c.e}, p, out[r], s);
  });
}

}  // extern "C"
