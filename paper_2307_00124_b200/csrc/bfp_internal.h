// bfp_internal.h -- host-side structures and op launchers shared by the C-ABI
// (bfp_lib.cu) and the native multigrid driver (bfp_solver.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../../include/bfpmg_b200.h"
#include "bfp_dev.cuh"
#include "bfp_ops.cuh"

struct bfp_vec_s {
  int dim = 0, l = 0, ebytes = 4;
  int z0 = 0, nz = 0;  // slab: global index of local plane 0 / local planes (slowest axis)
  int64_t nlog = 0, span = 0, halo = 0;
  char* base = nullptr;  // device allocation (halo + span + halo)
  void* data = nullptr;  // element 0
  bfpdev::Hdr* hdr = nullptr;
  void* stage = nullptr;  // device staging in logical order (uploads / downloads)
  size_t stage_bytes = 0;
  double* tab = nullptr;  // sine table (generator)
  int64_t* dot_acc = nullptr;  // exact-dot accumulator of the synchronous bfp_dot_exact*
  int64_t tab_n = 0;
};

struct bfp_csr_s {
  bfpdev::CsrDev d;
  int64_t* buf = nullptr;
};

namespace bfpdev {
// fused coarse-level op list entry (bfp_coarse.cuh: coarse_kernel)
enum { FK_GEMV = 0, FK_JACOBI, FK_SCAL, FK_AXPBY, FK_RESTRICT, FK_PROLONG, FK_PCORR, FK_ZERO };
constexpr int kFusedThreads = 512;
constexpr int kArenaMaxBytes = 200 * 1024;  // dynamic shared memory of the fused kernel
constexpr int kLeanMaxVec = 128;  // block headers of one fused list (lean engine)
// one vector of an arena-resident fused op list: data (halos included) and header
struct ArenaEntry {
  char* gbase;
  Hdr* ghdr;
  int64_t bytes;      // data bytes staged in shared memory (0: the data stays global)
  int32_t off, hoff;  // byte offsets in the CTA's shared memory
  int32_t wb, pad;    // written by the op list: copied back when the launch ends
};
// The lean engine's digest of an op record (host-filled, bfp_solver.cu): everything its
// control lane and workers need that is static, in one 64-byte block.
struct LeanRec {
  uint8_t ok;           // statically eligible for the fast path (lean_static_ok)
  uint8_t vout, va, vb; // arena vector ids of the output and the two operands (0xff: none)
  uint8_t gv[3];        // vector ids of the gamma terms (0xff: X = 1)
  uint8_t ng;           // gamma terms
  int16_t w_out, nnq;
  int32_t n4;           // 4-groups of the output
  int8_t dim, l;
  int8_t nnq_next;      // the next op of the list is nnqcomp
  int8_t pad1;
  int32_t ea;           // e_A (gemv), 2l (jacobi), e_R (restrict), e_P (prolong / pcorr)
  int32_t am, ae, bm, be;  // coefficients: gemv / axpby / pcorr alpha, beta; jacobi / scal c
  const int32_t* x;     // operand data (arena offsets until rebased)
  const int32_t* y;
  int32_t* out;
};
static_assert(sizeof(LeanRec) == 64, "LeanRec is four 16-byte chunks");
struct alignas(16) FusedOp {
  int32_t kind, pad;
  int64_t q;
  uint64_t rb[2];  // bit w: the record's 8-byte word w is an arena offset (rebased on fetch)
  LeanRec lr;
  Vec out;
  WinParams p;
  union U {
    GemvOp gemv;
    JacobiOp jac;
    ScalOp scal;
    AxpbyOp axpby;
    RestrictOp rst;
    ProlongOp pro;
    ProlongCorrectOp pc;
  } u;
};
}  // namespace bfpdev

namespace bfp {

using bfpdev::ArenaEntry;
using bfpdev::FusedOp;
using bfpdev::GammaRule;
using bfpdev::Scal;
using bfpdev::WinParams;

bfpdev::Vec view(const bfp_vec_s* v);
int vec_alloc(int dim, int level, int64_t n, int ebytes, bfp_vec_s** out);
int vec_alloc_slab(int dim, int level, int64_t n, int z_lo, int z_hi, int ebytes, bfp_vec_s** out);
void vec_free(bfp_vec_s* v);
int set_zero(bfp_vec_s* v, int64_t q, cudaStream_t s);

WinParams win_params(int mode, int64_t w_out, int64_t w_tmp, int force);
int window_finalize(bfp_vec_s* out, WinParams p, int stage, const int64_t* part, cudaStream_t s);
GammaRule gamma_literal(int64_t m, int64_t e);  // (declared for the solver too)

// windowed ops (mode in p: MODE_QCOMP launches pass 1 + recompute, MODE_NNQ one pass)
// operator representation overrides (reference-algorithm mode): kDefaultRep keeps the
// config operators (stencil e_A = 2l, full weighting e_R = -2d, prolongation e_P = -d)
constexpr int kDefaultRep = -0x40000000;
int op_gemv(bfp_vec_s* x, bfp_vec_s* y, Scal al, Scal be, const WinParams& p, bfp_vec_s* out,
            cudaStream_t s, int ea = kDefaultRep, int gs = 0, int st9 = 0);
int op_jacobi(bfp_vec_s* x, bfp_vec_s* b, Scal c, const WinParams& p, bfp_vec_s* out,
              cudaStream_t s);
int op_scal(bfp_vec_s* r, Scal c, const WinParams& p, bfp_vec_s* out, cudaStream_t s);
int op_axpby(bfp_vec_s* x, bfp_vec_s* y, Scal al, Scal be, const WinParams& p, bfp_vec_s* out,
             cudaStream_t s);
int op_restrict(bfp_vec_s* r, const WinParams& p, bfp_vec_s* out, cudaStream_t s,
                int er = kDefaultRep, int gs = 0);
int op_prolong(bfp_vec_s* xc, const WinParams& p, bfp_vec_s* out, cudaStream_t s,
               int ep = kDefaultRep, int gs = 0);
int op_prolong_correct(bfp_vec_s* ec, bfp_vec_s* y, const WinParams& p, bfp_vec_s* out,
                       cudaStream_t s, int ep = kDefaultRep, int gs = 0,
                       Scal al = Scal{1, 2, 0}, Scal be = Scal{1, 2, 0});

int gen_uniform(bfp_vec_s* v, int64_t p, uint64_t seed, uint64_t stream_id, cudaStream_t s);
int gen_sine(bfp_vec_s* v, int64_t p, cudaStream_t s);

void jacobi_coeff(int dim, int level, int64_t qc, int64_t* cm, int64_t* ce);
int fused_make(int kind, bfp_vec_s* a, bfp_vec_s* b, Scal s1, Scal s2, const WinParams& p,
               int64_t q, bfp_vec_s* out, FusedOp* f);
int fused_launch(const FusedOp* d_ops, int n, const ArenaEntry* d_ar, int nar, int arena_bytes,
                 int zoff, int64_t* zglobal, int loff, int ebytes, cudaStream_t s);
void count_launch(int n = 1);
int64_t launches();
// launches per kernel family (evidence of which pipelines a solve used; bfp_kernel_family_counts)
enum KernelFamily { FAM_GRID = 0, FAM_BULK2, FAM_BULK3, FAM_MARCH, FAM_PRO3, FAM_RST3, FAM_PRO2,
                    FAM_RST2, FAM_FLAT, FAM_FUSED, FAM_COARSE, FAM_N = 16 };
void count_family(int fam);
// exact dot (op_dot.cu): limb accumulator d_acc[5] = {L0..L3, e}, value sum_k L_k 2^(48k);
// normalise: carry the limbs into [0, 2^48) (before a multi-rank SUM)
int dot_limbs(bfp_vec_s* x, bfp_vec_s* y, int64_t* d_acc, cudaStream_t s, bool normalise);
constexpr int kMaxLimbRanks = 64;  // in-process rank groups (LocalComm)
struct LimbPtrs {
  int64_t* p[kMaxLimbRanks];
};
int limb_sum_local(int64_t* const* d_ptrs, int P, cudaStream_t s);

}  // namespace bfp
