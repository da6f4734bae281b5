// Launchers of the device kernels (one declaration per hand-written kernel family).
#pragma once

#include "common.cuh"

namespace vsie {

// ------------------------------------------------------------------ entries (entries.cu)
struct EntryGeom {
  int n1, n2, n3;
  double ox, oy, oz;      // voxel (0,0,0) centre
  double hx, hy, hz;
  double dx, dy, dz;      // Gauss offsets h / (2 sqrt 3)
  double w;               // h1 h2 h3 / 8
  double pw[8];           // per-node factor 1/(4 pi) x PWL test function at node p (1 for PWC)
  double k0, inv_k0;
  int taylor;             // 1: one sincos per source node + order-7 Taylor phase per pair (entries.cu)
  int nodes;              // voxel nodes: 8 (2 x 2 x 2 Gauss) or 1 (centre, quad_rule 1)
  int nsrc;               // source records per RWG read: 6 (3-point rule x 2 triangles) or 2
  double scale_re, scale_im;
  const double* src;     // [m][36] device
  int64_t m;
  int64_t nv;
};

// out[i] = Z[idx[2i], idx[2i+1]] (explicit list).
void launch_entries_list(const EntryGeom& g, const int64_t* idx, int64_t count, cplx* out,
                         cudaStream_t st);

// Structured supercore block:
//   M[(a, i_k), (i_{k+1}, b)] = A_chi(I_{<=k-1}[a], i_k, i_{k+1}, J_{>k+1}[b]),
//   columns [col0, col1) of the (rl * nk) x (nk1 * rr) matrix, written column-major
//   (all rows) with leading dimension ld >= rl * nk at out + ld * (c - col0).
//   left: int32 [rl][2] device (k=2: i1; k=3: (i1, i2)); right: int32 [rr][2] device
//   (k=1: (i3, n); k=2: n).
struct BlockDesc {
  int chi, k;
  int64_t rl, nk, nk1, rr;
  const int32_t* left;
  const int32_t* right;
  int64_t col0, col1;
  int64_t ld;
  int64_t row0 = 0, row1 = 0;   // rows [row0, row1) only when row1 > row0 (written at out + (r - row0))
};
void launch_entries_block(const EntryGeom& g, const BlockDesc& b, cplx* out, cudaStream_t st);

// ------------------------------------------------------------------ TT apply (ttapply.cu)
// y[chi] = alpha * A[chi] x[chi]   (A column-major R x C), deterministic split-K
struct GemvN {
  const cplx* A[3];
  const cplx* x[3];
  cplx* y[3];
  int64_t R[3], C[3];
  int64_t lda[3];   // column stride of A (0 = R: a contiguous matrix)
  int nbatch;
};
// y[chi][c] = sum_r A[chi][r + R c] x[chi][r]  (plain transpose); if sum_batch,
// y[0][c] = sum_chi (...) (the Eq. 18 sum over chi).
struct GemvT {
  const cplx* A[3];
  const cplx* x[3];
  cplx* y[3];
  int64_t R[3], C[3];
  int64_t lda[3];   // column stride of A (0 = R)
  int nbatch;
  bool sum_batch;
  bool conj_out;  // store conj(y) (op C post-conjugation)
};

// TMA-streamed G4 pass of the GMRES pair (pairg4.cu): for every chi b < nbatch,
// y4[b] = A[b] x (CTA partials at partials[(b ns + s) rstride + r], summed in fixed order)
// and z = sum_b A[b]^T z3[b] (conj if conj_z), one read of every A[b] (R[b] x C, R <= 2048;
// R > 320 takes the row-band variant).
// x == nullptr: transpose only; z3[0] == nullptr: forward only.
struct PairG4 {
  const cplx* A[3];
  const cplx* z3[3];
  cplx* y4[3];
  const cplx* x;
  cplx* z;
  cplx* partials;
  int64_t R[3];
  int64_t C, rstride;
  int64_t ccta;   // set by the launcher: max columns per CTA
  int nslots;      // set by the launcher (large-r3 band kernel): ring slots
  int64_t slot_elems;  // set by the launcher (band kernel): complex elements per slot
  int nbatch;
  bool conj_z;
};
// false when the shape is unsupported (R > 2048 or smem): the caller falls back
bool launch_pair_g4(const PairG4& a, int max_ctas, cudaStream_t st);
int pair_g4_max_rank();
// TMA-streamed GEMV on column-major R[b] x C[b] matrices, batched over b < nbatch
// (segemv.cu, the G3 steps): op N y[b] = A[b] x[b]; op T y[b] = A[b]^T x[b] through
// per-CTA partials ([b][ns][rstride], rstride >= max C) summed in fixed order.
// false when the shape is unsupported (the caller falls back to k_gemv_n / k_gemv_t).
struct SegGemv {
  const cplx* A[3];   // row-blocked (Shard::G3b): block q = rows [R q / nsb, R (q + 1) / nsb)
  const cplx* x[3];
  cplx* y[3];
  cplx* partials;
  int64_t R[3], C[3];
  int64_t rstride;
  int nbatch;
  int nsb;            // row blocks of the layout (= CTAs)
  // op T: when xparts[b] > 0, x[b][r] = sum_{q < xparts[b]} xpart[b][q * xpart_stride[b] + r]
  // (the split-K partials of the producing GEMM, summed in fixed order on load)
  const cplx* xpart[3];
  int xparts[3];
  int64_t xpart_stride[3];
  // mode 3 (both directions from one pass): op T input xt (W2) and output yt (z3)
  const cplx* xt[3];
  cplx* yt[3];
  int64_t cmax;       // set by the launcher
  int nslots;         // set by the launcher: ring slots
  int64_t stage_elems;  // set by the launcher: complex elements per ring stage
};
bool launch_seg_gemv_mode(const SegGemv& a, int mode, cudaStream_t st, bool small_ring = false);
bool launch_seg_gemv(const SegGemv& a, bool transpose, cudaStream_t st);
bool seg_gemv_supported(int64_t R, int64_t C, int nsb);
// W2[b] = G2[b]^T W1[b] (g2t.cu): M[b] = r2, K[b] = r1 n2 rows of the column-major
// (r1 n2) x r2 core, N = n3l columns of W1 (ld K); one launch over the batch, no split-K
// partials (K split over the 8 warps of a CTA, fixed-order smem tree)
struct G2tArgs {
  const cplx* G2[3];
  const cplx* W1[3];
  cplx* W2[3];
  int M[3], K[3], ldw[3];
  int N;
  int nbatch;
};
void launch_g2t(const G2tArgs& a, cudaStream_t st);
// fixed-order sum of ns split partials ([b][s][rmax]) into a.y[b][0 .. a.R[b])
void launch_gemv_sum(const GemvN& a, cplx* partials, int ns, int64_t rmax, cudaStream_t st);
int sm_count_dev();

// partials_cap: capacity (elements) of the split-K partial buffer; the split is
// lowered so that it always fits.
void launch_gemv_n(const GemvN& a, cplx* partials, int64_t partials_cap, int max_splits, cudaStream_t st);
void launch_gemv_t(const GemvT& a, cplx* partials, int64_t partials_cap, int max_splits, cudaStream_t st);

// Expansion y[chi][i1 + n1 c] = sum_a G1[i1 + n1 a] Y2[a + r1 c], c in [0, ncol),
// with RHS blocks: column c belongs to rhs j = c / cols_per_rhs and is written at
// y + j * ld_rhs + (c % cols_per_rhs) * n1.
struct ExpandArgs {
  const cplx* G1[3];
  const cplx* Y2[3];
  cplx* y[3];
  int n1;
  int r1[3];
  int64_t ncol, cols_per_rhs, ld_rhs;
  int nbatch;
  int balanced;   // set by the launcher: contiguous (task, i1 tile) unit ranges per warp
};
void launch_expand_g1(const ExpandArgs& a, cudaStream_t st);

// Reduction W1[chi][a + r1 c] = sum_i1 G1[i1 + n1 a] u[chi][i1 + n1 c] (op T), with
// conj(u) when conj_u (op C pre-conjugation), and the same RHS block addressing
// for u as ExpandArgs::y.
struct ReduceArgs {
  const cplx* G1[3];
  const cplx* u[3];
  cplx* W1[3];
  int n1;
  int r1[3];
  int64_t ncol, cols_per_rhs, ld_rhs;
  int nbatch;
  bool conj_u;
};
// tma: the TMA-ring kernel (one launch for a batch that owns the GPU, single RHS); false keeps
// the small-footprint k_reduce_g1 (a chain kernel that shares the SMs with a concurrent stream)
void launch_reduce_g1(const ReduceArgs& a, cudaStream_t st, bool tma = false);

// out[i + ld_out j] = sum_{c<3} in[c * chi_stride + i + ld_in j] (fixed order), conj if asked;
// i < rows, j < k  (the Eq. 18 sum over chi of the per-chi transposes)
void launch_sum3(const cplx* in, int64_t chi_stride, int64_t ld_in, int64_t rows, int k, cplx* out, int64_t ld_out,
                 bool conj_out, cudaStream_t st);

// ------------------------------------------------------------------ dense complex LA (linalg.cu)
enum Trans { kN = 0, kT = 1, kC = 2 };
// C = alpha op(A) op(B) + beta C, column-major; batched over up to 3 problems with
// individual shapes.  ws/ws_elems: split-K partial workspace (may be null -> no split).
struct Zgemm {
  Trans ta = kN, tb = kN;
  int64_t M[3], N[3], K[3];
  const cplx* A[3];
  int64_t lda[3];
  const cplx* B[3];
  int64_t ldb[3];
  cplx* C[3];
  int64_t ldc[3];
  cplx alpha = {1, 0}, beta = {0, 0};
  int nbatch = 1;
};
void launch_zgemm(const Zgemm& g, cplx* ws, int64_t ws_elems, cudaStream_t st);
// same contract on FP64 tensor cores (DMMA), warp-tiled, for small / skinny
// problems; op(B) must be N.
void launch_zgemm_dmma(const Zgemm& g, cplx* ws, int64_t ws_elems, cudaStream_t st);
// conj in place
void launch_conj(cplx* x, int64_t n, cudaStream_t st);
// y[i] += x[i]
void launch_axpy1(const cplx* x, cplx* y, int64_t n, cudaStream_t st);

}  // namespace vsie
