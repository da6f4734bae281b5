/*
 * vsie_coupling.h — C ABI of the B200-native Z_bc coupling library
 * (hybrid VSIE of arXiv 2206.12409, the remote-conductor coupling block).
 *
 * What the library computes (PAPER.md = P:<line>):
 *   Z_bc in C^{q n_v x m}, q = 3 (PWC voxel testing), m RWG basis
 *   functions on the far conductors, mapping surface currents to the
 *   fields tested in the body through the dyadic Green's function
 *   G = (I + grad grad / k0^2) g, g = exp(-i k0 R)/(4 pi R).
 *   Each chi-component is a 4-D tensor n1 x n2 x n3 x m held in
 *   TT format with cores G1 (n1 x r1), G2 (r1 x n2 x r2), G3 (r2 x n3 x r3),
 *   G4 (r3 x m) (Eq. 14), built by DMRG TT-cross from an
 *   index -> value entry function and applied forward
 *    and transposed on every GMRES iteration.
 *
 * Conventions (binding):
 *  - complex values are interleaved (re, im) float64 pairs
 *    (== C99 double _Complex == torch.complex128);
 *  - row of Z: rho = chi * n_v + i1 + n1 * (i2 + n2 * i3), chi in {0,1,2} = (x,y,z)
 *    (P:227 component-major, column-major voxels);
 *  - column of Z: RWG id in canonical order: per mesh (in input order) the
 *    interior edges sorted by (min vertex id, max vertex id); T+ = the
 *    adjacent triangle with the smaller id;
 *  - entry Z[rho, n] = scale * sum_{p=1..8} w_p sum_{s=1..6} [G(r_p - r_s) J_s]_chi
 *    with 2x2x2 Gauss nodes per voxel (weights h1 h2 h3 / 8) and the interior
 *    3-point rule per triangle, J_{+,q} = (l/6)(r_{+,q} - p+),
 *    J_{-,q} = (l/6)(p- - r_{-,q});
 *  - TT cores are column-major: core k element (a, i, b) at
 *    a + r_{k-1} * (i + n_k * b), r_0 = r_4 = 1.
 *
 * Ownership: the handle owns all device memory it allocates (cores,
 * workspaces).  The caller owns every pointer it passes; device pointers must
 * stay valid until the stream-ordered call completes.  Mesh and grid arrays are
 * read during build / import only (copied).
 *
 * Errors: every int-returning call returns VSIE_OK (0), a negative error code
 * (the output handle, if any, is set to NULL) or a positive warning (valid
 * handle).  vsie_last_error_message() returns a thread-local description of
 * the last error of the calling thread.
 *
 * Threading: a handle is not re-entrant; independent handles are.
 */
#ifndef VSIE_COUPLING_H_
#define VSIE_COUPLING_H_

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VSIE_ABI_VERSION 4

/* status codes */
#define VSIE_OK 0
#define VSIE_WARN_NOT_CONVERGED 1  /* rank cap / max sweeps reached; best TT kept, error in info */
#define VSIE_ERR_ARG (-1)          /* null pointer, n <= 0, h <= 0, tol <= 0, freq <= 0, op/nrhs out of range */
#define VSIE_ERR_GEOMETRY (-2)     /* degenerate triangle, edge shared by > 2 triangles, or source nodes closer
                                      than 10 max(h) to the voxel-node bounding box (non-singular rule) */
#define VSIE_ERR_CUDA (-3)
#define VSIE_ERR_NOMEM (-4)
#define VSIE_ERR_NCCL (-5)
#define VSIE_ERR_STATE (-6)        /* call not valid for this handle (e.g. no cores yet) */

/* apply operators */
#define VSIE_OP_N 0  /* y = Z x            (forward, Eq. 17)                  */
#define VSIE_OP_T 1  /* z = Z^T u          (plain transpose, Eqs. 18-19)      */
#define VSIE_OP_C 2  /* z = Z^H u          (conjugate transpose = conj(Z^T conj u)) */

typedef struct vsie_coupling_s* vsie_coupling_t;

/* Uniform voxel grid n1 x n2 x n3.  origin = centre of voxel (0,0,0);
 * centre of voxel (i1,i2,i3) = origin + (i1 h1, i2 h2, i3 h3). */
typedef struct {
  int32_t n[3];
  double h[3];
  double origin[3];
} vsie_grid;

/* One triangulated far-domain surface (host arrays, read during build only). */
typedef struct {
  int64_t n_vertices;
  const double* xyz;     /* [n_vertices][3] */
  int64_t n_triangles;
  const int32_t* tri;    /* [n_triangles][3] vertex ids */
} vsie_mesh;

/* Build options; call vsie_build_opts_default() first, then override.  */
typedef struct {
  int32_t max_rank;      /* TT-rank cap per bond, default 2048                          */
  int32_t max_sweeps;    /* DMRG sweeps (L->R + R->L), default 8                         */
  int32_t oversample;    /* randomized range-finder oversampling p, default 16           */
  int32_t direct_svd_max;/* supercores with min dim <= this use a direct Jacobi SVD, default 384 */
  int32_t heldout;       /* held-out validation sample per chi, default 1000              */
  int32_t nrhs_max;      /* workspace sizing for block applies, default 64               */
  uint64_t seed;         /* cross initialisation + sketches + held-out sample, default 12409010 */
  double scale_re, scale_im;  /* global prefactor of every entry, default 1 + 0i          */
  int32_t rank, world;   /* this process's rank and the number of ranks, default 0, 1   */
  int32_t loopback;      /* 1: emulate `world` ranks inside this process on one GPU       */
  const void* nccl_unique_id; /* 128 bytes from vsie_nccl_unique_id() on rank 0, world > 1 */
  int32_t device;        /* CUDA device ordinal, -1 = current device                      */
  int32_t verbose;       /* 1: progress lines on stderr                                   */
  int32_t test_moment;   /* PWL test moment of the handle's 3 chi blocks (P:90 q = 12; P:381
                          * "linear terms"): 0 = PWC testing (default); l = 1, 2, 3 weights
                          * every voxel node p by (r_p - c)_l / h_l, the linear PWL test
                          * function along axis l.  The q = 12 coupling is the four handles
                          * l = 0..3 (vsie_coupling_apply_pwl).  Out of range: VSIE_ERR_ARG. */
  const char* ipc_name;  /* world > 1 without loopback: NULL (default) = NCCL (one GPU per rank, the
                          * nccl_unique_id above); else the ranks are processes sharing ONE GPU and
                          * combine through CUDA-IPC buffers and a host barrier in the POSIX shared-
                          * memory segment "/vsie_<ipc_name>" (unique per job, <= 200 chars; the
                          * segment is unlinked once every rank attached).  A test transport: every
                          * collective synchronises the stream, so applies run eagerly (no graphs). */
  int32_t quad_rule;     /* entry quadrature: 0 = 2 x 2 x 2 Gauss voxel nodes x the 3-point triangle rule
                          * (48 pairs per entry; default); 1 = the paper's rule for the far
                          * coupling block Z_bc^f, "1 volume and 1 surface integration point":
                          * the voxel centre with weight h1 h2 h3 x each triangle's centroid with the
                          * whole triangle's weight (2 pairs per entry; linear PWL moments vanish).
                          * Other values: VSIE_ERR_ARG. */
} vsie_build_opts;

typedef struct {
  int32_t n[3];
  int64_t m;
  int32_t ranks[3][3];          /* [chi][k]: r1, r2, r3                                       */
  int64_t core_bytes;           /* device bytes of all cores held by this handle (all shards) */
  int64_t compression_num, compression_den; /* (3 n_v m) / sum|cores| as a reduced fraction */
  int64_t entries_evaluated;    /* entry-function calls made by the build (all ranks)        */
  int32_t sweeps[3];
  double heldout_err[3];        /* relative L2 error of TT vs entries on the held-out sample */
  double build_s;               /* wall seconds of vsie_coupling_build                       */
  double build_entry_s, build_factor_s, build_maxvol_s; /* build breakdown (device time)      */
  int32_t slab[2];              /* this rank's owned i3 planes [slab0, slab1)                 */
  int64_t cols[2];              /* this rank's owned G4 columns [cols0, cols1)                */
  int32_t world, rank, loopback;
  double k0;
  int64_t apply_launches;       /* kernel launches made by vsie_coupling_apply* so far (this handle) */
  int64_t apply_calls;
  int32_t test_moment;          /* vsie_build_opts.test_moment of the build / import         */
  int32_t pair_schedule;        /* schedule of vsie_coupling_apply_pair: 1 = G4 read once (transpose
                                 * front, one G4 pass for both products, forward tail), 2 = G3 read
                                 * once (forward G4 pass, one G3 pass for both products, transpose
                                 * G4 pass); chosen to move fewer bytes unless configured       */
  int32_t quad_rule;            /* vsie_build_opts.quad_rule of the build / import            */
} vsie_info;

/* Per-kernel device timing of apply calls (opt-in, see vsie_coupling_set_timing). */
typedef struct {
  char name[32];
  int64_t launches;
  double total_ms;
  int64_t bytes_per_launch;     /* algorithmic HBM bytes of one launch (SURVEY §8d formula)  */
  int64_t flops_per_launch;
} vsie_timer;

int32_t vsie_abi_version(void);

/* Device-memory hook (SURVEY §8(b) "torch caching allocator hook"), process-wide: every
 * device buffer the library allocates after this call (cores, workspaces, build scratch,
 * the surface-surface blocks) comes from dev_alloc(bytes, ctx), which must return memory of
 * the current CUDA device, 256-B aligned, or NULL (the calling API returns VSIE_ERR_NOMEM).
 * Each buffer is returned through the dev_free of the hook that allocated it, after a
 * cudaDeviceSynchronize (cudaFree's ordering: a caching allocator reuses memory at once).
 * The hook functions must stay callable until every buffer they allocated is freed (the
 * handles holding them destroyed), also after another hook was installed.
 * Both NULL restores cudaMalloc / cudaFree; exactly one NULL is VSIE_ERR_ARG.  Not
 * thread-safe against concurrent library calls.  The CUDA-IPC test transport's exchange
 * buffer stays on cudaMalloc (IPC handles need it). */
int32_t vsie_set_allocator(void* (*dev_alloc)(size_t bytes, void* ctx), void (*dev_free)(void* ptr, void* ctx),
                           void* ctx);
void vsie_build_opts_default(vsie_build_opts* opts);
const char* vsie_status_string(int32_t status);
const char* vsie_last_error_message(void);

/* Slab partition of design (iii), host-only: rank `rank` of `world`
 * owns voxel planes i3 in [slab[0], slab[1]) and G4 columns [cols[0], cols[1]);
 * planes are split as n3 p / P, columns in equal padded chunks ceil(m / P) (the
 * allgather of z needs equal counts).  Pure function, no CUDA call. */
int32_t vsie_slab_partition(int32_t n3, int64_t m, int32_t world, int32_t rank, int32_t slab[2], int64_t cols[2]);

/* 128-byte NCCL unique id for a multi-process group (rank 0 calls it and
 * broadcasts the bytes; every rank passes them in vsie_build_opts). */
int32_t vsie_nccl_unique_id(void* out128);

/* Build Z_bc in TT form by DMRG TT-cross over the entry function.
 * Collective and synchronous: every rank calls it with identical arguments
 * except opts->rank.  tol is the relative Frobenius target per chi-tensor
 * (P:287 uses 1e-3; BASELINE configs use 1e-8 / 1e-6).  On VSIE_OK or
 * VSIE_WARN_NOT_CONVERGED *out is a valid handle. */
int32_t vsie_coupling_build(const vsie_grid* grid, const vsie_mesh* meshes, int32_t n_meshes,
                            double freq_hz, double tol, const vsie_build_opts* opts,
                            vsie_coupling_t* out);

/* Create a handle from existing cores (the "store and recycle" of P:375).
 * ranks[chi*3 + k] = r_{k+1}; host_cores[chi*4 + k] = column-major core k+1
 * (complex128) of component chi.  Each rank keeps only its owned shards. */
int32_t vsie_coupling_import_cores(const vsie_grid* grid, const vsie_mesh* meshes, int32_t n_meshes,
                                   double freq_hz, const int32_t ranks[9],
                                   const void* const host_cores[12], const vsie_build_opts* opts,
                                   vsie_coupling_t* out);

/* Copy core k (0..3) of component chi (0..2) to host (full core, assembled from
 * the loopback shards).  Single-process handles only (VSIE_ERR_STATE for a
 * multi-process handle, whose ranks hold only their slabs).  With host_dst ==
 * NULL only *nelems is written. */
int32_t vsie_coupling_export_cores(vsie_coupling_t h, int32_t chi, int32_t k, void* host_dst,
                                   int64_t* nelems);

/* TT rounding (recompression) of the handle's cores in place: SURVEY §8(f) NEXT-1,
 * motivated by PAPER.md P:389 ("[cross] might overestimate the TT-ranks") and built
 * from the unfolding SVDs of P:126 (TT-SVD of the tensor already in TT form, the
 * "TT-rounding" of the cited Oseledets 2011; restated in oracle/ttround.py):
 * right-to-left orthogonalisation of cores 4..2, then left-to-right truncated SVDs
 * with per-bond threshold tol / sqrt(3) * ||Z~chi||_F, so that the rounded TT is
 * within tol ||Z~chi||_F of the unrounded one for each chi, at the TT-SVD ranks of
 * that tensor.  tol in [0, 1); tol = 0 removes only numerically redundant ranks
 * (singular values <= 1e-14 of the largest).  Synchronous; afterwards vsie_info
 * reports the new ranks and previously captured apply graphs are dropped.
 * Single-process handles only (world 1 or loopback): VSIE_ERR_STATE otherwise. */
int32_t vsie_coupling_round(vsie_coupling_t h, double tol);

/* Apply the TT operator on `stream` (cudaStream_t, NULL = legacy default).
 *  OP_N: x = device complex128 [m x nrhs] (column-major, ld = m, replicated on
 *        every rank) -> y = device complex128 [3 * n1 * n2 * (slab1 - slab0) x nrhs]
 *        (the rank's slab; chi-major, i1 fastest; ld = rows).
 *  OP_T / OP_C: x = the rank's slab of u (layout as y above) -> y = z [m x nrhs],
 *        replicated on every rank after the collective.
 * 1 <= nrhs <= nrhs_max.  Asynchronous; collective when world > 1. */
int32_t vsie_coupling_apply(vsie_coupling_t h, const void* x, void* y, int32_t op, int32_t nrhs,
                            void* stream);

/* The coupling pair of one GMRES matvec of the hybrid system (Eq. 11 / 15: the
 * body rows need Z_bc j_c, the conductor rows Z_cb j_b = Z_bc^T j_b, Eqs. 17-19):
 * y = Z x (layouts as OP_N above) and z = Z^T u (adj_op = OP_T) or Z^H u (OP_C) (layouts
 * as OP_T), single right-hand side, in one call.  One of the two large cores is streamed
 * once for both directions (vsie_info.pair_schedule): G4 (r3 x m) when it is the larger,
 * by running the transpose's G1-G3 steps first so that one TMA-streamed pass over G4 forms
 * y4 = G4 x and z = sum_chi G4^T z3 (the chi sum of Eq. 18), else G3 ((r2 n3) x r3), by
 * running the forward's G4 pass first so that one pass over G3 forms Y3 = G3 y4 and
 * z3 = G3^T W2.  Results equal two vsie_coupling_apply calls to rounding and are bitwise
 * reproducible.  Asynchronous; collective when world > 1. */
int32_t vsie_coupling_apply_pair(vsie_coupling_t h, const void* x, void* y, const void* u, void* z, int32_t adj_op,
                                 void* stream);

/* Same as apply but x and y are HOST buffers: H2D copy, apply, D2H copy,
 * synchronous (the end-to-end call of a CPU-resident GMRES). */
int32_t vsie_coupling_apply_host(vsie_coupling_t h, const void* x_host, void* y_host, int32_t op,
                                 int32_t nrhs);

/* apply_pair with HOST buffers (H2D of x and u, the pair, D2H of y and z; synchronous).
 * Pinned host buffers are strongly recommended (pageable ones serialise the copies).
 * Single process, chain schedule: the forward (needs only x) runs first on one stream and
 * its voxel result is copied out while u is copied in on a second stream for the
 * transpose, so the two large copies overlap; the results equal apply_pair's to rounding
 * (the G4 pass is not shared in this schedule).  Otherwise the fused device pair. */
int32_t vsie_coupling_apply_pair_host(vsie_coupling_t h, const void* x_host, void* y_host, const void* u_host,
                                      void* z_host, int32_t adj_op);

/* PWL (q = 12) coupling: the four handles h[l] built with
 * test_moment = l (l = 0..3) on the same grid, meshes, frequency and partition.
 * The 12 n_v-row operator stacks their blocks moment-major:
 *   OP_N:       y = [Z_0 x; Z_1 x; Z_2 x; Z_3 x]; y holds 4 consecutive blocks, block l
 *               = Z_l X as in vsie_coupling_apply (3 n_v,loc x nrhs, ld 3 n_v,loc).  For
 *               nrhs = 1 this is the vector ordered (moment, chi, voxel).
 *   OP_T/OP_C:  z = sum_l Z_l^op u_l, u in the same 4-block layout, z m x nrhs; the four
 *               partial products are summed in the order l = 0, 1, 2, 3 on device.
 * Device pointers, stream-ordered on `stream`; x, y, u, z as in vsie_coupling_apply.  A
 * device scratch of 3 m nrhs complex128 is held by h[0].  On one process the four handles
 * run concurrently on four streams (VSIE_PWL_CONCURRENT=0: in turn); multi-process
 * handles (world > 1, each with its own NCCL unique id) run in turn.  Errors: VSIE_ERR_ARG for a NULL
 * handle, handles with moments other than 0, 1, 2, 3 in that order, or mismatched
 * geometry / partition; otherwise as vsie_coupling_apply. */
int32_t vsie_coupling_apply_pwl(const vsie_coupling_t h[4], const void* x, void* y, int32_t op, int32_t nrhs,
                                void* stream);

/* The q = 12 GMRES coupling pair (single RHS): y = Z_pwl x and z = Z_pwl^T u (adj_op
 * OP_T) or Z_pwl^H u (OP_C), layouts as vsie_coupling_apply_pwl; each moment handle runs
 * its fused pair (vsie_coupling_apply_pair), then the z sum in the order l = 0..3.
 * Errors as vsie_coupling_apply_pwl and vsie_coupling_apply_pair. */
int32_t vsie_coupling_apply_pair_pwl(const vsie_coupling_t h[4], const void* x, void* y, const void* u, void* z,
                                     int32_t adj_op, void* stream);

/* Exact quadrature entries (the cross's black box, not the TT value):
 * idx = device int64 [count][2] (row, col), out = device complex128 [count].
 * Rows and columns are global indices (any rank may evaluate any entry). */
int32_t vsie_coupling_entries(vsie_coupling_t h, const int64_t* idx, int64_t count, void* out,
                              void* stream);

/* Structured supercore block of the TT-cross (the cross evaluates the
 * entry function on index sets, not on arbitrary lists): the matrix
 *   M_k[(a, i_k), (i_{k+1}, b)] = Z_chi(I[a], i_k, i_{k+1}, J[b]),  rows a + n_left i_k, columns
 *   i_{k+1} + n_{k+1} b,  k = 1, 2, 3, evaluated by the same entry kernel as the build.
 * left: device int32 [n_left][2] -- k = 1: ignored (n_left = 1), k = 2: (i1, -), k = 3: (i1, i2);
 * right: device int32 [n_right][2] -- k = 1: (i3, n), k = 2: (n, -), k = 3: ignored (n_right = 1).
 * out: device complex128, column-major (n_left n_k) x (n_{k+1} n_right).  Entries are the exact
 * quadrature values (same definition as vsie_coupling_entries).  Errors: VSIE_ERR_ARG for
 * chi / k out of range, n_left / n_right < 1, NULL pointers. */
int32_t vsie_coupling_supercore(vsie_coupling_t h, int32_t chi, int32_t k, const int32_t* left, int32_t n_left,
                                const int32_t* right, int32_t n_right, void* out, void* stream);

/* TT value at (row, col) pairs (Eq. 9 chain product), same
 * layout as vsie_coupling_entries.  world == 1 handles only. */
int32_t vsie_coupling_tt_eval(vsie_coupling_t h, const int64_t* idx, int64_t count, void* out,
                              void* stream);

int32_t vsie_coupling_info(vsie_coupling_t h, vsie_info* out);

/* Per-kernel CUDA-event timing of subsequent apply calls: enable = 1 starts
 * (and resets) it with the chains serialised on the caller's stream (clean per-kernel
 * durations), enable = 2 keeps the chains concurrent (timeline, vsie_coupling_trace),
 * 0 stops it.  vsie_coupling_timers copies up to `max`
 * accumulated timers (synchronises the handle's streams). */
int32_t vsie_coupling_set_timing(vsie_coupling_t h, int32_t enable);
int32_t vsie_coupling_timers(vsie_coupling_t h, vsie_timer* out, int32_t max, int32_t* n_out);

/* Execution strategy: use_graphs = 1 (default) replays each apply / pair (op, nrhs, pointers)
 * as a captured CUDA graph (single-process handles), 0 launches eagerly.  pair_schedule
 * selects the schedule of vsie_coupling_apply_pair: 0 (default) the one that moves fewer
 * bytes, 1 G4 read once, 2 G3 read once.  Negative = keep.  Synchronises the device. */
int32_t vsie_coupling_configure(vsie_coupling_t h, int32_t use_graphs, int32_t pair_schedule);

/* Timeline of apply calls made with vsie_coupling_set_timing(h, 2): the chi chains run
 * concurrently (as in the captured graph, but launched eagerly) with a CUDA event pair
 * around every kernel; each record gives the kernel's start / end in ms relative to the
 * start of its apply call.  Copies up to `max` records, clears them, *n_out = count. */
typedef struct {
  char name[32];
  int32_t chi;                  /* chain (0..2), -1 for the join / combine steps      */
  int32_t call;                 /* index of the apply call since timing was enabled   */
  double t0_ms, t1_ms;
} vsie_trace;
int32_t vsie_coupling_trace(vsie_coupling_t h, vsie_trace* out, int32_t max, int32_t* n_out);

void vsie_coupling_destroy(vsie_coupling_t h);

#ifdef __cplusplus
}
#endif
#endif /* VSIE_COUPLING_H_ */
