// Standalone self-test of the hot-path kernels against naive host loops
// (developer tool; built and run on the GPU box:  see tools/run_selftest.sh).
#include <cstdio>
#include <cstdlib>
#include <complex>
#include <random>
#include <vector>

#include "../paper_2206_12409_b200/csrc/kernels.cuh"

using namespace vsie;
typedef std::complex<double> zc;

static std::mt19937_64 rng(1234);
static std::vector<zc> randv(size_t n) {
  std::normal_distribution<double> d;
  std::vector<zc> v(n);
  for (auto& x : v) x = zc(d(rng), d(rng));
  return v;
}
static cplx* up(const std::vector<zc>& v) {
  cplx* p;
  cudaMalloc(&p, v.size() * 16 + 16);
  cudaMemcpy(p, v.data(), v.size() * 16, cudaMemcpyHostToDevice);
  return p;
}
static std::vector<zc> down(const cplx* p, size_t n) {
  std::vector<zc> v(n);
  cudaDeviceSynchronize();
  cudaMemcpy(v.data(), p, n * 16, cudaMemcpyDeviceToHost);
  return v;
}
static double relerr(const std::vector<zc>& a, const std::vector<zc>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) { num += std::norm(a[i] - b[i]); den += std::norm(b[i]); }
  return std::sqrt(num / (den > 0 ? den : 1));
}
static int fails = 0;
static void report(const char* what, double e) {
  printf("%-40s rel err %.3e %s\n", what, e, e < 1e-13 ? "ok" : "FAIL");
  if (!(e < 1e-13)) ++fails;
}

static zc opel(const std::vector<zc>& A, int64_t ld, int t, int64_t r, int64_t c) {
  if (t == kN) return A[r + ld * c];
  zc v = A[c + ld * r];
  return t == kC ? std::conj(v) : v;
}

void test_zgemm(int ta, int tb, int64_t M, int64_t N, int64_t K, bool ws, bool use_dmma = false) {
  int64_t lda = ta == kN ? M : K, ldb = tb == kN ? K : N;
  auto A = randv(lda * (ta == kN ? K : M)), B = randv(ldb * (tb == kN ? N : K)), Cc = randv(M * N);
  cplx *dA = up(A), *dB = up(B), *dC = up(Cc);
  cplx* dws = nullptr;
  if (ws) cudaMalloc(&dws, 64 * M * N * 16);
  Zgemm g{};
  g.ta = (Trans)ta; g.tb = (Trans)tb; g.nbatch = 1;
  g.M[0] = M; g.N[0] = N; g.K[0] = K; g.A[0] = dA; g.lda[0] = lda; g.B[0] = dB; g.ldb[0] = ldb;
  g.C[0] = dC; g.ldc[0] = M; g.alpha = cmk(0.5, -1); g.beta = cmk(2, 0.25);
  if (use_dmma) launch_zgemm_dmma(g, dws, ws ? 64 * M * N : 0, 0); else launch_zgemm(g, dws, ws ? 64 * M * N : 0, 0);
  auto got = down(dC, M * N);
  std::vector<zc> ref(M * N);
  for (int64_t j = 0; j < N; ++j)
    for (int64_t i = 0; i < M; ++i) {
      zc s = 0;
      for (int64_t k = 0; k < K; ++k) s += opel(A, lda, ta, i, k) * opel(B, ldb, tb, k, j);
      ref[i + M * j] = zc(0.5, -1) * s + zc(2, 0.25) * Cc[i + M * j];
    }
  char buf[128];
  snprintf(buf, sizeof buf, "zgemm%s ta%d tb%d %ldx%ldx%ld ws%d", use_dmma ? "_dmma" : "", ta, tb, (long)M, (long)N, (long)K, (int)ws);
  report(buf, relerr(got, ref));
  cudaFree(dA); cudaFree(dB); cudaFree(dC); if (dws) cudaFree(dws);
}

void test_gemv_n(int64_t R, int64_t C) {
  auto A = randv(R * C), x = randv(C);
  cplx *dA = up(A), *dx = up(x), *dy;
  cudaMalloc(&dy, R * 16);
  cplx* part; cudaMalloc(&part, 3 * 1024 * (R + 256) * 16);
  unsigned* ctr; cudaMalloc(&ctr, 3 * 8192 * 4); cudaMemset(ctr, 0, 3 * 8192 * 4);
  GemvN g{};
  g.nbatch = 1; g.A[0] = dA; g.x[0] = dx; g.y[0] = dy; g.R[0] = R; g.C[0] = C;
  launch_gemv_n(g, part, 3 * 1024 * (R + 256), 1024, 0);
  auto got = down(dy, R);
  std::vector<zc> ref(R, 0);
  for (int64_t c = 0; c < C; ++c) for (int64_t r = 0; r < R; ++r) ref[r] += A[r + R * c] * x[c];
  char buf[128]; snprintf(buf, sizeof buf, "gemv_n %ldx%ld", (long)R, (long)C);
  report(buf, relerr(got, ref));
  // run again: counters must have been reset
  launch_gemv_n(g, part, 3 * 1024 * (R + 256), 1024, 0);
  report("gemv_n repeat", relerr(down(dy, R), ref));
  cudaFree(dA); cudaFree(dx); cudaFree(dy); cudaFree(part); cudaFree(ctr);
}

void test_gemv_t(int64_t R, int64_t C, bool sum3) {
  int nb = sum3 ? 3 : 1;
  std::vector<std::vector<zc>> A(nb), x(nb);
  GemvT g{};
  g.nbatch = nb; g.sum_batch = sum3; g.conj_out = false;
  cplx* dy; cudaMalloc(&dy, C * 16);
  for (int b = 0; b < nb; ++b) {
    int64_t Rb = R + 3 * b;
    A[b] = randv(Rb * C); x[b] = randv(Rb);
    g.A[b] = up(A[b]); g.x[b] = up(x[b]); g.y[b] = dy; g.R[b] = Rb; g.C[b] = C;
  }
  cplx* part; cudaMalloc(&part, 3 * 1024 * (C + 64) * 16);
  unsigned* ctr; cudaMalloc(&ctr, 3 * 8192 * 4); cudaMemset(ctr, 0, 3 * 8192 * 4);
  launch_gemv_t(g, part, 3 * 1024 * (C + 64), 1024, 0);
  auto got = down(dy, C);
  std::vector<zc> ref(C, 0);
  for (int b = 0; b < nb; ++b)
    for (int64_t c = 0; c < C; ++c) for (int64_t r = 0; r < g.R[b]; ++r) ref[c] += A[b][r + g.R[b] * c] * x[b][r];
  char buf[128]; snprintf(buf, sizeof buf, "gemv_t %ldx%ld sum%d", (long)R, (long)C, (int)sum3);
  report(buf, relerr(got, ref));
}

void test_expand(int n1, int r1, int64_t ncol, int64_t cpr) {
  auto G1 = randv(n1 * r1), Y2 = randv(r1 * ncol);
  int64_t nrhs = (ncol + cpr - 1) / cpr, ld = n1 * cpr + 7;
  cplx *dG = up(G1), *dY2 = up(Y2), *dy;
  cudaMalloc(&dy, ld * nrhs * 16); cudaMemset(dy, 0, ld * nrhs * 16);
  ExpandArgs e{};
  e.nbatch = 1; e.n1 = n1; e.r1[0] = r1; e.G1[0] = dG; e.Y2[0] = dY2; e.y[0] = dy;
  e.ncol = ncol; e.cols_per_rhs = cpr; e.ld_rhs = ld;
  launch_expand_g1(e, 0);
  auto got = down(dy, ld * nrhs);
  std::vector<zc> ref(ld * nrhs, 0);
  for (int64_t c = 0; c < ncol; ++c)
    for (int i = 0; i < n1; ++i) {
      zc s = 0;
      for (int a = 0; a < r1; ++a) s += G1[i + n1 * a] * Y2[a + r1 * c];
      ref[(c / cpr) * ld + (c % cpr) * n1 + i] = s;
    }
  char buf[128]; snprintf(buf, sizeof buf, "expand n1=%d r1=%d ncol=%ld", n1, r1, (long)ncol);
  report(buf, relerr(got, ref));
}

void test_reduce(int n1, int r1, int64_t ncol, int64_t cpr, bool cj) {
  int64_t nrhs = (ncol + cpr - 1) / cpr, ld = n1 * cpr + 5;
  auto G1 = randv(n1 * r1), u = randv(ld * nrhs);
  cplx *dG = up(G1), *du = up(u), *dW;
  cudaMalloc(&dW, r1 * ncol * 16);
  ReduceArgs r{};
  r.nbatch = 1; r.n1 = n1; r.r1[0] = r1; r.G1[0] = dG; r.u[0] = du; r.W1[0] = dW;
  r.ncol = ncol; r.cols_per_rhs = cpr; r.ld_rhs = ld; r.conj_u = cj;
  launch_reduce_g1(r, 0);
  auto got = down(dW, r1 * ncol);
  std::vector<zc> ref(r1 * ncol, 0);
  for (int64_t c = 0; c < ncol; ++c)
    for (int a = 0; a < r1; ++a) {
      zc s = 0;
      for (int i = 0; i < n1; ++i) {
        zc uv = u[(c / cpr) * ld + (c % cpr) * n1 + i];
        s += G1[i + n1 * a] * (cj ? std::conj(uv) : uv);
      }
      ref[a + r1 * c] = s;
    }
  char buf[128]; snprintf(buf, sizeof buf, "reduce n1=%d r1=%d ncol=%ld cj=%d", n1, r1, (long)ncol, (int)cj);
  report(buf, relerr(got, ref));
}

void jacobi_probe(int64_t p, int q, double decades);
int main(int argc, char** argv) {
  if (argc > 1) {
    jacobi_probe(7370, 272, 4);
    jacobi_probe(7370, 272, 14);
    jacobi_probe(272, 272, 7);
    return 0;
  }
  for (int ta = 0; ta < 3; ++ta)
    for (int tb = 0; tb < 3; ++tb) test_zgemm(ta, tb, 84, 12, 31, false);
  test_zgemm(0, 0, 130, 70, 300, true);
  test_zgemm(1, 0, 63, 220, 2400, true);
  test_zgemm(2, 0, 200, 33, 1000, true);
  for (int ta = 0; ta < 3; ++ta) test_zgemm(ta, 0, 84, 12, 31, false, true);
  test_zgemm(0, 0, 1200, 110, 71, true, true);
  test_zgemm(1, 0, 71, 110, 1200, true, true);
  test_zgemm(2, 0, 37, 5, 1001, true, true);
  test_gemv_n(73, 1128);
  test_gemv_n(372, 73);
  test_gemv_n(1000, 3000);
  test_gemv_t(372, 73, false);
  test_gemv_t(73, 1128, true);
  test_gemv_t(5000, 300, false);
  test_expand(12, 7, 144, 144);
  test_expand(100, 10, 1000, 300);
  test_expand(200, 16, 517, 517);
  test_reduce(12, 7, 144, 144, false);
  test_reduce(100, 10, 1000, 300, true);
  test_reduce(200, 20, 517, 517, false);
  test_reduce(64, 32, 300, 100, true);
  test_expand(64, 32, 300, 100);
  test_gemv_n(7810, 267);
  test_gemv_n(267, 10080);
  test_gemv_t(7810, 267, false);
  cudaError_t e = cudaDeviceSynchronize();
  printf("cuda: %s\n", cudaGetErrorString(e));
  printf("%s (%d failures)\n", fails ? "SELFTEST FAILED" : "SELFTEST PASSED", fails);
  return fails ? 1 : 0;
}

// ---- Jacobi convergence / timing probe (developer tool, not a test)
#include "../paper_2206_12409_b200/csrc/crosskern.cuh"
#include <chrono>
void jacobi_probe(int64_t p, int q, double decades) {
  // A = random (p x q) with columns scaled by 10^(-decades j / q): graded
  auto A = randv(p * q);
  for (int j = 0; j < q; ++j) {
    double s = std::pow(10.0, -decades * j / q);
    for (int64_t i = 0; i < p; ++i) A[i + p * j] *= s;
  }
  cplx* dA = up(A);
  int Q = q + (q & 1);
  std::vector<int2> pairs;
  std::vector<int> L(Q);
  for (int t = 0; t < Q - 1; ++t) {
    L[0] = 0;
    for (int i = 0; i < Q - 1; ++i) L[i + 1] = (t + i) % (Q - 1) + 1;
    for (int k = 0; k < Q / 2; ++k) pairs.push_back(make_int2(L[k], L[Q - 1 - k]));
  }
  int2* dp; cudaMalloc(&dp, pairs.size() * sizeof(int2));
  cudaMemcpy(dp, pairs.data(), pairs.size() * sizeof(int2), cudaMemcpyHostToDevice);
  unsigned* cnt; cudaMalloc(&cnt, 4);
  auto t0 = std::chrono::steady_clock::now();
  int sweeps = 0;
  for (; sweeps < 40; ++sweeps) {
    cudaMemset(cnt, 0, 4);
    for (int t = 0; t < Q - 1; ++t) launch_jacobi_round(dA, p, p, nullptr, q, dp + (int64_t)t * (Q / 2), Q / 2, 1e-12, 0.0, cnt, 0);
    unsigned h = 0; cudaMemcpy(&h, cnt, 4, cudaMemcpyDeviceToHost);
    printf("   sweep %d rotations %u\n", sweeps, h);
    if (!h) break;
  }
  double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  printf("jacobi probe p=%ld q=%d decades=%.0f: %d sweeps, %.3f s, %.1f us/round\n", (long)p, q, decades, sweeps + 1, s, 1e6 * s / ((sweeps + 1) * (Q - 1)));
  cudaFree(dA); cudaFree(dp); cudaFree(cnt);
}
