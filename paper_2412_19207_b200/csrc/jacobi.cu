// jacobi.cu — batched two-sided cyclic Jacobi eigensolver for symmetric matrices (FP64).
//
// Serves the PCA (eigenvectors of the Gram SᵀS and of the graded TᵀT that refines them; the
// reference takes a JacobiSVD of S, reduction.hpp:91) and the rank-deficient fallback of the
// Schwarz local solves (SelfAdjointEigenSolver, schwarz.hpp:131). One CTA per matrix; the
// upper triangle is held packed in shared memory when it fits (n <= 223), otherwise in an
// L2-resident global scratch. Rounds follow the round-robin tournament ordering (n/2 disjoint
// pairs per round, n-1 rounds per sweep); every round applies A <- JᵀAJ blockwise on 2x2
// blocks of pair-pairs and V <- VJ. Rotations use the symmetric Schur form (Golub–Van Loan
// 8.5.1) and the relative threshold |a_pq| > tol·sqrt(|a_pp a_qq|), which is what makes Jacobi
// relatively accurate on graded matrices (Demmel–Veselić) — the property the PCA refinement
// relies on.
#include "ctx.hpp"

namespace rdd {

namespace {

constexpr int kThreads = 512;
constexpr int kSmemMaxN = 223;  // n(n+1)/2 doubles + pair tables within 227 KB

__device__ __forceinline__ long long pidx(int i, int j) {  // packed upper, column-major
  if (i > j) {
    const int t = i;
    i = j;
    j = t;
  }
  return static_cast<long long>(j) * (j + 1) / 2 + i;
}

__device__ __forceinline__ int player(int pos, int r, int nn) {  // round-robin tournament
  return pos == 0 ? 0 : 1 + (pos - 1 + r) % (nn - 1);
}

__global__ void __launch_bounds__(kThreads) k_syevj(const double* __restrict__ Ain, double* __restrict__ Vout,
                                                    double* __restrict__ ev, const int* __restrict__ nvec,
                                                    const long long* __restrict__ off,
                                                    const long long* __restrict__ ev_off, double* __restrict__ scratch,
                                                    const long long* __restrict__ scr_off, int max_sweeps, double tol,
                                                    int* __restrict__ sweeps_out, int use_smem,
                                                    double2* __restrict__ rot, const long long* __restrict__ rot_off) {
  extern __shared__ double smem[];
  const int b = blockIdx.x;
  const int n = nvec[b];
  if (n <= 0) return;
  const int nn = n + (n & 1);  // even number of players (dummy = n)
  const int np = nn / 2;
  const long long smem_tri = scr_off[gridDim.x];  // packed size of the largest matrix
  const double* A = Ain + off[b];
  double2* R = rot + rot_off[b];
  (void)Vout;
  const bool in_smem = use_smem != 0;
  double* P = in_smem ? smem : scratch + scr_off[b];
  double* cs = in_smem ? smem + smem_tri : smem;  // [np] c, [np] s
  double* sn = cs + np;
  int* pp = reinterpret_cast<int*>(sn + np);
  int* qq = pp + np;
  __shared__ int active;
  __shared__ double dmax;

  // load packed upper triangle, V = I
  const long long tot = static_cast<long long>(n) * (n + 1) / 2;
  (void)tot;
  for (long long e = threadIdx.x; e < static_cast<long long>(n) * n; e += blockDim.x) {
    const int i = static_cast<int>(e % n), j = static_cast<int>(e / n);
    if (i <= j) P[pidx(i, j)] = A[e];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int i = 0; i < n; ++i) m = fmax(m, fabs(P[pidx(i, i)]));
    dmax = m;
  }
  __syncthreads();
  const double floor_abs = 1e-32 * dmax;

  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (threadIdx.x == 0) active = 0;
    __syncthreads();
    int local_active = 0;
    for (int r = 0; r < nn - 1; ++r) {
      // 1. rotations for the np disjoint pairs of this round
      for (int k = threadIdx.x; k < np; k += blockDim.x) {
        int p = player(k, r, nn), q = player(nn - 1 - k, r, nn);
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        double c = 1.0, s = 0.0;
        if (q < n) {
          const double apq = P[pidx(p, q)];
          const double app = P[pidx(p, p)], aqq = P[pidx(q, q)];
          if (fabs(apq) > floor_abs && fabs(apq) > tol * sqrt(fabs(app) * fabs(aqq))) {
            const double theta = (aqq - app) / (2.0 * apq);
            const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
            local_active = 1;
          }
        }
        cs[k] = c;
        sn[k] = s;
        pp[k] = p;
        qq[k] = q;
      }
      __syncthreads();
      // 2. A <- Jᵀ A J on unordered pair-pair blocks (P <= Q)
      for (int e = threadIdx.x; e < np * np; e += blockDim.x) {
        const int Pp = e % np, Q = e / np;
        if (Pp > Q) continue;
        const double c1 = cs[Pp], s1 = sn[Pp], c2 = cs[Q], s2 = sn[Q];
        if (s1 == 0.0 && s2 == 0.0) continue;
        const int p1 = pp[Pp], q1 = qq[Pp], p2 = pp[Q], q2 = qq[Q];
        if (Pp == Q) {
          if (q1 >= n) continue;
          const double app = P[pidx(p1, p1)], aqq = P[pidx(q1, q1)], apq = P[pidx(p1, q1)];
          const double t = s1 / c1;
          P[pidx(p1, p1)] = app - t * apq;
          P[pidx(q1, q1)] = aqq + t * apq;
          P[pidx(p1, q1)] = 0.0;
          continue;
        }
        const bool v1 = q1 < n, v2 = q2 < n;  // dummy player rows/cols do not exist
        const double a11 = P[pidx(p1, p2)];
        const double a12 = v2 ? P[pidx(p1, q2)] : 0.0;
        const double a21 = v1 ? P[pidx(q1, p2)] : 0.0;
        const double a22 = (v1 && v2) ? P[pidx(q1, q2)] : 0.0;
        // left: [[c1, -s1], [s1, c1]] ; right: [[c2, s2], [-s2, c2]]
        const double l11 = c1 * a11 - s1 * a21, l12 = c1 * a12 - s1 * a22;
        const double l21 = s1 * a11 + c1 * a21, l22 = s1 * a12 + c1 * a22;
        P[pidx(p1, p2)] = l11 * c2 - l12 * s2;
        if (v2) P[pidx(p1, q2)] = l11 * s2 + l12 * c2;
        if (v1) P[pidx(q1, p2)] = l21 * c2 - l22 * s2;
        if (v1 && v2) P[pidx(q1, q2)] = l21 * s2 + l22 * c2;
      }
      // 3. log the rotations; V is accumulated afterwards, row-parallel (k_apply_rotations)
      for (int k = threadIdx.x; k < np; k += blockDim.x)
        R[(static_cast<long long>(sweep) * (nn - 1) + r) * np + k] = make_double2(cs[k], sn[k]);
      __syncthreads();
    }
    if (local_active) atomicOr(&active, 1);
    __syncthreads();
    if (!active) break;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) ev[ev_off[b] + i] = P[pidx(i, i)];
  if (threadIdx.x == 0 && sweeps_out) sweeps_out[b] = sweep;
}

// V = J_1 J_2 ... J_R (all logged rounds): rows are independent, so each CTA keeps kRows rows
// of V in shared memory and replays the rotation log on them.
constexpr int kRows = 32;
__global__ void __launch_bounds__(256) k_apply_rotations(double* __restrict__ Vout, const int* __restrict__ nvec,
                                                         const long long* __restrict__ off,
                                                         const double2* __restrict__ rot,
                                                         const long long* __restrict__ rot_off,
                                                         const int* __restrict__ sweeps) {
  extern __shared__ double vs[];  // kRows x (n+1)
  const int b = blockIdx.y;
  const int n = nvec[b];
  const int r0 = blockIdx.x * kRows;
  if (r0 >= n) return;
  const int rows = min(kRows, n - r0);
  const int nn = n + (n & 1), np = nn / 2, ld = n + 1;
  for (int e = threadIdx.x; e < kRows * n; e += blockDim.x) {
    const int rr = e / n, col = e % n;
    vs[rr * ld + col] = (rr < rows && r0 + rr == col) ? 1.0 : 0.0;
  }
  __syncthreads();
  const double2* R = rot + rot_off[b];
  const int total = sweeps[b] * (nn - 1);
  for (int t = 0; t < total; ++t) {
    const int r = t % (nn - 1);
    const double2* Rt = R + static_cast<long long>(t) * np;
    for (int e = threadIdx.x; e < np * kRows; e += blockDim.x) {
      const int k = e / kRows, rr = e % kRows;
      const double2 csn = Rt[k];
      if (csn.y == 0.0 || rr >= rows) continue;
      int p = player(k, r, nn), q = player(nn - 1 - k, r, nn);
      if (p > q) {
        const int tmp = p;
        p = q;
        q = tmp;
      }
      double* row = vs + rr * ld;
      const double a = row[p], bq = row[q];
      row[p] = csn.x * a - csn.y * bq;
      row[q] = csn.y * a + csn.x * bq;
    }
    __syncthreads();
  }
  double* V = Vout + off[b];
  for (int e = threadIdx.x; e < rows * n; e += blockDim.x) {
    const int rr = e % rows, col = e / rows;
    V[(r0 + rr) + static_cast<long long>(col) * n] = vs[rr * ld + col];
  }
}

}  // namespace

// A: batch of symmetric n_b x n_b column-major matrices at offA[b] (only the upper triangle is
// read); V receives eigenvectors (same layout), evals[offE] the eigenvalues (unsorted).
void batched_syevj(Ctx& c, double* A, double* V, double* evals, const std::vector<int>& n,
                   const std::vector<long long>& offA, int max_sweeps, bool relative) {
  ScopedKernelTimer tk(c, "syevj");
  const int B = static_cast<int>(n.size());
  if (B == 0) return;
  std::vector<long long> offE(B), offS(B);
  long long e = 0, s = 0;
  int nmax = 0;
  for (int b = 0; b < B; ++b) nmax = std::max(nmax, n[b]);
  const bool use_smem = nmax <= kSmemMaxN;
  for (int b = 0; b < B; ++b) {
    offE[b] = e;
    e += n[b];
    offS[b] = s;
    if (!use_smem) s += static_cast<long long>(n[b]) * (n[b] + 1) / 2;
  }
  offS.push_back(use_smem ? static_cast<long long>(nmax) * (nmax + 1) / 2 : 0);  // smem triangle size
  DBuf<int> dn;
  DBuf<long long> doff, doffE, doffS;
  DBuf<double> scr, devals;
  DBuf<int> dsw;
  dn.upload(n, c.stream);
  doff.upload(offA, c.stream);
  doffE.upload(offE, c.stream);
  doffS.upload(offS, c.stream);
  scr.ensure(std::max<long long>(1, s));
  dsw.ensure(B);
  const int np = (nmax + 1) / 2;
  size_t smem = 0;
  if (use_smem)
    smem = static_cast<size_t>(nmax) * (nmax + 1) / 2 * sizeof(double);
  smem += static_cast<size_t>(np) * (2 * sizeof(double) + 2 * sizeof(int));
  RDD_CUDA(cudaFuncSetAttribute(k_syevj, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  std::vector<long long> roff(B);
  long long rtot = 0;
  for (int b = 0; b < B; ++b) {
    roff[b] = rtot;
    const int nn = n[b] + (n[b] & 1);
    rtot += static_cast<long long>(max_sweeps) * std::max(1, nn - 1) * std::max(1, nn / 2);
  }
  DBuf<double2> rot;
  DBuf<long long> droff;
  rot.ensure(std::max<long long>(1, rtot));
  droff.upload(roff, c.stream);
  const double tol = relative ? 1e-15 : 1e-15;
  k_syevj<<<B, kThreads, smem, c.stream>>>(A, V, evals, dn.p, doff.p, doffE.p, scr.p, doffS.p, max_sweeps, tol,
                                           dsw.p, use_smem ? 1 : 0, rot.p, droff.p);
  RDD_LAUNCH_CHECK();
  const size_t vsm = static_cast<size_t>(kRows) * (nmax + 1) * sizeof(double);
  RDD_CUDA(cudaFuncSetAttribute(k_apply_rotations, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(vsm)));
  k_apply_rotations<<<dim3(ceil_div(nmax, kRows), B), 256, vsm, c.stream>>>(V, dn.p, doff.p, rot.p, droff.p, dsw.p);
  RDD_LAUNCH_CHECK();
  if (c.verbose) {
    std::vector<int> sw(B);
    dsw.download(sw.data(), B, c.stream);
    RDD_CUDA(cudaStreamSynchronize(c.stream));
    int mx = 0;
    for (int v : sw) mx = std::max(mx, v);
    std::fprintf(stderr, "[syevj] B=%d nmax=%d max_sweeps_used=%d\n", B, nmax, mx);
  }
  RDD_CUDA(cudaStreamSynchronize(c.stream));
}

}  // namespace rdd
