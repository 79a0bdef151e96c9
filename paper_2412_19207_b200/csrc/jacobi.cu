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
#include <cooperative_groups.h>

#include <cstdlib>

#include "ctx.hpp"

namespace rdd {

namespace {

constexpr int kThreads = 512;
constexpr double kMinAngle = 1e-18;  // rotations by smaller angles cannot change V: skipped
constexpr size_t kCtaSmem = 227 * 1024;

struct Crit {
  double tol;        // relative (|a_pq| > tol sqrt|a_pp a_qq|) or absolute (|a_pq| > tol * dmax) threshold
  int absolute;
  double floor_lam;  // pairs with both diagonals below this are not rotated
  double conv_lam;   // only rotations touching a diagonal above this keep the sweep loop going
  double conv_angle; // ... and only those turning by more than this (|tan θ|)
  double tiny;
};

// returns 0: skip, 1: rotate (inactive for convergence), 2: rotate and count as active
__device__ __forceinline__ int rot_decision(const Crit& k, double app, double aqq, double apq) {
  const double a = fabs(apq);
  if (!(a > k.tiny)) return 0;
  const double dm = fmax(app, aqq);
  if (!(dm > k.floor_lam)) return 0;
  if (k.absolute ? !(a > k.tol) : !(a * a > k.tol * k.tol * (fabs(app) * fabs(aqq)))) return 0;
  if (!(a > kMinAngle * fabs(app - aqq))) return 0;
  return dm > k.conv_lam ? 2 : 1;
}
__device__ __forceinline__ void schur2(double app, double aqq, double apq, double& c, double& s) {
  // t = sign(θ)/(|θ| + sqrt(1 + θ²)), θ = (aqq - app)/(2 apq), rewritten with one sqrt and one
  // division: t = 2 apq sign(d) / (|d| + sqrt(d² + 4 apq²)), d = aqq - app
  const double d = aqq - app, two = 2.0 * apq;
  const double t = (d >= 0.0 ? two : -two) / (fabs(d) + sqrt(fma(d, d, two * two)));
  c = rsqrt(fma(t, t, 1.0));
  s = t * c;
}

constexpr int kRows = 32;  // rows of V per CTA in the global-memory replay

// Odd-even (Luk–Park) ordering on full column-major storage in global memory (orders whose packed
// triangle does not fit a cluster's shared memory):
// step t pairs positions (o+2k, o+2k+1), o = t&1, and every pair is rotated *and swapped*
// (Ĵ = J·Π), which makes the index movement a transposition network so all pairs meet every n
// steps, while each 2x2 update touches two contiguous 16-byte column segments.
__global__ void __launch_bounds__(1024) k_syevj_oe(double* __restrict__ Aw, const int* __restrict__ nvec,
                                                   const long long* __restrict__ off, double* __restrict__ ev,
                                                   const long long* __restrict__ ev_off, int max_sweeps,
                                                   int* __restrict__ sweeps_out, double2* __restrict__ rot,
                                                   const long long* __restrict__ rot_off, Crit crit_in,
                                                   double floor_rel, double conv_rel) {
  extern __shared__ double sm[];
  const int b = blockIdx.x;
  const int n = nvec[b];  // even (padded by the host)
  if (n <= 0) return;
  double* A = Aw + off[b];
  double* cs = sm;
  double* sn = cs + n / 2 + 1;
  double2* R = rot + rot_off[b];
  __shared__ int active;
  __shared__ double dmax;
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int i = 0; i < n; ++i) m = fmax(m, fabs(A[i + static_cast<long long>(i) * n]));
    dmax = m;
  }
  __syncthreads();
  Crit crit = crit_in;
  crit.tiny = 1e-32 * dmax;
  crit.floor_lam = fmax(floor_rel * dmax, crit_in.floor_lam);
  crit.conv_lam = fmax(conv_rel * dmax, crit_in.conv_lam);
  if (crit.absolute) crit.tol = crit_in.tol * dmax;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (threadIdx.x == 0) active = 0;
    __syncthreads();
    int local_active = 0;
    for (int t = 0; t < n; ++t) {
      const int o = t & 1;
      const int npair = o ? n / 2 - 1 : n / 2;
      for (int k = threadIdx.x; k < npair; k += blockDim.x) {
        const int p = o + 2 * k, q = p + 1;
        const double app = A[p + static_cast<long long>(p) * n], aqq = A[q + static_cast<long long>(q) * n];
        const double apq = A[p + static_cast<long long>(q) * n];
        double c = 1.0, s = 0.0;
        const int d = rot_decision(crit, app, aqq, apq);
        if (d) {
          schur2(app, aqq, apq, c, s);
          if (d == 2 && fabs(s) > crit.conv_angle * c) local_active = 1;
        }
        cs[k] = c;
        sn[k] = s;
        R[(static_cast<long long>(sweep) * n + t) * (n / 2) + k] = make_double2(c, s);
      }
      __syncthreads();
      // units: o=0 -> pairs (2u, 2u+1); o=1 -> {0}, pairs (2u-1, 2u), {n-1}
      const int nu = o ? n / 2 + 1 : n / 2;
      for (int e = threadIdx.x; e < nu * nu; e += blockDim.x) {
        const int U = e % nu, W = e / nu;
        if (U > W) continue;
        int u0, us, w0, ws;  // first index and size of each unit; pair slot for rotation lookup
        auto unit = [&](int X, int& x0, int& xs) {
          if (!o) {
            x0 = 2 * X;
            xs = 2;
          } else if (X == 0) {
            x0 = 0;
            xs = 1;
          } else if (X == nu - 1) {
            x0 = n - 1;
            xs = 1;
          } else {
            x0 = 2 * X - 1;
            xs = 2;
          }
        };
        unit(U, u0, us);
        unit(W, w0, ws);
        const int ku = o ? U - 1 : U, kw = o ? W - 1 : W;
        // Ĵ = [[s, c], [c, -s]] for a pair (rotation followed by the swap); identity for singletons
        const double cu = us == 2 ? cs[ku] : 1.0, su = us == 2 ? sn[ku] : 0.0;
        const double cw = ws == 2 ? cs[kw] : 1.0, sw = ws == 2 ? sn[kw] : 0.0;
        double* colw0 = A + static_cast<long long>(w0) * n;
        if (U == W) {
          if (us == 1) continue;
          const double app = colw0[u0], apq = colw0[u0 + n], aqq = (colw0 + n)[u0 + 1];
          const double tt = su / cu;
          colw0[u0] = aqq + tt * apq;              // swapped diagonal
          (colw0 + n)[u0 + 1] = app - tt * apq;
          colw0[u0 + 1] = 0.0;
          (colw0 + n)[u0] = 0.0;
          continue;
        }
        double a[2][2] = {{0, 0}, {0, 0}};
        for (int cc = 0; cc < ws; ++cc)
          for (int rr = 0; rr < us; ++rr) a[rr][cc] = colw0[static_cast<long long>(cc) * n + u0 + rr];
        // left: Ĵ_uᵀ, right: Ĵ_w
        double l[2][2];
        if (us == 2) {
          for (int cc = 0; cc < ws; ++cc) {
            l[0][cc] = su * a[0][cc] + cu * a[1][cc];
            l[1][cc] = cu * a[0][cc] - su * a[1][cc];
          }
        } else {
          for (int cc = 0; cc < ws; ++cc) l[0][cc] = a[0][cc];
        }
        double r[2][2];
        for (int rr = 0; rr < us; ++rr) {
          if (ws == 2) {
            r[rr][0] = sw * l[rr][0] + cw * l[rr][1];
            r[rr][1] = cw * l[rr][0] - sw * l[rr][1];
          } else {
            r[rr][0] = l[rr][0];
          }
        }
        double* colu0 = A + static_cast<long long>(u0) * n;
        for (int cc = 0; cc < ws; ++cc)
          for (int rr = 0; rr < us; ++rr) {
            colw0[static_cast<long long>(cc) * n + u0 + rr] = r[rr][cc];
            colu0[static_cast<long long>(rr) * n + w0 + cc] = r[rr][cc];
          }
      }
      __syncthreads();
    }
    if (local_active) atomicOr(&active, 1);
    __syncthreads();
    if (!active) {
      ++sweep;  // the idle sweep still permuted (swaps): keep it in the log
      break;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) ev[ev_off[b] + i] = A[i + static_cast<long long>(i) * n];
  if (threadIdx.x == 0) sweeps_out[b] = sweep;
}

__global__ void __launch_bounds__(256) k_apply_rotations_oe(double* __restrict__ Vout, const int* __restrict__ nvec,
                                                            const long long* __restrict__ off,
                                                            const double2* __restrict__ rot,
                                                            const long long* __restrict__ rot_off,
                                                            const int* __restrict__ sweeps, const int* __restrict__ ntrue,
                                                            int rpc) {
  // rpc rows of V per CTA (at most kRows; fewer for very large orders so the rows fit shared memory)
  extern __shared__ double vs[];
  const int b = blockIdx.y;
  const int n = nvec[b];  // padded (even)
  const int r0 = blockIdx.x * rpc;
  if (r0 >= n) return;
  const int rows = min(rpc, n - r0);
  const int ld = n + 1;
  for (int e = threadIdx.x; e < rpc * n; e += blockDim.x) {
    const int rr = e / n, col = e % n;
    vs[rr * ld + col] = (rr < rows && r0 + rr == col) ? 1.0 : 0.0;
  }
  __syncthreads();
  const double2* R = rot + rot_off[b];
  const int total = sweeps[b] * n;
  for (int t = 0; t < total; ++t) {
    const int o = t & 1;
    const int npair = o ? n / 2 - 1 : n / 2;
    const double2* Rt = R + static_cast<long long>(t) * (n / 2);
    for (int e = threadIdx.x; e < npair * rpc; e += blockDim.x) {
      const int k = e / rpc, rr = e % rpc;
      if (rr >= rows) continue;
      const double2 csn = Rt[k];
      const int p = o + 2 * k;
      double* row = vs + rr * ld;
      const double a = row[p], bq = row[p + 1];
      row[p] = csn.y * a + csn.x * bq;
      row[p + 1] = csn.x * a - csn.y * bq;
    }
    __syncthreads();
  }
  const int nt = ntrue[b];
  double* V = Vout + off[b];
  for (int e = threadIdx.x; e < rows * n; e += blockDim.x) {
    const int rr = e % rows, col = e / rows;
    V[(r0 + rr) + static_cast<long long>(col) * n] = vs[rr * ld + col];
  }
  (void)nt;
}


// Round-robin Jacobi with the packed triangle distributed over a K-CTA thread-block cluster
// (distributed shared memory): element e of the packed upper triangle lives in CTA e / chunk.
// Every CTA computes the round's rotations redundantly (identical inputs -> identical values),
// then updates its share of the pair-pair blocks; two cluster barriers per round.

// ============================================================================================
// Odd-even (Luk–Park) ordering on the packed upper triangle, distributed by whole columns over a
// K-CTA cluster (K = 1: one CTA). Step t pairs positions (o+2k, o+2k+1), o = t&1, and applies
// Ĵ = J·Π (rotation + swap), so after n steps every pair has met and data never moves.
//
// One cluster barrier per step. The inputs of the next step's rotation decisions — every
// diagonal entry and the superdiagonal entries (i, i+1), i ≡ o' (mod 2) — are produced in the
// update phase by whichever CTA updates them, and written into a double-buffered table that every
// CTA of the cluster holds. Each CTA then decides all pairs of the next step redundantly from its
// own table (identical inputs and code, so identical decisions) without remote reads; the only
// cross-CTA traffic is those table writes and the odd steps' boundary unit (one remote column).
// In the update phase each warp takes whole column units (largest first, snake order).
// ============================================================================================
template <int K>
__device__ __forceinline__ void publish(double* tab, int i, double v) {
  namespace cg = cooperative_groups;
#pragma unroll
  for (int r = 0; r < K; ++r) ((K > 1) ? cg::this_cluster().map_shared_rank(tab, r) : tab)[i] = v;
}

// Ĵ_Uᵀ A Ĵ_W on the blocks (U, W) of one column unit W at parity O (columns c0p, c1p; c1p unused
// for a singleton unit). Pair row units are indexed by their pair k = U - O: lane takes
// k = lane, lane+32, ..., rows (2k+O, 2k+O+1) — a branch-free loop. The singleton row unit {0} of
// odd steps, the diagonal block (with tan θ from the table, no division) and the publication of
// the next step's decision inputs are handled outside it.
template <int K, int O, class P1>
__device__ __forceinline__ void unit_update(double* c0p, P1 c1p, bool w2, double2 cw, double tw, int W, int lane,
                                            const double2* __restrict__ cs2, double* dgo, double* odo) {
  const int w0 = max(0, 2 * W - O);
  const int npu = W - O;  // pair row units above the diagonal block
  if (w2) {
    if (O == 1 && lane == 0 && W > 0) {  // block ({0}, W)
      const double a00 = c0p[0], a01 = c1p[0];
      const double r00 = cw.y * a00 + cw.x * a01, r01 = cw.x * a00 - cw.y * a01;
      c0p[0] = r00;
      c1p[0] = r01;
      if (W == 1) publish<K>(odo, 0, r00);
    }
    for (int k = lane; k < npu; k += 32) {
      const int u0 = 2 * k + O;
      const double2 cu = cs2[k];
      double a00, a10, a01, a11;
      if (O == 0) {
        const double2 x0 = *reinterpret_cast<const double2*>(c0p + u0);
        const double2 x1 = *reinterpret_cast<const double2*>(&c1p[u0]);
        a00 = x0.x;
        a10 = x0.y;
        a01 = x1.x;
        a11 = x1.y;
      } else {
        a00 = c0p[u0];
        a10 = c0p[u0 + 1];
        a01 = c1p[u0];
        a11 = c1p[u0 + 1];
      }
      // left Ĵ_Uᵀ: rows (u0, u0+1) <- (s a_u0 + c a_u1, c a_u0 - s a_u1); right Ĵ_W on the columns
      const double l00 = cu.y * a00 + cu.x * a10, l10 = cu.x * a00 - cu.y * a10;
      const double l01 = cu.y * a01 + cu.x * a11, l11 = cu.x * a01 - cu.y * a11;
      const double r00 = cw.y * l00 + cw.x * l01, r01 = cw.x * l00 - cw.y * l01;
      const double r10 = cw.y * l10 + cw.x * l11, r11 = cw.x * l10 - cw.y * l11;
      if (O == 0) {
        *reinterpret_cast<double2*>(c0p + u0) = make_double2(r00, r10);
        *reinterpret_cast<double2*>(&c1p[u0]) = make_double2(r01, r11);
      } else {
        c0p[u0] = r00;
        c0p[u0 + 1] = r10;
        c1p[u0] = r01;
        c1p[u0 + 1] = r11;
      }
    }
    if (npu > 0 && lane == ((npu - 1) & 31)) {  // (last row of unit W-1, column w0) pairs up next step
      const int r = 2 * (npu - 1) + O + 1;
      publish<K>(odo, (r - (1 - O)) >> 1, c0p[r]);
    }
    if (lane == (W & 31)) {  // diagonal block (pair unit)
      const double vpp = c0p[w0], vpq = c1p[w0], vqq = c1p[w0 + 1];
      double nd0 = vqq, nd1 = vpp;  // pure swap when s = 0
      if (cw.y != 0.0) {
        nd0 = vqq + tw * vpq;  // swapped diagonal of JᵀAJ
        nd1 = vpp - tw * vpq;
        c1p[w0] = 0.0;
      }
      c0p[w0] = nd0;
      c1p[w0 + 1] = nd1;
      publish<K>(dgo, w0, nd0);
      publish<K>(dgo, w0 + 1, nd1);
    }
  } else {  // singleton column unit (odd steps: {0} or {ne-1}): only the row rotations act
    for (int k = lane; k < npu; k += 32) {
      const int u0 = 2 * k + O;
      const double2 cu = cs2[k];
      const double a00 = c0p[u0], a10 = c0p[u0 + 1];
      c0p[u0] = cu.y * a00 + cu.x * a10;
      c0p[u0 + 1] = cu.x * a00 - cu.y * a10;
    }
    if (npu > 0 && lane == ((npu - 1) & 31)) {
      const int r = 2 * (npu - 1) + O + 1;
      publish<K>(odo, (r - (1 - O)) >> 1, c0p[r]);
    }
    if (lane == (W & 31)) publish<K>(dgo, w0, c0p[w0]);
  }
}

constexpr int kJT = 1024;  // threads per CTA (kJT/2 with two CTAs per SM for small batched blocks)
template <int K, int NT = kJT>
__global__ void __launch_bounds__(NT, kJT / NT) k_jacobi_oe(const double* __restrict__ Ain, double* __restrict__ ev,
                                                   const int* __restrict__ nvec, const long long* __restrict__ off,
                                                   const long long* __restrict__ ev_off, int max_sweeps, Crit crit_in,
                                                   double floor_rel, double conv_rel, int* __restrict__ sweeps_out,
                                                   double2* __restrict__ rot, const long long* __restrict__ rot_off,
                                                   int chunk, int nemax, int max_items, int exper) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) double smem[];
  int rank = 0;
  if constexpr (K > 1) rank = static_cast<int>(cg::this_cluster().block_rank());
  const int b = blockIdx.x / K;
  const int n = nvec[b];
  const int ne = n + (n & 1);           // even order (pad index ne-1 when n is odd: zero row/col)
  const int np = ne / 2;
  double* dg = smem + chunk;                                   // [2][nemax] diagonal tables
  double* od = dg + 2 * nemax;                                 // [2][nemax/2] next-pair superdiagonals
  double2* cs2 = reinterpret_cast<double2*>(od + nemax);       // [nemax/2] (c, s) of this step
  double* tn = reinterpret_cast<double*>(cs2 + nemax / 2);     // [nemax/2] tan θ of this step
  double** colp = reinterpret_cast<double**>(tn + nemax / 2);  // generic pointer to column j
  int* lcol = reinterpret_cast<int*>(colp + nemax);            // local start of column j
  int* items = lcol + nemax;                                   // [2][max_items] unit lists
  unsigned char* own = reinterpret_cast<unsigned char*>(items + 2 * max_items);
  __shared__ int active[2];
  __shared__ int nitems[2];
  __shared__ int cbeg, cend;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int NW = NT / 32;
  if (tid == 0) {  // even-aligned whole-column ranges of ~chunk elements; columns padded to even length
    int cur = 0, start = 0, e = 0;
    cbeg = (rank == 0) ? 0 : ne;
    cend = ne;
    for (int j = 0; j < ne; ++j) {
      if ((j & 1) == 0 && cur + 1 < K && e + 2 * j + 4 - start > chunk) {
        ++cur;
        start = e;
        if (cur == rank) cbeg = j;
        if (cur == rank + 1) cend = j;
      }
      own[j] = static_cast<unsigned char>(cur);
      lcol[j] = e - start;
      e += (j + 2) & ~1;  // column j holds rows 0..j, padded to even length
    }
    // per parity: the column units W whose first column is mine, largest first (unit W carries
    // W+1 blocks); warps take them in snake order
    for (int o = 0; o < 2; ++o) {
      int cnt = 0;
      const int nu = o ? np + 1 : np;
      for (int W = nu - 1; W >= 0; --W)
        if (own[max(0, 2 * W - o)] == rank) items[o * max_items + cnt++] = W;
      nitems[o] = cnt;
    }
    active[0] = active[1] = 0;
  }
  __syncthreads();
  for (int j = tid; j < ne; j += NT) {
    double* basep = smem;
    if constexpr (K > 1) basep = cg::this_cluster().map_shared_rank(smem, static_cast<int>(own[j]));
    colp[j] = basep + lcol[j];
  }
  const double* A = Ain + off[b];
  for (int j = cbeg + warp; j < cend; j += NW)
    for (int i = lane; i <= j; i += 32)
      smem[lcol[j] + i] = (i < n && j < n) ? A[i + static_cast<long long>(j) * n] : 0.0;
  // step-0 tables (even pairs (2k, 2k+1)) straight from global memory, in every CTA
  for (int i = tid; i < ne; i += NT) dg[i] = i < n ? A[i + static_cast<long long>(i) * n] : 0.0;
  for (int k = tid; k < np; k += NT) {
    const int p = 2 * k, q = p + 1;
    od[k] = q < n ? A[p + static_cast<long long>(q) * n] : 0.0;
  }
  if constexpr (K > 1) cg::this_cluster().sync(); else __syncthreads();
  double dmax = 0.0;
  for (int i = 0; i < n; ++i) dmax = fmax(dmax, fabs(dg[i]));
  Crit crit = crit_in;
  crit.tiny = 1e-32 * dmax;
  crit.floor_lam = fmax(floor_rel * dmax, crit_in.floor_lam);
  crit.conv_lam = fmax(conv_rel * dmax, crit_in.conv_lam);
  if (crit.absolute) crit.tol = crit_in.tol * dmax;
  double2* R = rot + rot_off[b];
  int sweep = 0;
  long long t_glob = 0;
  for (; sweep < max_sweeps; ++sweep) {
    const int sa = sweep & 1;
    for (int t = 0; t < ne; ++t, ++t_glob) {
      const int o = t & 1;
      const int bi = static_cast<int>(t_glob & 1), bo = bi ^ 1;
      const double* dgi = dg + bi * nemax;
      const double* odi = od + bi * (nemax / 2);
      const int npair = o ? np - 1 : np;
      // decide every pair of this step from the local tables
      for (int k = tid; k < npair; k += NT) {
        const int p = o + 2 * k, q = p + 1;
        const double app = dgi[p], aqq = dgi[q], apq = odi[k];
        double c = 1.0, sv = 0.0;
        const int d = exper == 2 ? 0 : rot_decision(crit, app, aqq, apq);
        if (d) {
          schur2(app, aqq, apq, c, sv);
          if (d == 2 && fabs(sv) > crit.conv_angle * c) active[sa] = 1;
        }
        cs2[k] = make_double2(c, sv);
        tn[k] = c != 0.0 ? sv / c : 0.0;
        if (rank == 0) R[(static_cast<long long>(sweep) * ne + t) * np + k] = make_double2(c, sv);
      }
      __syncthreads();
      double* dgo = dg + bo * nemax;
      double* odo = od + bo * (nemax / 2);
      const int nun = exper == 1 ? 0 : nitems[o];
      const int* ul = items + o * max_items;
      for (int r0 = 0; r0 < nun; r0 += NW) {
        const int x = r0 + (((r0 / NW) & 1) ? NW - 1 - warp : warp);
        if (x >= nun) continue;
        const int W = ul[x];
        const int w0 = max(0, 2 * W - o);
        const int kw = W - o;
        const bool w2 = kw >= 0 && kw < npair;
        const double2 cw = w2 ? cs2[kw] : make_double2(1.0, 0.0);
        const double tw = w2 ? tn[kw] : 0.0;
        double* c0p = smem + lcol[w0];  // the unit's first column is always mine
        if (!w2 || own[w0 + 1] == rank) {
          double* c1p = w2 ? smem + lcol[w0 + 1] : c0p;
          if (o) unit_update<K, 1>(c0p, c1p, w2, cw, tw, W, lane, cs2, dgo, odo);
          else unit_update<K, 0>(c0p, c1p, w2, cw, tw, W, lane, cs2, dgo, odo);
        } else {  // odd-step boundary unit: second column lives in the next CTA
          unit_update<K, 1>(c0p, colp[w0 + 1], w2, cw, tw, W, lane, cs2, dgo, odo);
        }
      }
      if constexpr (K > 1) cg::this_cluster().sync(); else __syncthreads();
    }
    const int any = active[sa];
    if (tid == 0) active[sa ^ 1] = 0;  // next sweep's flag (not read by anyone before the barrier)
    __syncthreads();
    if (!any) {
      ++sweep;  // the last sweep still swapped: it stays in the log
      break;
    }
  }
  if (rank == 0) {
    const double* dgf = dg + static_cast<int>(t_glob & 1) * nemax;
    for (int i = tid; i < ne; i += NT) ev[ev_off[b] + i] = dgf[i];
    if (tid == 0) sweeps_out[b] = sweep;
  }
  if constexpr (K > 1) cg::this_cluster().sync();  // keep shared memory alive for remote writers
}

// V = Π Ĵ_t: each warp owns one row of V in shared memory; its lanes split the (disjoint) pairs
// of a step and synchronise with __syncwarp only. The rotation log is streamed through shared
// memory in chunks of kLogRounds steps. Identity rotations (s = 0) still swap.
constexpr int kReplayWarps = 16;
constexpr int kLogRounds = 16;
__global__ void __launch_bounds__(kReplayWarps * 32) k_replay_oe(const int* __restrict__ nvec,
                                                                 const double2* __restrict__ rot,
                                                                 const long long* __restrict__ rot_off,
                                                                 const int* __restrict__ sweeps,
                                                                 double* __restrict__ Vpad,
                                                                 const long long* __restrict__ poff) {
  extern __shared__ __align__(16) double vs[];
  const int b = blockIdx.y;
  const int n = nvec[b];
  const int ne = n + (n & 1), np = ne / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * kReplayWarps + warp;
  double2* logc = reinterpret_cast<double2*>(vs + kReplayWarps * ne);  // kLogRounds x np
  double* v = vs + warp * ne;
  for (int c = lane; c < ne; c += 32) v[c] = (row == c) ? 1.0 : 0.0;
  const double2* R = rot + rot_off[b];
  const int total = sweeps[b] * ne;
  for (int t0 = 0; t0 < total; t0 += kLogRounds) {
    const int nr = min(kLogRounds, total - t0);
    __syncthreads();
    for (int e = threadIdx.x; e < nr * np; e += blockDim.x) logc[e] = R[static_cast<long long>(t0) * np + e];
    __syncthreads();
    if (row < ne) {
      for (int tt = 0; tt < nr; ++tt) {
        const int o = (t0 + tt) & 1;
        const int npair = o ? np - 1 : np;
        const double2* Rt = logc + tt * np;
        if (!o) {  // even step: aligned 16-byte pairs
          for (int k = lane; k < npair; k += 32) {
            const double2 csn = Rt[k];
            double2* vp = reinterpret_cast<double2*>(v + 2 * k);
            const double2 ab = *vp;
            *vp = make_double2(csn.y * ab.x + csn.x * ab.y, csn.x * ab.x - csn.y * ab.y);
          }
        } else {
          for (int k = lane; k < npair; k += 32) {
            const double2 csn = Rt[k];
            const int p = 1 + 2 * k;
            const double a = v[p], bq = v[p + 1];
            v[p] = csn.y * a + csn.x * bq;
            v[p + 1] = csn.x * a - csn.y * bq;
          }
        }
        __syncwarp();
      }
    }
  }
  if (row < ne) {  // row `row` of the (padded) eigenvector matrix
    double* out = Vpad + poff[b];
    for (int c = lane; c < ne; c += 32) out[row + static_cast<long long>(c) * ne] = v[c];
  }
}

// Register-resident replay: lane l of a warp holds positions [lE, lE+E) of R rows of V, so the
// even steps' pairs are lane-local and each odd step has one pair straddling lanes l and l+1
// (one shuffle each way). The rotation log is staged through shared memory kLogRounds steps at a
// time and read once per R rows; V rows leave through shared memory as coalesced columns.
constexpr int kRegWarps = 8;
template <int E, int R>
__global__ void __launch_bounds__(kRegWarps * 32) k_replay_reg(const int* __restrict__ nvec,
                                                               const double2* __restrict__ rot,
                                                               const long long* __restrict__ rot_off,
                                                               const int* __restrict__ sweeps,
                                                               double* __restrict__ Vpad,
                                                               const long long* __restrict__ poff) {
  extern __shared__ __align__(16) double2 logc[];  // kLogRounds x np, later kRegWarps*R x ne
  const int b = blockIdx.y;
  const int n = nvec[b];
  const int ne = n + (n & 1), np = ne / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rbase = blockIdx.x * kRegWarps * R;
  if (rbase >= ne) return;  // whole CTA idle (uniform)
  const int row0 = rbase + warp * R;
  const int c0 = lane * E;
  double v[R][E];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int e = 0; e < E; ++e) v[r][e] = (row0 + r == c0 + e) ? 1.0 : 0.0;
  const double2* Rl = rot + rot_off[b];
  const int total = sweeps[b] * ne;
  const int kb = c0 / 2;  // first pair index of this lane (even steps)
  for (int t0 = 0; t0 < total; t0 += kLogRounds) {
    const int nr = min(kLogRounds, total - t0);
    __syncthreads();
    for (int e = threadIdx.x; e < nr * np; e += blockDim.x) logc[e] = Rl[static_cast<long long>(t0) * np + e];
    __syncthreads();
    for (int tt = 0; tt < nr; ++tt) {
      const double2* Rt = logc + tt * np;
      if (((t0 + tt) & 1) == 0) {  // pairs (2k, 2k+1), k < np: all lane-local
#pragma unroll
        for (int i = 0; i < E / 2; ++i) {
          const int k = kb + i;
          if (k < np) {
            const double2 cs = Rt[k];
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const double a = v[r][2 * i], bb = v[r][2 * i + 1];
              v[r][2 * i] = cs.y * a + cs.x * bb;
              v[r][2 * i + 1] = cs.x * a - cs.y * bb;
            }
          }
        }
      } else {  // pairs (2k+1, 2k+2), k < np-1
        const int npair = np - 1;
        const int khi = kb + E / 2 - 1;  // (c0+E-1, c0+E): with lane+1
        const int klo = kb - 1;          // (c0-1, c0): with lane-1
        const double2 chi = khi < npair ? Rt[khi] : make_double2(1.0, 0.0);
        const double2 clo = (lane > 0 && klo < npair) ? Rt[klo] : make_double2(1.0, 0.0);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double nxt = __shfl_down_sync(0xffffffffu, v[r][0], 1);
          const double prv = __shfl_up_sync(0xffffffffu, v[r][E - 1], 1);
          const double hi = v[r][E - 1], lo = v[r][0];
          if (khi < npair) v[r][E - 1] = chi.y * hi + chi.x * nxt;
          if (lane > 0 && klo < npair) v[r][0] = clo.x * prv - clo.y * lo;
        }
#pragma unroll
        for (int i = 0; i < E / 2 - 1; ++i) {
          const int k = kb + i;
          if (k < npair) {
            const double2 cs = Rt[k];
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const double a = v[r][2 * i + 1], bb = v[r][2 * i + 2];
              v[r][2 * i + 1] = cs.y * a + cs.x * bb;
              v[r][2 * i + 2] = cs.x * a - cs.y * bb;
            }
          }
        }
      }
    }
  }
  // stage rows through shared memory, write columns of the padded V (column-major, ld ne)
  __syncthreads();
  double* st = reinterpret_cast<double*>(logc);
  const int RC = kRegWarps * R;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (c0 + e < ne) st[(c0 + e) * RC + warp * R + r] = v[r][e];
  __syncthreads();
  const int nrow = min(RC, ne - rbase);
  double* out = Vpad + poff[b];
  for (int e = threadIdx.x; e < ne * RC; e += blockDim.x) {
    const int cc = e / RC, rr = e % RC;
    if (rr < nrow) out[rbase + rr + static_cast<long long>(cc) * ne] = st[e];
  }
}

// pad to even order (zero row/column; the pad direction stays decoupled: every entry touching
// it is an exact zero) / compact back, dropping the pad eigenpair
__global__ void k_pad_copy(const double* __restrict__ A, const long long* __restrict__ off, const int* __restrict__ n,
                           double* __restrict__ W, const long long* __restrict__ woff, const int* __restrict__ npad) {
  const int b = blockIdx.x;
  const int nn = n[b], np = npad[b];
  for (long long e = threadIdx.x; e < static_cast<long long>(np) * np; e += blockDim.x) {
    const int r = static_cast<int>(e % np), cc = static_cast<int>(e / np);
    W[woff[b] + e] = (r < nn && cc < nn) ? A[off[b] + r + static_cast<long long>(cc) * nn] : 0.0;
  }
}
__global__ void k_compact(const double* __restrict__ Vp, const double* __restrict__ evp,
                          const long long* __restrict__ woff, const long long* __restrict__ eoffp,
                          const int* __restrict__ n, const int* __restrict__ npad, double* __restrict__ V,
                          const long long* __restrict__ off, double* __restrict__ ev, const long long* __restrict__ eoff) {
  const int b = blockIdx.x;
  const int nn = n[b], np = npad[b];
  __shared__ int padcol;
  if (threadIdx.x == 0) {
    padcol = -1;
    if (np != nn)
      for (int cc = 0; cc < np; ++cc)
        if (Vp[woff[b] + (np - 1) + static_cast<long long>(cc) * np] != 0.0) {
          padcol = cc;
          break;
        }
  }
  __syncthreads();
  for (long long e = threadIdx.x; e < static_cast<long long>(nn) * nn; e += blockDim.x) {
    const int r = static_cast<int>(e % nn), cc = static_cast<int>(e / nn);
    const int src = (padcol >= 0 && cc >= padcol) ? cc + 1 : cc;
    V[off[b] + e] = Vp[woff[b] + r + static_cast<long long>(src) * np];
  }
  for (int cc = threadIdx.x; cc < nn; cc += blockDim.x) {
    const int src = (padcol >= 0 && cc >= padcol) ? cc + 1 : cc;
    ev[eoff[b] + cc] = evp[eoffp[b] + src];
  }
}

// random symmetric test matrices (benchmark only): a_ij = hash(i, j, b) in [-1, 1], diagonal + n
__global__ void k_rand_sym(double* __restrict__ A, int n) {
  const int b = blockIdx.y;
  double* a = A + static_cast<size_t>(b) * n * n;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < static_cast<long long>(n) * n;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e % n), c = static_cast<int>(e / n);
    const int lo = min(r, c), hi = max(r, c);
    unsigned long long x = (static_cast<unsigned long long>(b) * 1000003ull + lo) * 1000033ull + hi;
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    const double v = static_cast<double>(x >> 11) * (2.0 / 9007199254740992.0) - 1.0;
    a[e] = (r == c) ? v + n : v;
  }
}

}  // namespace

// Jacobi throughput probe: B random symmetric matrices of order n, exactly `sweeps` sweeps
// (every pair rotates), eigenvalues and eigenvectors; returns milliseconds (CUDA events).
double bench_syevj(Ctx& c, int n, int B, int sweeps) {
  DBuf<double> A, V, ev;
  A.ensure(static_cast<size_t>(B) * n * n);
  V.ensure(static_cast<size_t>(B) * n * n);
  ev.ensure(static_cast<size_t>(B) * n);
  k_rand_sym<<<dim3(64, B), 256, 0, c.stream>>>(A.p, n);
  RDD_LAUNCH_CHECK();
  std::vector<int> nn(B, n);
  std::vector<long long> off(B);
  for (int b = 0; b < B; ++b) off[b] = static_cast<long long>(b) * n * n;
  EigOpts o;
  o.absolute = 1;
  o.tol = 1e-300;
  o.max_sweeps = sweeps;
  batched_syevj(c, A.p, V.p, ev.p, nn, off, o);  // warm-up (workspaces, attributes)
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, c.stream);
  batched_syevj(c, A.p, V.p, ev.p, nn, off, o);
  cudaEventRecord(e1, c.stream);
  RDD_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return ms;
}

// shared memory of k_jacobi_oe<K> for even order ne
static size_t oe_chunk(int ne, int K) {
  size_t tri = 0;  // columns padded to even length (aligned 16-byte row pairs)
  for (int j = 0; j < ne; ++j) tri += static_cast<size_t>((j + 2) & ~1);
  const size_t c = K == 1 ? tri : (tri + K - 1) / K + 2 * static_cast<size_t>(ne) + 4;
  return (c + 1) & ~static_cast<size_t>(1);  // tables behind it hold double2
}
static int oe_items(int ne) { return ne / 2 + 1; }  // column units of one parity
static size_t oe_smem(int ne, int K) {
  return oe_chunk(ne, K) * sizeof(double) + static_cast<size_t>(3 * ne) * sizeof(double) +
         static_cast<size_t>(ne / 2) * (sizeof(double2) + sizeof(double)) +
         static_cast<size_t>(ne) * (sizeof(double*) + sizeof(int) + 1) +
         static_cast<size_t>(2 * oe_items(ne)) * sizeof(int) + 64;
}
// smallest cluster that holds the packed triangle: more matrices in flight beat more threads per
// matrix (order 386, batch 512: K = 3 291 ms, K = 4 351 ms, K = 8 684 ms; tools/jacobi_one.py)
static int oe_k(int ne) {
  for (int K : {1, 2, 3, 4, 8})
    if (oe_smem(ne, K) <= kCtaSmem) return K;
  return 0;
}

// A: batch of symmetric n_b x n_b column-major matrices at offA[b] (the upper triangle is read);
// V receives eigenvectors (same layout), evals the eigenvalues (unsorted, concatenated).
void batched_syevj(Ctx& c, double* A, double* V, double* evals, const std::vector<int>& n,
                   const std::vector<long long>& offA, const EigOpts& o) {
  ScopedKernelTimer tk(c, "syevj");
  const int B = static_cast<int>(n.size());
  if (B == 0) return;
  const int max_sweeps = o.max_sweeps;
  Crit crit{};
  crit.tol = o.tol;
  crit.absolute = o.absolute;
  crit.floor_lam = o.floor_abs;
  crit.conv_lam = o.conv_abs;
  crit.conv_angle = o.conv_angle;
  int nmax = 0;
  for (int b = 0; b < B; ++b) nmax = std::max(nmax, n[b]);
  std::vector<long long> offE(B);
  long long e = 0;
  for (int b = 0; b < B; ++b) {
    offE[b] = e;
    e += n[b];
  }
  // padded (even-order) work layout shared by all paths
  std::vector<int> npad(B);
  std::vector<long long> woff(B), eoffp(B), roff(B);
  long long wt = 0, et = 0, rt = 0;
  for (int b = 0; b < B; ++b) {
    npad[b] = n[b] + (n[b] & 1);
    woff[b] = wt;
    wt += static_cast<long long>(npad[b]) * npad[b];
    eoffp[b] = et;
    et += npad[b];
    roff[b] = rt;
    rt += static_cast<long long>(max_sweeps) * npad[b] * std::max(1, npad[b] / 2);
  }
  DBuf<int> dn, dsw, dnp;
  DBuf<long long> doff, doffE, droff, dwoff, deoffp;
  struct WS2 {
    double2* p;
  } rot{nullptr};
  struct WS {
    double* p;
  } Vp{nullptr}, evp{nullptr};
  dn.upload(n, c.stream);
  doff.upload(offA, c.stream);
  doffE.upload(offE, c.stream);
  dnp.upload(npad, c.stream);
  dwoff.upload(woff, c.stream);
  deoffp.upload(eoffp, c.stream);
  droff.upload(roff, c.stream);
  dsw.ensure(B);
  Vp.p = c.ws("syevj.Vp", wt);
  evp.p = c.ws("syevj.ev", et);
  rot.p = reinterpret_cast<double2*>(c.ws("syevj.rot", 2 * static_cast<size_t>(std::max<long long>(1, rt))));
  const int ne = nmax + (nmax & 1);
  int K = oe_k(ne);
  const char* ex = std::getenv("RDD_JACOBI_EXP");  // tuning experiments only: 1 no update, 2 no rotation
  const int exper = ex ? std::atoi(ex) : 0;
  if (const char* e = std::getenv("RDD_JACOBI_K")) {  // experiment override (larger clusters only)
    const int k = std::atoi(e);
    if (K > 0 && k <= 8 && ((k > K && (k & (k - 1)) == 0) || (k == 3 && oe_smem(ne, 3) <= kCtaSmem))) K = k;
  }
  int swmax = 0;
  if (K > 0) {
    // ---- odd-even ordering, packed triangle on chip (one CTA or a K-CTA cluster)
    const int chunk = static_cast<int>(oe_chunk(ne, K));
    const size_t smem = oe_smem(ne, K);
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(B * K);
    // small single-CTA blocks in batches larger than the SM count: two 512-thread CTAs per SM keep
    // the whole batch resident (no partial second wave) and overlap one CTA's barrier waits
    const bool half = K == 1 && B > c.prop.multiProcessorCount && 2 * smem + 2048 <= kCtaSmem + 1024;
    // cluster CTAs: 512 threads (RDD_JACOBI_NT experiment override)
    const char* ent = std::getenv("RDD_JACOBI_NT");
    const bool half_cl = K > 1 && ent && std::atoi(ent) == 512;
    lc.blockDim = dim3(half || half_cl ? kJT / 2 : kJT);
    lc.dynamicSmemBytes = smem;
    lc.stream = c.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = K;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = K > 1 ? 1 : 0;
    auto launch = [&](auto kern) {
      RDD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      RDD_CUDA(cudaLaunchKernelEx(&lc, kern, static_cast<const double*>(A), evp.p, static_cast<const int*>(dn.p),
                                  static_cast<const long long*>(doff.p), static_cast<const long long*>(deoffp.p),
                                  max_sweeps, crit, o.floor_rel, o.conv_rel, dsw.p, rot.p,
                                  static_cast<const long long*>(droff.p), chunk, ne, oe_items(ne), exper));
      ++launch_counter();
    };
    if (K == 1 && half) launch(k_jacobi_oe<1, kJT / 2>);
    else if (K == 1) launch(k_jacobi_oe<1>);
    else if (K == 2) half_cl ? launch(k_jacobi_oe<2, kJT / 2>) : launch(k_jacobi_oe<2>);
    else if (K == 3) launch(k_jacobi_oe<3>);
    else if (K == 4) half_cl ? launch(k_jacobi_oe<4, kJT / 2>) : launch(k_jacobi_oe<4>);
    else half_cl ? launch(k_jacobi_oe<8, kJT / 2>) : launch(k_jacobi_oe<8>);
    const int E = ((ne + 31) / 32 + 1) & ~1;  // positions per lane, even
    if (E <= 16) {
      const int R = E <= 8 ? 4 : 2;
      const size_t vsm = std::max(static_cast<size_t>(kLogRounds) * (ne / 2) * sizeof(double2),
                                  static_cast<size_t>(kRegWarps) * R * ne * sizeof(double));
      const dim3 grid(ceil_div(ne, kRegWarps * R), B);
      auto rl = [&](auto kern) {
        RDD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(vsm)));
        kern<<<grid, kRegWarps * 32, vsm, c.stream>>>(dn.p, rot.p, droff.p, dsw.p, Vp.p, dwoff.p);
        RDD_LAUNCH_CHECK();
      };
      switch (E) {
        case 2: rl(k_replay_reg<2, 4>); break;
        case 4: rl(k_replay_reg<4, 4>); break;
        case 6: rl(k_replay_reg<6, 4>); break;
        case 8: rl(k_replay_reg<8, 4>); break;
        case 10: rl(k_replay_reg<10, 2>); break;
        case 12: rl(k_replay_reg<12, 2>); break;
        case 14: rl(k_replay_reg<14, 2>); break;
        default: rl(k_replay_reg<16, 2>); break;
      }
    } else {
      const size_t vsm = static_cast<size_t>(kReplayWarps) * ne * sizeof(double) +
                         static_cast<size_t>(kLogRounds) * (ne / 2) * sizeof(double2);
      RDD_CUDA(cudaFuncSetAttribute(k_replay_oe, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(vsm)));
      k_replay_oe<<<dim3(ceil_div(ne, kReplayWarps), B), kReplayWarps * 32, vsm, c.stream>>>(dn.p, rot.p, droff.p,
                                                                                             dsw.p, Vp.p, dwoff.p);
      RDD_LAUNCH_CHECK();
    }
  } else {
    // ---- odd-even ordering, full storage in global memory (very large orders)
    struct WS3 {
      double* p;
    } Wk{c.ws("syevj.Wk", wt)};
    k_pad_copy<<<B, 256, 0, c.stream>>>(A, doff.p, dn.p, Wk.p, dwoff.p, dnp.p);
    RDD_LAUNCH_CHECK();
    const size_t smem = static_cast<size_t>(ne + 2) * sizeof(double);
    k_syevj_oe<<<B, 1024, smem, c.stream>>>(Wk.p, dnp.p, dwoff.p, evp.p, deoffp.p, max_sweeps, dsw.p, rot.p, droff.p,
                                             crit, o.floor_rel, o.conv_rel);
    RDD_LAUNCH_CHECK();
    // rows of V per CTA: kRows, or as many as fit shared memory (orders above ~900)
    const int rpc = std::max(1, std::min<int>(kRows, static_cast<int>(kCtaSmem / (static_cast<size_t>(ne + 1) * sizeof(double)))));
    const size_t vsm = static_cast<size_t>(rpc) * (ne + 1) * sizeof(double);
    RDD_CUDA(cudaFuncSetAttribute(k_apply_rotations_oe, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(vsm)));
    k_apply_rotations_oe<<<dim3(ceil_div(ne, rpc), B), 256, vsm, c.stream>>>(Vp.p, dnp.p, dwoff.p, rot.p, droff.p,
                                                                               dsw.p, dn.p, rpc);
    RDD_LAUNCH_CHECK();
  }
  k_compact<<<B, 256, 0, c.stream>>>(Vp.p, evp.p, dwoff.p, deoffp.p, dn.p, dnp.p, V, doff.p, evals, doffE.p);
  RDD_LAUNCH_CHECK();
  if (c.verbose) {
    std::vector<int> sw(B);
    dsw.download(sw.data(), B, c.stream);
    RDD_CUDA(cudaStreamSynchronize(c.stream));
    double swsum = 0.0;
    for (int v : sw) {
      swmax = std::max(swmax, v);
      swsum += v;
    }
    std::fprintf(stderr, "[syevj] B=%d nmax=%d path=%s K=%d max_sweeps_used=%d mean=%.2f\n", B, nmax,
                 K == 1 ? "oe-smem" : (K ? "oe-cluster" : "oe-global"), K, swmax, swsum / B);
  }
  RDD_CUDA(cudaStreamSynchronize(c.stream));
}

}  // namespace rdd
