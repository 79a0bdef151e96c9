// diag.cu — §8(f) row 4: the dense diagnostics of the reference (krylov.hpp:403-440 `spectrum`,
// `singular_values`, `condition_number`; runner.hpp:344-362 `spectrum_cmd`, :372-400 `sweep_tau`)
// on the device.
//
//   spectrum(A)         Householder reduction to upper Hessenberg form (one reflector per column:
//                       generate, apply from the left one warp per column, apply from the right as
//                       row partials + ordered sum + rank-1 update), then the Francis double-shift
//                       QR iteration for the eigenvalues only (the EISPACK hqr form: deflation on a
//                       negligible subdiagonal, exceptional shifts every 10 iterations) in one CTA.
//                       Eigen's EigenSolver (computeEigenvectors = false) runs the same reduction and
//                       real-Schur iteration.
//   symmetric spectrum  the same reduction of a symmetric matrix is tridiagonal; its eigenvalues
//                       come from Sturm-count bisection, one thread per eigenvalue.
//   singular_values(A)  Householder bidiagonalisation (column, then row reflectors), then bisection
//                       on the Golub–Kahan tridiagonal [[0, B], [Bᵀ, 0]] whose eigenvalues are ±σ.
//                       Eigen's BDCSVD also starts from a bidiagonalisation.
//   condition_number    σ_max / smallest positive σ (krylov.hpp:430-440).
//
// All three reductions are HBM/L2-bound streams over the n×n matrix (Σ_k ~4·(n−k)·n doubles);
// the QR iteration and the bisection are latency-bound. Dense cap 4000 as kDenseSpectrumCap.
#include <algorithm>
#include <cfloat>
#include <complex>

#include "ctx.hpp"

namespace rdd {

namespace {

constexpr int kHT = 256;

__device__ __forceinline__ double block_sum_d(double v, double* sh) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) sh[0] = t;
  }
  __syncthreads();
  return sh[0];
}

// Reflector of x[0..L) (stride inc), dlarfg form: H = I − τ v vᵀ with v_0 = 1 maps x to β e_0.
// x[0] = β, x[1..] = 0; v written contiguously; scal[0] = τ.
__global__ void __launch_bounds__(kHT) k_house(double* __restrict__ x, long long inc, int L, double* __restrict__ v,
                                               double* __restrict__ scal) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int i = 1 + threadIdx.x; i < L; i += blockDim.x) {
    const double t = x[i * inc];
    s += t * t;
  }
  const double xnorm = sqrt(block_sum_d(s, sh));
  const double alpha = x[0];
  double tau = 0.0, scale = 0.0, beta = alpha;
  if (xnorm > 0.0) {
    beta = -copysign(hypot(alpha, xnorm), alpha);
    tau = (beta - alpha) / beta;
    scale = 1.0 / (alpha - beta);
  }
  for (int i = 1 + threadIdx.x; i < L; i += blockDim.x) {
    v[i] = x[i * inc] * scale;
    x[i * inc] = 0.0;
  }
  if (threadIdx.x == 0) {
    v[0] = 1.0;
    x[0] = beta;
    scal[0] = tau;
  }
}

// A[r0:r0+L, j] −= τ v (vᵀ A[r0:r0+L, j]) for j in [c0, c1): one warp per column
__global__ void k_left_apply(double* __restrict__ A, long long lda, int r0, int L, int c0, int c1,
                             const double* __restrict__ v, const double* __restrict__ scal) {
  const int j = c0 + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= c1) return;
  const double tau = scal[0];
  if (tau == 0.0) return;
  double* a = A + j * lda + r0;
  double s = 0.0;
  for (int i = lane; i < L; i += 32) s += v[i] * a[i];
  s = warp_sum(s) * tau;
  for (int i = lane; i < L; i += 32) a[i] -= s * v[i];
}

// right application A[r0:r1, c0:c0+L] (I − τ v vᵀ): (1) u partials over 64-column chunks,
// (2) ordered sum of the chunks, (3) rank-1 update
constexpr int kRC = 64;
__global__ void k_right_part(const double* __restrict__ A, long long lda, int r0, int r1, int c0, int L,
                             const double* __restrict__ v, double* __restrict__ part, long long ldp) {
  const int i = r0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r1) return;
  const int q0 = blockIdx.y * kRC, q1 = min(L, q0 + kRC);
  double s = 0.0;
  for (int q = q0; q < q1; ++q) s += A[(c0 + q) * lda + i] * v[q];
  part[blockIdx.y * ldp + (i - r0)] = s;
}
__global__ void k_right_sum(const double* __restrict__ part, long long ldp, int nch, int R, const double* __restrict__ scal,
                            double* __restrict__ u) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= R) return;
  double s = 0.0;
  for (int c = 0; c < nch; ++c) s += part[c * ldp + i];
  u[i] = s * scal[0];
}
__global__ void k_right_update(double* __restrict__ A, long long lda, int r0, int r1, int c0, int L,
                               const double* __restrict__ v, const double* __restrict__ u, const double* __restrict__ scal) {
  if (scal[0] == 0.0) return;
  const int i = r0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r1) return;
  const int q0 = blockIdx.y * kRC, q1 = min(L, q0 + kRC);
  const double ui = u[i - r0];
  for (int q = q0; q < q1; ++q) A[(c0 + q) * lda + i] -= ui * v[q];
}

// ---- Francis double-shift QR on an upper Hessenberg matrix, eigenvalues only (EISPACK hqr).
// One CTA. Lane 0 of warp 0 owns the 4×3 corner block of each bulge-chasing step (row and
// column modifications inside it, then the next step's reflector); warps 1.. own the remaining
// row-modification columns (j ≥ k+3, by column) and column-modification rows (i < k, by row).
// Those sets are disjoint within a step and owner-stable across steps, so one barrier per step
// suffices (the reflector slot is double-buffered by step parity).
constexpr int kQRT = 512, kQU = 4;
struct Refl {
  double X, Y, Z, Q, R;
  int on;
};

__device__ __forceinline__ int block_max_i(int v, int* shi) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) shi[threadIdx.x >> 5] = v;
  __syncthreads();
  int r = shi[0];
  for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) r = max(r, shi[w]);
  __syncthreads();
  return r;
}

// p, q, r at row m for shifts (x, y, w), normalised by |p|+|q|+|r| (hqr's m-loop body)
__device__ __forceinline__ void hqr_pqr(const double* A, long long n, int m, double x, double y, double w, double& p,
                                        double& q, double& r, double& zz) {
#define AA(i, j) A[(i) + static_cast<long long>(j) * n]
  zz = AA(m, m);
  const double rr = x - zz, ss = y - zz;
  p = (rr * ss - w) / AA(m + 1, m) + AA(m, m + 1);
  q = AA(m + 1, m + 1) - zz - rr - ss;
  r = AA(m + 2, m + 1);
  const double s = fabs(p) + fabs(q) + fabs(r);
  p /= s;
  q /= s;
  r /= s;
#undef AA
}

__device__ __forceinline__ bool make_refl(double p, double q, double r, Refl& o, double& s) {
  s = copysign(sqrt(p * p + q * q + r * r), p);
  if (s == 0.0) {
    o.on = 0;
    return false;
  }
  p += s;
  const double is = 1.0 / s, ip = 1.0 / p;
  o.X = p * is;
  o.Y = q * is;
  o.Z = r * is;
  o.Q = q * ip;
  o.R = r * ip;
  o.on = 1;
  return true;
}

__global__ void __launch_bounds__(kQRT) k_hqr(double* __restrict__ Ag, long long ldg, int n, double* __restrict__ wr,
                                              double* __restrict__ wi, int* __restrict__ status, int max_its,
                                              int use_smem) {
  // use_smem: the block is copied to shared memory first (small blocks; Ag is left untouched)
  extern __shared__ double hsm[];
  double* A = Ag;
  long long ld = ldg;
  if (use_smem) {
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) hsm[e] = Ag[(e % n) + (e / n) * ldg];
    __syncthreads();
    A = hsm;
    ld = n;
  }
#define AA(i, j) A[(i) + static_cast<long long>(j) * ld]
  __shared__ double sh[32];
  __shared__ int shi[32];
  __shared__ Refl slot[2];
  const int tid = threadIdx.x;
  const int ws0 = blockDim.x > 32 ? 32 : 1;  // workers: warps 1.. (or lanes 1.. of a one-warp CTA)
  const int nw = blockDim.x - ws0, wid = tid - ws0;
  // anorm = Σ |a_ij| over the Hessenberg part
  double s0 = 0.0;
  for (long long e = tid; e < static_cast<long long>(n) * n; e += blockDim.x) {
    const int i = static_cast<int>(e % n), j = static_cast<int>(e / n);
    if (i <= j + 1) s0 += fabs(AA(i, j));
  }
  const double anorm = block_sum_d(s0, sh);
  int nn = n - 1;
  double t = 0.0;
  while (nn >= 0) {
    int its = 0;
    for (;;) {
      // largest l in [1, nn] with a negligible subdiagonal a(l, l-1); 0 if none
      int lc = 0;
      for (int l = 1 + tid; l <= nn; l += blockDim.x) {
        double s = fabs(AA(l - 1, l - 1)) + fabs(AA(l, l));
        if (s == 0.0) s = anorm;
        if (fabs(AA(l, l - 1)) + s == s) lc = max(lc, l);
      }
      const int l = block_max_i(lc, shi);
      if (l >= 1 && tid == 0) AA(l, l - 1) = 0.0;
      __syncthreads();
      double x = AA(nn, nn);
      if (l == nn) {  // one root
        if (tid == 0) {
          wr[nn] = x + t;
          wi[nn] = 0.0;
        }
        --nn;
        break;
      }
      double y = AA(nn - 1, nn - 1), w = AA(nn, nn - 1) * AA(nn - 1, nn);
      if (l == nn - 1) {  // two roots
        if (tid == 0) {
          const double p = 0.5 * (y - x), q = p * p + w, z = sqrt(fabs(q));
          x += t;
          if (q >= 0.0) {
            const double zz = p + copysign(z, p);
            wr[nn - 1] = wr[nn] = x + zz;
            if (zz != 0.0) wr[nn] = x - w / zz;
            wi[nn - 1] = wi[nn] = 0.0;
          } else {
            wr[nn - 1] = wr[nn] = x + p;
            wi[nn - 1] = -z;
            wi[nn] = z;
          }
        }
        nn -= 2;
        break;
      }
      if (its == max_its) {
        if (tid == 0) status[0] = 1;
        return;
      }
      if (its > 0 && its % 10 == 0) {  // exceptional shift
        t += x;
        for (int i = tid; i <= nn; i += blockDim.x) AA(i, i) -= x;
        __syncthreads();
        const double s = fabs(AA(nn, nn - 1)) + fabs(AA(nn - 1, nn - 2));
        y = x = 0.75 * s;
        w = -0.4375 * s * s;
      }
      ++its;
      // m: largest in [l+1, nn-2] where two consecutive small subdiagonals allow the bulge to start
      int mc = l;
      for (int m = l + 1 + tid; m <= nn - 2; m += blockDim.x) {
        double p, q, r, z;
        hqr_pqr(A, ld, m, x, y, w, p, q, r, z);
        const double u = fabs(AA(m, m - 1)) * (fabs(q) + fabs(r));
        const double v = fabs(p) * (fabs(AA(m - 1, m - 1)) + fabs(z) + fabs(AA(m + 1, m + 1)));
        if (u + v == v) mc = max(mc, m);
      }
      const int m = block_max_i(mc, shi);
      for (int i = m + 2 + tid; i <= nn; i += blockDim.x) {
        AA(i, i - 2) = 0.0;
        if (i != m + 2) AA(i, i - 3) = 0.0;
      }
      if (tid == 0) {
        double p, q, r, z, s;
        hqr_pqr(A, ld, m, x, y, w, p, q, r, z);
        if (make_refl(p, q, r, slot[m & 1], s) && l != m) AA(m, m - 1) = -AA(m, m - 1);
      }
      __syncthreads();
      for (int k = m; k <= nn - 1; ++k) {
        const Refl R = slot[k & 1];
        const bool three = k + 1 != nn;
        if (tid == 0) {
          // corner block B[r][c] = a(k+r, k+c), rows k..min(nn,k+3), cols k..min(nn,k+2)
          double B[4][3];
          const int rmax = min(nn, k + 3) - k, cmax = min(nn, k + 2) - k;
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) B[r][c] = (r <= rmax && c <= cmax) ? AA(k + r, k + c) : 0.0;
          if (R.on) {
#pragma unroll
            for (int c = 0; c < 3; ++c)
              if (c <= cmax) {  // row modification, columns k..k+2
                double p = B[0][c] + R.Q * B[1][c];
                if (three) {
                  p += R.R * B[2][c];
                  B[2][c] -= p * R.Z;
                }
                B[1][c] -= p * R.Y;
                B[0][c] -= p * R.X;
              }
#pragma unroll
            for (int r = 0; r < 4; ++r)
              if (r <= rmax) {  // column modification, rows k..min(nn, k+3)
                double p = R.X * B[r][0] + R.Y * B[r][1];
                if (three) {
                  p += R.Z * B[r][2];
                  B[r][2] -= p * R.R;
                }
                B[r][1] -= p * R.Q;
                B[r][0] -= p;
              }
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
              for (int c = 0; c < 3; ++c)
                if (r <= rmax && c <= cmax) AA(k + r, k + c) = B[r][c];
          }
          if (k + 1 <= nn - 1) {  // next step's reflector from a(k+1..k+3, k)
            double p = B[1][0], q = B[2][0], r = (k + 2 != nn) ? B[3][0] : 0.0;
            const double xs = fabs(p) + fabs(q) + fabs(r);
            Refl& o = slot[(k + 1) & 1];
            if (xs != 0.0) {
              p /= xs;
              q /= xs;
              r /= xs;
              double s;
              if (make_refl(p, q, r, o, s)) AA(k + 1, k) = -s * xs;
            } else {
              o.on = 0;
            }
          }
        } else if (tid >= ws0 && R.on) {
          // loads of kQU owned columns/rows are issued before any store (the stores may alias)
          for (int j0 = k + 3 + wid; j0 <= nn; j0 += kQU * nw) {  // row modification, columns k+3..nn
            double a0[kQU], a1[kQU], a2[kQU];
#pragma unroll
            for (int u = 0; u < kQU; ++u) {
              const int j = j0 + u * nw;
              if (j <= nn) {
                a0[u] = AA(k, j);
                a1[u] = AA(k + 1, j);
                a2[u] = three ? AA(k + 2, j) : 0.0;
              }
            }
#pragma unroll
            for (int u = 0; u < kQU; ++u) {
              const int j = j0 + u * nw;
              if (j <= nn) {
                double p = a0[u] + R.Q * a1[u];
                if (three) {
                  p += R.R * a2[u];
                  AA(k + 2, j) = a2[u] - p * R.Z;
                }
                AA(k + 1, j) = a1[u] - p * R.Y;
                AA(k, j) = a0[u] - p * R.X;
              }
            }
          }
          for (int i0 = l + wid; i0 < k; i0 += kQU * nw) {  // column modification, rows l..k-1
            double b0[kQU], b1[kQU], b2[kQU];
#pragma unroll
            for (int u = 0; u < kQU; ++u) {
              const int i = i0 + u * nw;
              if (i < k) {
                b0[u] = AA(i, k);
                b1[u] = AA(i, k + 1);
                b2[u] = three ? AA(i, k + 2) : 0.0;
              }
            }
#pragma unroll
            for (int u = 0; u < kQU; ++u) {
              const int i = i0 + u * nw;
              if (i < k) {
                double p = R.X * b0[u] + R.Y * b1[u];
                if (three) {
                  p += R.Z * b2[u];
                  AA(i, k + 2) = b2[u] - p * R.R;
                }
                AA(i, k + 1) = b1[u] - p * R.Q;
                AA(i, k) = b0[u] - p;
              }
            }
          }
        }
        __syncthreads();
      }
    }
  }
#undef AA
}

// ---- windowed multi-bulge sweeps (small-bulge multishift QR) for large active blocks.
// nb bulges, each carrying a shift pair from the trailing 2·nb×2·nb block's eigenvalues, are
// introduced at the top of the active block [l, nn] three rows apart and chased to the bottom.
// Steps of different bulges act on disjoint index triples, so at each "time" t every active
// bulge moves one position (reflectors, then all row modifications, then all column
// modifications). The chase runs in a kw×kw diagonal window held in shared memory; the window's
// orthogonal transform U (product of the step reflectors) is applied afterwards to the rows to
// its right (Uᵀ·panel) and the columns above it (panel·U) by separate multi-CTA kernels.
constexpr int kMsKW = 112, kMsT = 512, kMsNB = 16;

__global__ void k_hess_norm(const double* __restrict__ A, int n, double* __restrict__ out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (long long e = threadIdx.x; e < static_cast<long long>(n) * n; e += blockDim.x) {
    const int i = static_cast<int>(e % n), j = static_cast<int>(e / n);
    if (i <= j + 1) s += fabs(A[e]);
  }
  s = block_sum_d(s, sh);
  if (threadIdx.x == 0) out[0] = s;
}

// bottom deflation (hqr's l-scan, one and two roots) until the active block is at least 3 wide;
// ctl = {nn, l} in and out
__global__ void __launch_bounds__(256) k_deflate(double* __restrict__ A, int n, const double* __restrict__ anorm_p,
                                                 int* __restrict__ ctl, double* __restrict__ wr, double* __restrict__ wi) {
#define AA(i, j) A[(i) + static_cast<long long>(j) * n]
  __shared__ int shi[32];
  const double anorm = anorm_p[0];
  int nn = ctl[0], l = 0;
  while (nn >= 0) {
    int lc = 0;
    for (int q = 1 + threadIdx.x; q <= nn; q += blockDim.x) {
      double s = fabs(AA(q - 1, q - 1)) + fabs(AA(q, q));
      if (s == 0.0) s = anorm;
      if (fabs(AA(q, q - 1)) + s == s) lc = max(lc, q);
    }
    l = block_max_i(lc, shi);
    if (l >= 1 && threadIdx.x == 0) AA(l, l - 1) = 0.0;
    __syncthreads();
    if (l == nn) {
      if (threadIdx.x == 0) {
        wr[nn] = AA(nn, nn);
        wi[nn] = 0.0;
      }
      --nn;
    } else if (l == nn - 1) {
      if (threadIdx.x == 0) {
        double x = AA(nn, nn);
        const double y = AA(nn - 1, nn - 1), w = AA(nn, nn - 1) * AA(nn - 1, nn);
        const double p = 0.5 * (y - x), q = p * p + w, z = sqrt(fabs(q));
        if (q >= 0.0) {
          const double zz = p + copysign(z, p);
          wr[nn - 1] = wr[nn] = x + zz;
          if (zz != 0.0) wr[nn] = x - w / zz;
          wi[nn - 1] = wi[nn] = 0.0;
        } else {
          wr[nn - 1] = wr[nn] = x + p;
          wi[nn - 1] = -z;
          wi[nn] = z;
        }
      }
      nn -= 2;
    } else {
      break;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    ctl[0] = nn;
    ctl[1] = nn >= 0 ? l : 0;
  }
#undef AA
}

// shift pairs (sum, product) from the ns eigenvalues of the trailing block: complex conjugate
// pairs as they come, real shifts paired in order; exceptional sweeps spread ad hoc real shifts
__global__ void k_ms_shifts(const double* __restrict__ sr, const double* __restrict__ si, int ns,
                            const double* __restrict__ A, int n, int nn, int exceptional, double* __restrict__ td) {
  if (threadIdx.x != 0) return;
  int b = 0;
  double pend = 0.0;
  bool have = false;
  if (exceptional) {
    const double s = fabs(A[nn + static_cast<long long>(nn - 1) * n]) + fabs(A[(nn - 1) + static_cast<long long>(nn - 2) * n]);
    const double h = A[nn + static_cast<long long>(nn) * n];
    for (int q = 0; q < ns / 2; ++q) {
      const double x = h + 0.75 * s * (1.0 + q / static_cast<double>(ns)), y = h - 0.4375 * s * (1.0 + q / static_cast<double>(ns));
      td[2 * q] = x + y;
      td[2 * q + 1] = x * y;
    }
    return;
  }
  for (int i = 0; i < ns && b < ns / 2; ++i) {
    if (si[i] != 0.0 && i + 1 < ns) {
      td[2 * b] = sr[i] + sr[i + 1];
      td[2 * b + 1] = sr[i] * sr[i] + si[i] * si[i];
      ++b;
      ++i;
    } else if (have) {
      td[2 * b] = pend + sr[i];
      td[2 * b + 1] = pend * sr[i];
      ++b;
      have = false;
    } else {
      pend = sr[i];
      have = true;
    }
  }
  for (; b < ns / 2; ++b) {  // odd leftovers: double real shift
    td[2 * b] = 2.0 * pend;
    td[2 * b + 1] = pend * pend;
  }
}

// one window of a multi-bulge sweep: times [tA, tB), diagonal block [w0, w1) in shared memory
__global__ void __launch_bounds__(kMsT) k_ms_window(double* __restrict__ A, int n, int l, int nn, int nb, int w0,
                                                    int w1, int tA, int tB, const double* __restrict__ td,
                                                    double* __restrict__ Ug) {
  extern __shared__ double sm[];
  const int kw = w1 - w0, ls = kw + 1;  // padded leading dimension: conflict-free row sweeps
  double* Hs = sm;            // kw × kw, column-major
  double* Us = sm + kw * ls;  // kw × kw
  __shared__ Refl rf[kMsNB];
  __shared__ int rk[kMsNB];
  const int tid = threadIdx.x;
  for (int e = tid; e < kw * kw; e += blockDim.x) {
    const int i = e % kw, j = e / kw;
    Hs[i + j * ls] = A[(w0 + i) + static_cast<long long>(w0 + j) * n];
    Us[i + j * ls] = i == j ? 1.0 : 0.0;
  }
  __syncthreads();
#define HS(i, j) Hs[((i) - w0) + ((j) - w0) * ls]
  for (int t = tA; t < tB; ++t) {
    // phase 1: reflectors of the active bulges
    if (tid < nb) {
      const int b = tid, k = l + t - 3 * b;
      Refl& o = rf[b];
      o.on = 0;
      rk[b] = -1;
      if (k >= l && k <= nn - 1) {
        rk[b] = k;
        const bool three = k + 1 != nn;
        double p, q, r, s;
        if (k == l) {  // first column of (H − s1)(H − s2) at rows l..l+2
          const double tt = td[2 * b], dd = td[2 * b + 1];
          const double h00 = HS(l, l), h10 = HS(l + 1, l), h01 = HS(l, l + 1), h11 = HS(l + 1, l + 1);
          const double h21 = three ? HS(l + 2, l + 1) : 0.0;
          p = h00 * (h00 - tt) + h01 * h10 + dd;
          q = h10 * (h00 + h11 - tt);
          r = h10 * h21;
          const double x = fabs(p) + fabs(q) + fabs(r);
          if (x != 0.0) {
            const double ix = 1.0 / x;
            p *= ix;
            q *= ix;
            r *= ix;
            make_refl(p, q, r, o, s);
          }
        } else {
          p = HS(k, k - 1);
          q = HS(k + 1, k - 1);
          r = three ? HS(k + 2, k - 1) : 0.0;
          const double x = fabs(p) + fabs(q) + fabs(r);
          if (x != 0.0) {
            const double ix = 1.0 / x;
            p *= ix;
            q *= ix;
            r *= ix;
            if (make_refl(p, q, r, o, s)) {
              HS(k, k - 1) = -s * x;
              HS(k + 1, k - 1) = 0.0;
              if (three) HS(k + 2, k - 1) = 0.0;
            }
          }
        }
      }
    }
    __syncthreads();
    // phase 2: row modifications (rows k..k+2, window columns k..w1-1), all bulges at once
    for (int e = tid; e < nb * kw; e += blockDim.x) {
      const int b = e / kw, j = w0 + e % kw, k = rk[b];
      if (k < 0 || j < k || !rf[b].on) continue;
      const Refl& R = rf[b];
      const bool three = k + 1 != nn;
      const double a0 = HS(k, j), a1 = HS(k + 1, j);
      double p = a0 + R.Q * a1;
      if (three) {
        const double a2 = HS(k + 2, j);
        p += R.R * a2;
        HS(k + 2, j) = a2 - p * R.Z;
      }
      HS(k + 1, j) = a1 - p * R.Y;
      HS(k, j) = a0 - p * R.X;
    }
    __syncthreads();
    // phase 3: column modifications (window rows w0..min(nn, k+3)) and U ← U·P, all bulges
    for (int e = tid; e < nb * 2 * kw; e += blockDim.x) {
      const int b = e / (2 * kw), q = e % (2 * kw), k = rk[b];
      if (k < 0 || !rf[b].on) continue;
      double* c0;
      if (q < kw) {
        if (w0 + q > min(nn, k + 3)) continue;
        c0 = &HS(w0 + q, k);
      } else {
        c0 = Us + (q - kw) + (k - w0) * ls;
      }
      const Refl& R = rf[b];
      const bool three = k + 1 != nn;
      const double b0 = c0[0], b1 = c0[ls];
      double p = R.X * b0 + R.Y * b1;
      if (three) {
        const double b2 = c0[2 * ls];
        p += R.Z * b2;
        c0[2 * ls] = b2 - p * R.R;
      }
      c0[ls] = b1 - p * R.Q;
      c0[0] = b0 - p;
    }
    __syncthreads();
  }
#undef HS
  for (int e = tid; e < kw * kw; e += blockDim.x) {
    const int i = e % kw, j = e / kw;
    A[(w0 + i) + static_cast<long long>(w0 + j) * n] = Hs[i + j * ls];
    Ug[e] = Us[i + j * ls];
  }
}

// H[w0:w1, c0:c1] ← Uᵀ·H[w0:w1, c0:c1]: CTA per 16-column chunk, in place
__global__ void __launch_bounds__(256) k_ms_right(double* __restrict__ A, int n, int w0, int kw, int c0, int c1,
                                                  const double* __restrict__ U) {
  extern __shared__ double sm[];
  const int ls = kw + 1;
  double* Us = sm;             // kw × kw, padded
  double* P = sm + kw * ls;    // kw × 16
  const int j0 = c0 + blockIdx.x * 16, nc = min(16, c1 - j0);
  for (int e = threadIdx.x; e < kw * kw; e += blockDim.x) Us[(e % kw) + (e / kw) * ls] = U[e];
  for (int e = threadIdx.x; e < kw * nc; e += blockDim.x) P[e] = A[(w0 + e % kw) + static_cast<long long>(j0 + e / kw) * n];
  __syncthreads();
  for (int e = threadIdx.x; e < kw * nc; e += blockDim.x) {
    const int i = e % kw, c = e / kw;
    const double* u = Us + i * ls;  // column i of U
    const double* pc = P + c * kw;
    double s = 0.0;
    for (int r = 0; r < kw; ++r) s += u[r] * pc[r];
    A[(w0 + i) + static_cast<long long>(j0 + c) * n] = s;
  }
}

// H[r0:r1, w0:w1] ← H[r0:r1, w0:w1]·U: CTA per 32-row chunk, in place
__global__ void __launch_bounds__(256) k_ms_top(double* __restrict__ A, int n, int w0, int kw, int r0, int r1,
                                                const double* __restrict__ U) {
  extern __shared__ double sm[];
  double* Us = sm;             // kw × kw
  double* P = sm + kw * kw;    // 32 × kw (row chunk, column-major, ld 32)
  const int i0 = r0 + blockIdx.x * 32, nr = min(32, r1 - i0);
  for (int e = threadIdx.x; e < kw * kw; e += blockDim.x) Us[e] = U[e];
  for (int e = threadIdx.x; e < 32 * kw; e += blockDim.x) {
    const int i = e % 32, j = e / 32;
    P[e] = i < nr ? A[(i0 + i) + static_cast<long long>(w0 + j) * n] : 0.0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 32 * kw; e += blockDim.x) {
    const int i = e % 32, j = e / 32;
    if (i >= nr) continue;
    const double* u = Us + j * kw;  // column j of U
    double s = 0.0;
    for (int r = 0; r < kw; ++r) s += P[i + r * 32] * u[r];
    A[(i0 + i) + static_cast<long long>(w0 + j) * n] = s;
  }
}

// eigenvalues of the symmetric tridiagonal (a, b) by Sturm-count bisection; thread per index.
// k-th smallest (0-based) for k in [k0, k0 + cnt); out[k - k0]
__device__ __forceinline__ int sturm_count(const double* a, const double* b2, int N, double x, double pivmin) {
  int cnt = 0;
  double q = a[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += q < 0.0;
  for (int i = 1; i < N; ++i) {
    q = a[i] - x - b2[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
}
__global__ void k_bisect(const double* __restrict__ a, const double* __restrict__ b2, int N, double gl, double gu,
                         double pivmin, int k0, int cnt, int descending, double* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt) return;
  const int k = k0 + t;  // k-th smallest
  double lo = gl, hi = gu;
  for (int it = 0; it < 1200; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (sturm_count(a, b2, N, mid, pivmin) <= k) lo = mid;
    else hi = mid;
  }
  out[descending ? cnt - 1 - t : t] = 0.5 * (lo + hi);
}

// diagonal / subdiagonal (or superdiagonal) of a reduced matrix
__global__ void k_band(const double* __restrict__ A, long long lda, int n, int upper, double* __restrict__ d,
                       double* __restrict__ e) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  d[i] = A[i + i * lda];
  if (i + 1 < n) e[i] = upper ? A[i + (i + 1) * lda] : A[(i + 1) + i * lda];
}

// normal blocks H_j1ᵀH_j2 (j1 ≤ j2) -> dense symmetric p×p (assembly.hpp:206-215 densify of the map)
__global__ void k_densify_nb(const double* __restrict__ NB, const long long* __restrict__ off, const int* __restrict__ j1s,
                             const int* __restrict__ j2s, const int* __restrict__ col_off, int p, double* __restrict__ D) {
  const int k = blockIdx.y;
  const int j1 = j1s[k], j2 = j2s[k];
  const int a0 = col_off[j1], p1 = col_off[j1 + 1] - a0, b0 = col_off[j2], p2 = col_off[j2 + 1] - b0;
  const double* blk = NB + off[k];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < p1 * p2; e += gridDim.x * blockDim.x) {
    const int r = e % p1, c = e / p1;
    const double v = blk[e];
    D[(a0 + r) + static_cast<long long>(b0 + c) * p] = v;
    if (j1 != j2) D[(b0 + c) + static_cast<long long>(a0 + r) * p] = v;
  }
}

}  // namespace

// Householder reflector helpers over a column-major matrix
static void house(Ctx& c, double* x, long long inc, int L, double* v, double* scal) {
  k_house<<<1, kHT, 0, c.stream>>>(x, inc, L, v, scal);
  RDD_LAUNCH_CHECK();
}
static void left_apply(Ctx& c, double* A, long long lda, int r0, int L, int c0, int c1, const double* v,
                       const double* scal) {
  if (c1 <= c0 || L <= 0) return;
  k_left_apply<<<ceil_div(c1 - c0, 8), 256, 0, c.stream>>>(A, lda, r0, L, c0, c1, v, scal);
  RDD_LAUNCH_CHECK();
}
static void right_apply(Ctx& c, double* A, long long lda, int r0, int r1, int c0, int L, const double* v,
                        const double* scal, double* part, double* u) {
  if (r1 <= r0 || L <= 0) return;
  const int R = r1 - r0, nch = ceil_div(L, kRC);
  const dim3 g(ceil_div(R, 128), nch);
  k_right_part<<<g, 128, 0, c.stream>>>(A, lda, r0, r1, c0, L, v, part, R);
  RDD_LAUNCH_CHECK();
  k_right_sum<<<ceil_div(R, 256), 256, 0, c.stream>>>(part, R, nch, R, scal, u);
  RDD_LAUNCH_CHECK();
  k_right_update<<<g, 128, 0, c.stream>>>(A, lda, r0, r1, c0, L, v, u, scal);
  RDD_LAUNCH_CHECK();
}

// A (n×n, column-major, device) -> upper Hessenberg in place (orthogonal similarity)
static void hessenberg(Ctx& c, double* A, int n) {
  double* v = c.ws("dg_v", n);
  double* scal = c.ws("dg_scal", 2);
  double* part = c.ws("dg_part", static_cast<size_t>(ceil_div(n, kRC)) * n);
  double* u = c.ws("dg_u", n);
  for (int k = 0; k + 2 < n; ++k) {
    const int L = n - k - 1;
    house(c, A + (k + 1) + static_cast<long long>(k) * n, 1, L, v, scal);
    left_apply(c, A, n, k + 1, L, k + 1, n, v, scal);
    right_apply(c, A, n, 0, n, k + 1, L, v, scal, part, u);
  }
}

// A (m×n, m ≥ n, column-major, device) -> upper bidiagonal in place (d on the diagonal, e above)
static void bidiagonalize(Ctx& c, double* A, int m, int n) {
  double* v = c.ws("dg_v", std::max(m, n));
  double* scal = c.ws("dg_scal", 2);
  double* part = c.ws("dg_part", static_cast<size_t>(ceil_div(n, kRC)) * m);
  double* u = c.ws("dg_u", m);
  for (int k = 0; k < n; ++k) {
    house(c, A + k + static_cast<long long>(k) * m, 1, m - k, v, scal);
    left_apply(c, A, m, k, m - k, k + 1, n, v, scal);
    if (k + 2 < n) {
      house(c, A + k + static_cast<long long>(k + 1) * m, m, n - k - 1, v, scal);
      right_apply(c, A, m, k + 1, m, k + 1, n - k - 1, v, scal, part, u);
    }
  }
}

// all eigenvalues of the symmetric tridiagonal (d, e): ascending (or descending) into out (device)
static void tridiag_eigs(Ctx& c, const std::vector<double>& d, const std::vector<double>& e, int k0, int cnt,
                         bool descending, double* out_dev) {
  const int N = static_cast<int>(d.size());
  double gl = DBL_MAX, gu = -DBL_MAX, bmax2 = 0.0;
  for (int i = 0; i < N; ++i) {
    const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < N ? fabs(e[i]) : 0.0);
    gl = std::min(gl, d[i] - r);
    gu = std::max(gu, d[i] + r);
    if (i + 1 < N) bmax2 = std::max(bmax2, e[i] * e[i]);
  }
  const double tnorm = std::max(fabs(gl), fabs(gu));
  gl -= 2.0 * DBL_EPSILON * tnorm * N + DBL_MIN;
  gu += 2.0 * DBL_EPSILON * tnorm * N + DBL_MIN;
  const double pivmin = DBL_MIN * std::max(1.0, bmax2);
  std::vector<double> hb(2 * static_cast<size_t>(N));
  for (int i = 0; i < N; ++i) hb[i] = d[i];
  for (int i = 0; i + 1 < N; ++i) hb[N + i] = e[i] * e[i];
  double* dd = c.ws("dg_tri", hb.size());
  RDD_CUDA(cudaMemcpyAsync(dd, hb.data(), sizeof(double) * hb.size(), cudaMemcpyHostToDevice, c.stream));
  k_bisect<<<ceil_div(cnt, 128), 128, 0, c.stream>>>(dd, dd + N, N, gl, gu, pivmin, k0, cnt, descending ? 1 : 0, out_dev);
  RDD_LAUNCH_CHECK();
  RDD_CUDA(cudaStreamSynchronize(c.stream));  // hb must outlive the async copy
}

static void band_host(Ctx& c, const double* A, long long lda, int n, bool upper, std::vector<double>& d,
                      std::vector<double>& e) {
  double* dd = c.ws("dg_band", 2 * static_cast<size_t>(n));
  k_band<<<ceil_div(n, 256), 256, 0, c.stream>>>(A, lda, n, upper ? 1 : 0, dd, dd + n);
  RDD_LAUNCH_CHECK();
  d.resize(n);
  e.resize(n > 0 ? n - 1 : 0);
  RDD_CUDA(cudaMemcpyAsync(d.data(), dd, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
  if (n > 1) RDD_CUDA(cudaMemcpyAsync(e.data(), dd + n, sizeof(double) * (n - 1), cudaMemcpyDeviceToHost, c.stream));
  RDD_CUDA(cudaStreamSynchronize(c.stream));
}

void check_dense_cap(long long n, int cap) {  // krylov.hpp:405-409
  if (n > cap)
    throw std::invalid_argument("matrix of size " + std::to_string(n) + " exceeds the dense diagnostics cap (" +
                                std::to_string(cap) + ")");
}

static void hqr_block(Ctx& c, double* A, long long ld, int nb, double* wr, double* wi, int* st, bool smem) {
  const size_t sm = smem ? sizeof(double) * nb * nb : 0;
  // set on every call: the attribute is per device, and a context may live on any device
  RDD_CUDA(cudaFuncSetAttribute(k_hqr, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sizeof(double) * kMsKW * kMsKW)));
  k_hqr<<<1, smem ? 32 : kQRT, sm, c.stream>>>(A, ld, nb, wr, wi, st, 60, smem ? 1 : 0);
  RDD_LAUNCH_CHECK();
}

// one multi-bulge sweep over the active block [l, nn] with nbul bulges (shift pairs in td)
static void ms_sweep(Ctx& c, double* A, int n, int l, int nn, int nbul, const double* td, double* U) {
  // per call (per device), as hqr_block
  RDD_CUDA(cudaFuncSetAttribute(k_ms_window, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sizeof(double) * 2 * kMsKW * (kMsKW + 1))));
  RDD_CUDA(cudaFuncSetAttribute(k_ms_right, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sizeof(double) * (kMsKW * (kMsKW + 1) + kMsKW * 16))));
  RDD_CUDA(cudaFuncSetAttribute(k_ms_top, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sizeof(double) * (kMsKW * kMsKW + 32 * kMsKW))));
  const int S = 3 * (nbul - 1), T = (nn - l) + S, steps = kMsKW - S - 4;
  for (int tA = 0; tA < T;) {
    const int tB = std::min(T, tA + steps);
    const int w0 = std::max(l, l + tA - S - 1), w1 = std::min(nn + 1, l + tB + 3), kw = w1 - w0;
    k_ms_window<<<1, kMsT, sizeof(double) * 2 * kw * (kw + 1), c.stream>>>(A, n, l, nn, nbul, w0, w1, tA, tB, td, U);
    RDD_LAUNCH_CHECK();
    if (w1 <= nn) {
      k_ms_right<<<ceil_div(nn + 1 - w1, 16), 256, sizeof(double) * (kw * (kw + 1) + kw * 16), c.stream>>>(
          A, n, w0, kw, w1, nn + 1, U);
      RDD_LAUNCH_CHECK();
    }
    if (w0 > l) {
      k_ms_top<<<ceil_div(w0 - l, 32), 256, sizeof(double) * (kw * kw + 32 * kw), c.stream>>>(A, n, w0, kw, l, w0, U);
      RDD_LAUNCH_CHECK();
    }
    tA = tB;
    c.stats["diag_windows"].launches += 1;
  }
}

// eigenvalues of an upper Hessenberg matrix (device, destroyed) into device wr/wi: bottom
// deflation, single-bulge hqr on blocks up to kMsKW (shared memory), multi-bulge windowed sweeps
// on larger active blocks with the trailing block's eigenvalues as shifts
static void hessenberg_eigenvalues(Ctx& c, double* A, int n, double* wr, double* wi, int* st) {
  const int ns = 2 * kMsNB;
  double* anorm = c.ws("dg_anorm", 1);
  double* sw = c.ws("dg_shift", 2 * ns + ns);  // shift eigenvalues, then (sum, product) pairs
  double* U = c.ws("dg_U", kMsKW * kMsKW);
  DBuf<int> ctl;
  ctl.zero(4, c.stream);  // ctl[0..1] = (nn, l); ctl[2] = shift-block status
  k_hess_norm<<<1, 1024, 0, c.stream>>>(A, n, anorm);
  RDD_LAUNCH_CHECK();
  int nn = n - 1, last_nn = n, stall = 0;
  int h[2];
  while (nn >= 0) {
    RDD_CUDA(cudaMemcpyAsync(ctl.p, &nn, sizeof(int), cudaMemcpyHostToDevice, c.stream));
    k_deflate<<<1, 256, 0, c.stream>>>(A, n, anorm, ctl.p, wr, wi);
    RDD_LAUNCH_CHECK();
    RDD_CUDA(cudaMemcpyAsync(h, ctl.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    RDD_CUDA(cudaStreamSynchronize(c.stream));
    nn = h[0];
    const int l = h[1];
    if (nn < 0) break;
    const int size = nn - l + 1;
    stall = nn < last_nn ? 0 : stall + 1;
    last_nn = nn;
    if (size <= kMsKW || stall >= 60) {  // small block (or no progress): single-bulge hqr on the block
      ScopedKernelTimer tb(c, "diag_block");
      hqr_block(c, A + l + static_cast<long long>(l) * n, n, size, wr + l, wi + l, st, size <= kMsKW);
      nn = l - 1;
      last_nn = n;
      continue;
    }
    const long long b0 = static_cast<long long>(nn - ns + 1);
    {
      ScopedKernelTimer ts(c, "diag_shifts");
      hqr_block(c, A + b0 + b0 * n, n, ns, sw, sw + ns, ctl.p + 2, true);
    }
    k_ms_shifts<<<1, 32, 0, c.stream>>>(sw, sw + ns, ns, A, n, nn, stall > 0 && stall % 10 == 0 ? 1 : 0, sw + 2 * ns);
    RDD_LAUNCH_CHECK();
    {
      ScopedKernelTimer tw(c, "diag_sweep");
      ms_sweep(c, A, n, l, nn, kMsNB, sw + 2 * ns, U);
    }
  }
}

// eigenvalues of a general square matrix (device, destroyed); host wr/wi sorted by (real, imag)
void dense_eigenvalues_dev(Ctx& c, double* A, int n, std::vector<double>& wr, std::vector<double>& wi) {
  ScopedKernelTimer tk(c, "diag_eig");
  wr.assign(n, 0.0);
  wi.assign(n, 0.0);
  if (n == 0) return;
  {
    ScopedKernelTimer th(c, "diag_hessenberg");
    hessenberg(c, A, n);
  }
  double* w = c.ws("dg_w", 2 * static_cast<size_t>(n));
  DBuf<int> st;
  st.zero(1, c.stream);
  {
    ScopedKernelTimer tq(c, "diag_qr");
    hessenberg_eigenvalues(c, A, n, w, w + n, st.p);
  }
  int status = 0;
  RDD_CUDA(cudaMemcpyAsync(&status, st.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  RDD_CUDA(cudaMemcpyAsync(wr.data(), w, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
  RDD_CUDA(cudaMemcpyAsync(wi.data(), w + n, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream));
  RDD_CUDA(cudaStreamSynchronize(c.stream));
  if (status) throw std::runtime_error("spectrum: the QR iteration did not converge");
  std::vector<std::complex<double>> z(n);
  for (int i = 0; i < n; ++i) z[i] = {wr[i], wi[i]};
  std::sort(z.begin(), z.end(), [](const std::complex<double>& a, const std::complex<double>& b) {
    return a.real() < b.real() || (a.real() == b.real() && a.imag() < b.imag());
  });
  for (int i = 0; i < n; ++i) {
    wr[i] = z[i].real();
    wi[i] = z[i].imag();
  }
}

// eigenvalues of a symmetric matrix (device, destroyed), ascending
void symmetric_eigenvalues_dev(Ctx& c, double* A, int n, std::vector<double>& ev) {
  ScopedKernelTimer tk(c, "diag_syev");
  ev.assign(n, 0.0);
  if (n == 0) return;
  hessenberg(c, A, n);  // tridiagonal for symmetric input
  std::vector<double> d, e;
  band_host(c, A, n, n, false, d, e);
  double* out = c.ws("dg_out", n);
  tridiag_eigs(c, d, e, 0, n, false, out);
  RDD_CUDA(cudaMemcpy(ev.data(), out, sizeof(double) * n, cudaMemcpyDeviceToHost));
}

// singular values of an m×n matrix (device, column-major, destroyed; m ≥ n), non-increasing
void singular_values_dev(Ctx& c, double* A, int m, int n, std::vector<double>& sv) {
  ScopedKernelTimer tk(c, "diag_svd");
  sv.assign(n, 0.0);
  if (n == 0) return;
  bidiagonalize(c, A, m, n);
  std::vector<double> d, e;
  band_host(c, A, m, n, true, d, e);
  // Golub–Kahan tridiagonal: zero diagonal, off-diagonal d1, e1, d2, e2, ..., dn; eigenvalues ±σ
  std::vector<double> gd(2 * static_cast<size_t>(n), 0.0), ge(2 * static_cast<size_t>(n) - 1, 0.0);
  for (int i = 0; i < n; ++i) {
    ge[2 * i] = d[i];
    if (i + 1 < n) ge[2 * i + 1] = e[i];
  }
  double* out = c.ws("dg_out", n);
  tridiag_eigs(c, gd, ge, n, n, true, out);  // the n largest, descending
  RDD_CUDA(cudaMemcpy(sv.data(), out, sizeof(double) * n, cudaMemcpyDeviceToHost));
  for (double& s : sv) s = std::max(s, 0.0);
}

double condition_from(const std::vector<double>& sv) {  // krylov.hpp:430-440
  double smin = 0.0;
  for (int i = static_cast<int>(sv.size()) - 1; i >= 0; --i)
    if (sv[i] > 0.0) {
      smin = sv[i];
      break;
    }
  if (smin == 0.0) throw std::domain_error("condition number undefined: all singular values are zero");
  return sv[0] / smin;
}

// dense HᵀH from the normal blocks (device, p×p)
void densify_normal(Ctx& c, double* D) {
  RDD_CUDA(cudaMemsetAsync(D, 0, sizeof(double) * c.p * c.p, c.stream));
  const int npair = static_cast<int>(c.nb_j1.size());
  if (npair == 0) return;
  DBuf<long long> off;
  DBuf<int> j1, j2;
  off.upload(c.nb_off.data(), npair, c.stream);
  j1.upload(c.nb_j1.data(), npair, c.stream);
  j2.upload(c.nb_j2.data(), npair, c.stream);
  k_densify_nb<<<dim3(8, npair), 256, 0, c.stream>>>(c.NB.p, off.p, j1.p, j2.p, c.dcol_off.p, c.p, D);
  RDD_LAUNCH_CHECK();
  RDD_CUDA(cudaStreamSynchronize(c.stream));
}

// runner.hpp:344-362 spectrum_cmd / :381-393 sweep_tau diagnostics on the assembled system
void spectra(Ctx& c, int cap, std::vector<double>& nre, std::vector<double>& nim, std::vector<double>* pre,
             std::vector<double>* pim, double* cond_n, double* cond_p) {
  const int n = c.p;
  check_dense_cap(n, cap);
  if (!c.NB.p || c.nb_j1.empty()) build_normal_blocks(c);
  const size_t nn = static_cast<size_t>(n) * n;
  double* A = c.ws("dg_A", nn);
  double* W = c.ws("dg_W", nn);
  densify_normal(c, A);
  // spectrum(AtA): symmetric input -> real eigenvalues (imag 0), ascending
  RDD_CUDA(cudaMemcpyAsync(W, A, sizeof(double) * nn, cudaMemcpyDeviceToDevice, c.stream));
  symmetric_eigenvalues_dev(c, W, n, nre);
  nim.assign(n, 0.0);
  if (cond_n) {
    RDD_CUDA(cudaMemcpyAsync(W, A, sizeof(double) * nn, cudaMemcpyDeviceToDevice, c.stream));
    std::vector<double> sv;
    singular_values_dev(c, W, n, n, sv);
    *cond_n = condition_from(sv);
  }
  if (c.pkind < 0 || !(pre || cond_p)) return;
  // MA = M⁻¹·AtA column by column (runner.hpp:358-360)
  double* MA = c.ws("dg_MA", nn);
  for (int col = 0; col < n; ++col) precond_apply_dev(c, A + static_cast<size_t>(col) * n, MA + static_cast<size_t>(col) * n, false);
  if (cond_p) {
    RDD_CUDA(cudaMemcpyAsync(W, MA, sizeof(double) * nn, cudaMemcpyDeviceToDevice, c.stream));
    std::vector<double> sv;
    singular_values_dev(c, W, n, n, sv);
    *cond_p = condition_from(sv);
  }
  if (pre) {
    std::vector<double> im;
    dense_eigenvalues_dev(c, MA, n, *pre, im);
    if (pim) *pim = im;
  }
}

}  // namespace rdd
