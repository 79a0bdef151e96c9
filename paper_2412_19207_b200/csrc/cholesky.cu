// cholesky.cu — K8: batched blocked Cholesky of the Schwarz local matrices A_i = (HᵀH)[S_i, S_i]
// (schwarz.hpp:112-130) and the per-iteration batched triangular solves that apply A_i⁻¹.
//
// The reference pseudo-inverts A_i through a full eigendecomposition (schwarz.hpp:131-146,
// ~9n³ flops) and applies V diag(1/λ) Vᵀ. When every eigenvalue is above the reference's cutoff
// (1e-12·λmax) that pseudo-inverse *is* A_i⁻¹, so the device factors A = LLᵀ once (n³/3 flops:
// right-looking, 64-wide panels, diagonal POTRF and panel TRSM in shared memory, trailing updates
// on DMMA) and applies A⁻¹ as a forward and a backward triangular solve per Krylov step — the
// same n² bytes per apply as a dense inverse, a third of its build flops, half its memory.
// L is stored tile-packed (64x64 column-major tiles (k, j<=k), block row after block row) with the
// diagonal tiles replaced by L_kk⁻¹, so both solves are chains of tile GEMVs. Matrices of different
// sizes are processed together; each factor step launches only the work of the matrices still
// active. A failed pivot flags the matrix for the eigen fallback (schwarz.cu).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "ctx.hpp"

namespace rdd {

namespace {

constexpr int NB = 64;
constexpr int kPairSmem = 2 * NB * (NB + 1) * sizeof(double);
constexpr int kSolveWarps = 8;

struct Mat {
  long long off;  // element offset of the matrix
  int n;          // order (= leading dimension)
};

// Layout of a packed explicit inverse (small-block mode): lower 64 x 64 tiles (k, j <= k), block row
// after block row, column-major; the tiles of the LAST block row keep only ld = inv_last_ld(n) rows
// (the n - 64(nb-1) valid ones rounded up to 8), so the zero padding below row n is not stored
// (n = 487: 40 of 64 rows, 8% of the bytes; n = 525: 16 of 64, 15%).
__host__ __device__ inline int inv_last_ld(int n) {
  const int bs = n - ((n + NB - 1) / NB - 1) * NB;
  return (bs + 7) & ~7;
}
__host__ __device__ inline int inv_tile_ld(int n, int k) { return k == (n + NB - 1) / NB - 1 ? inv_last_ld(n) : NB; }
__host__ __device__ inline long long inv_tile_off(int n, int k, int j) {  // in doubles
  return static_cast<long long>(k) * (k + 1) / 2 * (NB * NB) + static_cast<long long>(j) * NB * inv_tile_ld(n, k);
}

// A[k-block, k-block] <- chol (lower); pads beyond n act as identity. Also D_k = L_kk⁻¹ (lower,
// padding identity) into the per-matrix diagonal-inverse workspace: the panel solve becomes a DMMA
// product with D_kᵀ and the packed factor stores D_k.
__global__ void k_potrf_diag(double* __restrict__ A, const Mat* __restrict__ mats, const int* __restrict__ act, int k,
                             int* __restrict__ fail, double* __restrict__ Dinv, const long long* __restrict__ doff) {
  extern __shared__ double dsm[];
  double(*s)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm);
  double(*X)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm + NB * (NB + 1));
  const int q = act[blockIdx.x];
  const Mat M = mats[q];
  const int k0 = k * NB, bs = min(NB, M.n - k0);
  double* a = A + M.off + k0 + static_cast<long long>(k0) * M.n;
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e % NB, c = e / NB;
    s[r][c] = (r < bs && c < bs) ? a[r + static_cast<long long>(c) * M.n] : (r == c ? 1.0 : 0.0);
  }
  __syncthreads();
  // Right-looking elimination with the tile in registers: thread (ty, tx) of the 16 x 16 grid owns
  // the entries (ty + 16 i, tx + 16 j) (cyclic, so the shrinking active window stays spread over all
  // threads). Per column: its owners publish the raw column, 64 threads scale it (one sqrt, one
  // division each), everyone updates its own 16 entries — two barriers and no shared-memory
  // read-modify-write. Every entry sees the same operations in the same order as the textbook
  // loop (l = a / sqrt(a_cc); a_rq <- fma(-l_r, l_q, a_rq), c ascending).
  __shared__ double col[NB], lbuf[NB];
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  double t[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) t[i][j] = s[ty + 16 * i][tx + 16 * j];
#pragma unroll
  for (int jc = 0; jc < 4; ++jc) {
    for (int cc = 0; cc < 16; ++cc) {
      const int c = jc * 16 + cc;
      if (tx == cc) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (ty + 16 * i >= c) col[ty + 16 * i] = t[i][jc];
      }
      __syncthreads();
      if (threadIdx.x < NB && static_cast<int>(threadIdx.x) >= c) {
        const int r = threadIdx.x;
        const double v = col[c];
        const double d = sqrt(fmax(v, 1e-300));
        if (r == c && !(v > 0.0)) fail[q] = 1;
        const double l = r == c ? d : col[r] / d;
        s[r][c] = l;
        lbuf[r] = l;
      }
      __syncthreads();
      double lr[4], lq[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        lr[i] = lbuf[ty + 16 * i];
        lq[i] = lbuf[tx + 16 * i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r = ty + 16 * i, qq = tx + 16 * j;
          if (qq > c && qq <= r) t[i][j] = fma(-lr[i], lq[j], t[i][j]);
        }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e % NB, c = e / NB;
    if (r < bs && c < bs) a[r + static_cast<long long>(c) * M.n] = r >= c ? s[r][c] : 0.0;
  }
  // L⁻¹ by forward substitution down the rows, four lanes per column (a column only reads its own
  // earlier entries, so the four lanes synchronise within their warp only)
  {
    const int c = threadIdx.x >> 2, part = threadIdx.x & 3;
    for (int r = 0; r < NB; ++r) {
      double v = 0.0;
      if (r > c)
        for (int qq = c + part; qq < r; qq += 4) v += s[r][qq] * X[qq][c];
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      if (part == 0) X[r][c] = r < c ? 0.0 : ((r == c ? 1.0 : 0.0) - v) / s[r][r];
      __syncwarp();
    }
  }
  __syncthreads();
  double* o = Dinv + doff[q] + static_cast<long long>(k) * NB * NB;
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) o[e] = X[e % NB][e / NB];
}


// Block row k of the tile-packed factor: tiles (k, first_k <= j < k) copied from the factored matrix
// (zero padding past n) and the diagonal tile D_k = L_kk⁻¹ from the workspace. task = (matrix, k);
// ef/eb: the matrix's envelope (first tile and packed base of every block row, at eoff[matrix])
__global__ void k_pack_row(const double* __restrict__ A, const Mat* __restrict__ mats, const int2* __restrict__ tasks,
                           double* __restrict__ P, const long long* __restrict__ poff, const double* __restrict__ Dinv,
                           const long long* __restrict__ doff, const int* __restrict__ eoff,
                           const int* __restrict__ efirst, const int* __restrict__ ebase) {
  const int2 t = tasks[blockIdx.x];
  const Mat M = mats[t.x];
  const int k = t.y, k0 = k * NB, bs = min(NB, M.n - k0);
  const int f = efirst[eoff[t.x] + k];
  double* row = P + poff[t.x] + static_cast<long long>(ebase[eoff[t.x] + k]) * (NB * NB);  // tile (k, j) at row + j·64²
  for (int j = f; j < k; ++j) {
    const double* a = A + M.off + k0 + static_cast<long long>(j * NB) * M.n;
    double* o = row + static_cast<long long>(j) * NB * NB;
    for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
      const int r = e % NB, c = e / NB;
      o[e] = r < bs ? a[r + static_cast<long long>(c) * M.n] : 0.0;
    }
  }
  const double* d = Dinv + doff[t.x] + static_cast<long long>(k) * NB * NB;
  double* o = row + static_cast<long long>(k) * NB * NB;
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) o[e] = d[e];
}

// Mi[k-block, k-block] = D_k (task = (matrix, k)), for M = L⁻¹ by block rows
__global__ void k_set_diag(double* __restrict__ Mi, const Mat* __restrict__ mats, const int2* __restrict__ tasks,
                           const double* __restrict__ Dinv, const long long* __restrict__ doff) {
  const int2 t = tasks[blockIdx.x];
  const Mat M = mats[t.x];
  const int k0 = t.y * NB, bs = min(NB, M.n - k0);
  const double* d = Dinv + doff[t.x] + static_cast<long long>(t.y) * NB * NB;
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e % NB, cc = e / NB;
    if (r < bs && cc < bs) Mi[M.off + (k0 + r) + static_cast<long long>(k0 + cc) * M.n] = d[e];
  }
}
// block row k of the packed lower tiles of a full symmetric matrix (lower triangle valid), in the
// explicit-inverse layout (inv_tile_off / inv_tile_ld)
__global__ void k_pack_lower(const double* __restrict__ F, const Mat* __restrict__ mats, const int2* __restrict__ tasks,
                             double* __restrict__ P, const long long* __restrict__ poff) {
  const int2 t = tasks[blockIdx.x];
  const Mat M = mats[t.x];
  const int k = t.y, k0 = k * NB, bs = min(NB, M.n - k0);
  const int ld = inv_tile_ld(M.n, k);
  for (int j = 0; j <= k; ++j) {
    const double* a = F + M.off + k0 + static_cast<long long>(j * NB) * M.n;
    const int bj = min(NB, M.n - j * NB);
    double* o = P + poff[t.x] + inv_tile_off(M.n, k, j);
    for (int e = threadIdx.x; e < ld * NB; e += blockDim.x) {
      const int r = e % ld, c = e / ld;
      double v = 0.0;
      if (r < bs && c < bj) v = (j < k || r >= c) ? a[r + static_cast<long long>(c) * M.n]
                                                  : a[c + static_cast<long long>(r) * M.n];  // diag tile: mirror
      o[e] = v;
    }
  }
}

// ‖A‖_F of a symmetric matrix from its lower triangle (the upper one may hold garbage): kFrobParts
// CTAs per matrix stream column ranges (coalesced), partials summed per matrix in a fixed order
constexpr int kFrobParts = 64;
__global__ void k_frob_part(const double* __restrict__ A, const Mat* __restrict__ mats, double* __restrict__ part) {
  const Mat M = mats[blockIdx.y];
  double s = 0.0;
  for (int cc = blockIdx.x; cc < M.n; cc += gridDim.x) {
    const double* col = A + M.off + static_cast<long long>(cc) * M.n;
    for (int r = cc + threadIdx.x; r < M.n; r += blockDim.x) {
      const double v = col[r];
      s += (r == cc ? 1.0 : 2.0) * v * v;
    }
  }
  __shared__ double sh[32];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    s = warp_sum(s);
    if (threadIdx.x == 0) part[blockIdx.y * kFrobParts + blockIdx.x] = s;
  }
}
__global__ void k_frob_sum(const double* __restrict__ part, int B, double* __restrict__ out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  double s = 0.0;
  for (int x = 0; x < kFrobParts; ++x) s += part[b * kFrobParts + x];
  out[b] = sqrt(s);
}

// λmax of symmetric PSD matrices by power iteration (one CTA per matrix, x in shared memory)
__global__ void k_power(const double* __restrict__ A, const Mat* __restrict__ mats, int iters,
                        double* __restrict__ out) {
  extern __shared__ double x[];
  __shared__ double sh[32];
  __shared__ double nrm;
  const Mat M = mats[blockIdx.x];
  const double* a = A + M.off;
  double* y = x + M.n;
  for (int i = threadIdx.x; i < M.n; i += blockDim.x) x[i] = 1.0 + 0.25 * sin(0.7 * i + 0.3);
  __syncthreads();
  double lam = 0.0;
  for (int it = 0; it <= iters; ++it) {
    double part = 0.0;
    for (int r = threadIdx.x; r < M.n; r += blockDim.x) {
      double s = 0.0;
      for (int c = 0; c < M.n; ++c) s += a[r + static_cast<long long>(c) * M.n] * x[c];
      y[r] = s;
      part += s * s;
    }
    part = warp_sum(part);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0, xx = 0.0;
      for (int w = 0; w < (blockDim.x >> 5); ++w) t += sh[w];
      for (int i = 0; i < M.n; ++i) xx += x[i] * x[i];
      nrm = sqrt(t);
      lam = nrm / sqrt(xx);
      sh[0] = lam;
    }
    __syncthreads();
    lam = sh[0];
    const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
    for (int i = threadIdx.x; i < M.n; i += blockDim.x) x[i] = y[i] * inv;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = lam;
}

// GEMM tasks of one factor step, generated on the device from one descriptor per (matrix, kind):
// kind 0 = inside the outer panel (columns jb in (k, oend), K = 64 at column k), kind 1 = right of
// a completed outer panel (jb >= oend, K = the panel width): C[ib, jb] -= A_ib A_jbᵀ; kind 2 = the
// panel solve A[ib, k] <- A[ib, k] D_kᵀ for ib > k (in place: each CTA reads its whole tile before
// its epilogue writes it).
struct UpdDesc {
  long long off;   // matrix offset
  long long first; // first task index of this entry
  int n, k, ostart, oend, kind;
  int nbk;         // block rows to enumerate: one past the last row whose envelope reaches the step
  const double* D; // kind 2: D_k
  const int* ef;   // the matrix's envelope: first tile of every block row
};
// Envelope: a block row ib whose first tile lies right of the step's columns holds zeros there, so
// its panel solve and its updates (as row or as column of the updated tile) are skipped — the
// candidates are enumerated densely over the first nbk block rows and the skipped ones become
// empty tasks (M = 0: the GEMM CTA exits). After an outer panel the K range of an update starts at
// the later of the two rows' first tiles.
__global__ void k_make_updates(double* __restrict__ A, const UpdDesc* __restrict__ d, int nd, long long total,
                               GemmTask* __restrict__ out) {
  const long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (t >= total) return;
  int lo = 0, hi = nd - 1;  // last entry with first <= t
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (d[mid].first <= t) lo = mid;
    else hi = mid - 1;
  }
  const UpdDesc e = d[lo];
  long long loc = t - e.first;
  const int nb = e.nbk;
  double* base = A + e.off;
  GemmTask g{};
  g.gA = g.gB = nullptr;
  g.tm = g.tn = 0;
  if (e.kind == 2) {
    const int ib = e.k + 1 + static_cast<int>(loc), k0 = e.k * NB;
    g.A = base + ib * NB + static_cast<long long>(k0) * e.n;
    g.B = e.D;
    g.Cm = base + ib * NB + static_cast<long long>(k0) * e.n;
    g.M = e.ef[ib] <= e.k ? min(NB, e.n - ib * NB) : 0;
    g.N = g.K = min(NB, e.n - k0);
    g.lda = g.ldc = e.n;
    g.ldb = NB;
    g.beta = 0.0;
    g.alpha = 1.0;
    out[t] = g;
    return;
  }
  const int jb0 = e.kind == 0 ? e.k + 1 : e.oend;
  const int jb1 = e.kind == 0 ? min(e.oend, nb) : nb;  // exclusive
  int jb = jb0;
  for (; jb < jb1; ++jb) {  // column jb holds rows ib = jb .. nb-1
    const long long cnt = nb - jb;
    if (loc < cnt) break;
    loc -= cnt;
  }
  const int ib = jb + static_cast<int>(loc);
  const int last = e.kind == 0 ? e.k : e.oend - 1;  // last tile column of the step's K range
  const int fi = e.ef[ib], fj = e.ef[jb];
  const bool live = fi <= last && fj <= last;
  const int cb = e.kind == 0 ? e.k : max(e.ostart, max(fi, fj));
  const int c0 = cb * NB;
  const int kw = e.kind == 0 ? min(NB, e.n - c0) : min(e.n, e.oend * NB) - c0;
  g.A = base + ib * NB + static_cast<long long>(c0) * e.n;
  g.B = base + jb * NB + static_cast<long long>(c0) * e.n;
  g.Cm = base + ib * NB + static_cast<long long>(jb) * NB * e.n;
  g.M = live ? min(NB, e.n - ib * NB) : 0;
  g.N = min(NB, e.n - jb * NB);
  g.K = kw;
  g.lda = g.ldb = g.ldc = e.n;
  g.beta = 1.0;
  g.alpha = -1.0;
  out[t] = g;
}

// ---- batched solves with the tile-packed factor ---------------------------------------------
// tile (k, j) of a packed factor whose block row k starts at packed tile base eb[k] + ef[k]
__device__ __forceinline__ const double* ptile(const double* P, const int* eb, int k, int j) {
  return P + static_cast<long long>(eb[k] + j) * (NB * NB);
}

// v <- (L Lᵀ)⁻¹ v in shared memory (nb*64 entries, zero-padded past n); red: kSolveWarps*64.
// ef/eb: the factor's envelope (block row k holds tiles ef[k]..k).
// Forward (row by row) y_k = L_kk⁻¹ (v_k - Σ_{ef[k] <= j < k} L_kj y_j); backward, also row by row so
// that each block row is one contiguous stream: for k = nb-1..0, x_k = L_kk⁻ᵀ y_k, then
// y_j -= L_kjᵀ x_k for ef[k] <= j < k. Off-diagonal tiles are split over the warps, each tile column
// streamed as one 512-byte warp load; the transposed tiles of the backward pass reduce 32 columns
// per 31 shuffles and each is applied by its one warp (distinct j: no cross-warp sum).
__device__ void chol_solve(const double* __restrict__ P, int nb, double* v, double* red, const int* __restrict__ ef,
                           const int* __restrict__ eb) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
  for (int k = 0; k < nb; ++k) {
    double a0 = 0.0, a1 = 0.0;
    for (int j = ef[k] + warp; j < k; j += kSolveWarps) {
      const double2* t = reinterpret_cast<const double2*>(ptile(P, eb, k, j)) + lane;
      const double* y = v + j * NB;
#pragma unroll 16
      for (int c = 0; c < NB; ++c) {
        const double2 a = __ldcs(t + c * (NB / 2));
        a0 += a.x * y[c];
        a1 += a.y * y[c];
      }
    }
    red[warp * NB + 2 * lane] = a0;
    red[warp * NB + 2 * lane + 1] = a1;
    __syncthreads();
    if (tid < NB) {
      double s = v[k * NB + tid];
      for (int w = 0; w < kSolveWarps; ++w) s -= red[w * NB + tid];
      v[k * NB + tid] = s;
    }
    __syncthreads();
    {
      const double2* t = reinterpret_cast<const double2*>(ptile(P, eb, k, k)) + lane;
      const double* r = v + k * NB;
      double b0 = 0.0, b1 = 0.0;
#pragma unroll
      for (int c = warp * (NB / kSolveWarps); c < (warp + 1) * (NB / kSolveWarps); ++c) {
        const double2 a = __ldcs(t + c * (NB / 2));
        b0 += a.x * r[c];
        b1 += a.y * r[c];
      }
      red[warp * NB + 2 * lane] = b0;
      red[warp * NB + 2 * lane + 1] = b1;
    }
    __syncthreads();
    if (tid < NB) {
      double s = 0.0;
      for (int w = 0; w < kSolveWarps; ++w) s += red[w * NB + tid];
      v[k * NB + tid] = s;
    }
    __syncthreads();
  }
  for (int k = nb - 1; k >= 0; --k) {
    double mine = 0.0;  // x_k = D_kᵀ y_k: this warp's NB/kSolveWarps columns of the diagonal tile
    {
      const double* t = ptile(P, eb, k, k);
      const double r0 = v[k * NB + 2 * lane], r1 = v[k * NB + 2 * lane + 1];
      constexpr int CW = NB / kSolveWarps;
#pragma unroll
      for (int cc = 0; cc < CW; ++cc) {
        const double2 a = __ldcs(reinterpret_cast<const double2*>(t + (warp * CW + cc) * NB) + lane);
        const double s = warp_sum(a.x * r0 + a.y * r1);
        if (lane == cc) mine = s;
      }
    }
    __syncthreads();
    if (lane < NB / kSolveWarps) v[k * NB + warp * (NB / kSolveWarps) + lane] = mine;
    __syncthreads();
    const double x0 = v[k * NB + 2 * lane], x1 = v[k * NB + 2 * lane + 1];
    for (int j = ef[k] + warp; j < k; j += kSolveWarps) {  // y_j -= L_kjᵀ x_k
      const double* t = ptile(P, eb, k, j);
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        double p[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const double2 a = __ldcs(reinterpret_cast<const double2*>(t + (g * 32 + c) * NB) + lane);
          p[c] = a.x * x0 + a.y * x1;
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
          const bool up = (lane & o) != 0;
#pragma unroll
          for (int i = 0; i < o; ++i) {
            const double send = up ? p[i] : p[i + o];
            const double keep = up ? p[i + o] : p[i];
            p[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
        }
        v[j * NB + g * 32 + lane] -= p[0];
      }
    }
    __syncthreads();
  }
}

// v <- P v for a symmetric P stored as its lower 64x64 tiles (k, j<=k) in the same packed order
// (diagonal tiles full). Each tile is read once and serves both y_k += P_kj v_j and, for j < k,
// y_j += P_kjᵀ v_k (32 columns per 31 shuffles); every warp accumulates into its own partial
// vector in shared memory (part: kSolveWarps x nb*64), summed in warp order: deterministic.
__device__ void symv_packed(const double* __restrict__ P, int n, double* v, double* part, int t0 = 0, int tstep = 1) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
  const int nb = (n + NB - 1) / NB;
  const int len = nb * NB;
  double* my = part + static_cast<size_t>(warp) * len;
  for (int i = lane; i < len; i += 32) my[i] = 0.0;
  __syncwarp();
  const int T = nb * (nb + 1) / 2;
  const int first = t0 + warp * tstep, stride = kSolveWarps * tstep;  // this warp's tiles
  int k = 0, j = first;  // tile t = k(k+1)/2 + j
  while (j > k) {
    j -= k + 1;
    ++k;
  }
  for (int t = first; t < T; t += stride) {
    const double* tile = P + inv_tile_off(n, k, j);
    const int ld = inv_tile_ld(n, k);
    const bool rv = 2 * lane < ld;  // rows 2 lane, 2 lane + 1 are stored (ld is a multiple of 8)
    const double* gj = v + j * NB;
    const double gk0 = v[k * NB + 2 * lane], gk1 = v[k * NB + 2 * lane + 1];
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double p[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        double2 a = make_double2(0.0, 0.0);
        if (rv) a = __ldcs(reinterpret_cast<const double2*>(tile + (h * 32 + c) * ld) + lane);
        const double gc = gj[h * 32 + c];
        a0 += a.x * gc;
        a1 += a.y * gc;
        p[c] = a.x * gk0 + a.y * gk1;
      }
      if (j < k) {  // warp-uniform
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
          const bool up = (lane & o) != 0;
#pragma unroll
          for (int i = 0; i < o; ++i) {
            const double send = up ? p[i] : p[i + o];
            const double keep = up ? p[i + o] : p[i];
            p[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
        }
        my[j * NB + h * 32 + lane] += p[0];
      }
    }
    my[k * NB + 2 * lane] += a0;
    my[k * NB + 2 * lane + 1] += a1;
    __syncwarp();
    j += stride;
    while (j > k && k < nb) {
      j -= k + 1;
      ++k;
    }
  }
  __syncthreads();
  for (int i = tid; i < len; i += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < kSolveWarps; ++w) s += part[static_cast<size_t>(w) * len + i];
    v[i] = s;
  }
  __syncthreads();
}

// λmax(A⁻¹) by power iteration through the factor: one CTA per matrix
__global__ void __launch_bounds__(kSolveWarps * 32) k_chol_power(const double* __restrict__ P,
                                                                 const long long* __restrict__ poff,
                                                                 const int* __restrict__ nvec, int iters, int nbmax,
                                                                 double* __restrict__ out, int inverse,
                                                                 const int* __restrict__ eoff,
                                                                 const int* __restrict__ efirst,
                                                                 const int* __restrict__ ebase) {
  extern __shared__ double sm[];
  double* x = sm;
  double* red = sm + static_cast<size_t>(nbmax) * NB;  // solve: kSolveWarps*64; symv: kSolveWarps*nbmax*64
  __shared__ double nrm_s;
  const int i = blockIdx.x, n = nvec[i], nb = (n + NB - 1) / NB;
  for (int r = threadIdx.x; r < nb * NB; r += blockDim.x) x[r] = r < n ? 1.0 + 0.25 * sin(0.7 * r + 0.3) : 0.0;
  double lam = 0.0;
  for (int it = 0; it <= iters; ++it) {
    double s = 0.0;
    for (int r = threadIdx.x; r < n; r += blockDim.x) s += x[r] * x[r];
    s = warp_sum(s);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < kSolveWarps; ++w) t += red[w];
      nrm_s = sqrt(t);
    }
    __syncthreads();
    const double nrm = nrm_s;
    if (it > 0) lam = nrm;  // ‖A⁻¹ x‖ with ‖x‖ = 1
    if (it == iters || !(nrm > 0.0)) break;
    for (int r = threadIdx.x; r < n; r += blockDim.x) x[r] /= nrm;
    __syncthreads();
    if (inverse) symv_packed(P + poff[i], n, x, red);
    else chol_solve(P + poff[i], nb, x, red, efirst + eoff[i], ebase + eoff[i]);
  }
  if (threadIdx.x == 0) out[i] = lam;
}

}  // namespace

std::vector<double> batched_power(Ctx& c, const double* A, const std::vector<int>& n,
                                  const std::vector<long long>& off, int iters) {
  ScopedKernelTimer tk(c, "power");
  const int B = static_cast<int>(n.size());
  std::vector<double> out(B, 0.0);
  if (B == 0) return out;
  std::vector<Mat> mats(B);
  int nmax = 0;
  for (int i = 0; i < B; ++i) {
    mats[i] = {off[i], n[i]};
    nmax = std::max(nmax, n[i]);
  }
  DBuf<Mat> dm;
  DBuf<double> d;
  dm.upload(mats, c.stream);
  d.ensure(B);
  const size_t smem = 2 * sizeof(double) * nmax;
  if (smem > 32 * 1024)
    RDD_CUDA(cudaFuncSetAttribute(k_power, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  k_power<<<B, 256, smem, c.stream>>>(A, dm.p, iters, d.p);
  RDD_LAUNCH_CHECK();
  d.download(out.data(), B, c.stream);
  RDD_CUDA(cudaStreamSynchronize(c.stream));
  return out;
}

// In: A (batch at off[i], order n[i], symmetric, full storage) — destroyed (holds L).
// Out: the tile-packed factor at P + poff[i] (diagonal tiles inverted), fail[i] = 1 when a pivot
// was not positive, frob_A[i] = ‖A_i‖_F (an upper bound of λmax).
void batched_cholesky_pack(Ctx& c, double* A, const std::vector<int>& ids, const std::vector<int>& n,
                           const std::vector<long long>& off, double* P, const std::vector<long long>& poff,
                           std::vector<int>& fail, std::vector<double>& frob_A, bool inverse,
                           std::vector<double>* frob_P, double** Pfull_out) {
  ScopedKernelTimer tk(c, "cholesky");
  const int B = static_cast<int>(n.size());
  fail.assign(B, 0);
  frob_A.assign(B, 0.0);
  if (B == 0) return;
  std::vector<Mat> mats(B);
  int nmax = 0;
  for (int i = 0; i < B; ++i) {
    mats[i] = {off[i], n[i]};
    nmax = std::max(nmax, n[i]);
  }
  RDD_CUDA(cudaFuncSetAttribute(k_potrf_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, kPairSmem));
  DBuf<Mat> dm;
  DBuf<int> dfail, dact;
  DBuf<double> dfa;
  DBuf<long long> dpoff, ddoff;
  dm.upload(mats, c.stream);
  dfail.zero(B, c.stream);
  dfa.ensure(B);
  {
    DBuf<double> fpart;
    fpart.ensure(static_cast<size_t>(B) * kFrobParts);
    k_frob_part<<<dim3(kFrobParts, B), 256, 0, c.stream>>>(A, dm.p, fpart.p);
    RDD_LAUNCH_CHECK();
    k_frob_sum<<<ceil_div(B, 128), 128, 0, c.stream>>>(fpart.p, B, dfa.p);
    RDD_LAUNCH_CHECK();
  }
  std::vector<long long> doff(B);
  long long dtot = 0;
  for (int i = 0; i < B; ++i) {
    doff[i] = dtot;
    dtot += static_cast<long long>(ceil_div(n[i], NB)) * NB * NB;
  }
  double* Dinv = c.ws("chol.Dinv", std::max<long long>(1, dtot));
  ddoff.upload(doff, c.stream);
  // two-level blocking: 64-wide steps update only the columns of their 512-wide outer panel;
  // the trailing matrix right of an outer panel takes one K = 512 update when the panel is done.
  // Every step's work lists are built up front and uploaded once: the step loop only launches.
  const int nbmax = ceil_div(nmax, NB);
  int kOuter = 8;  // inner blocks per outer panel (8: measured best of 4/8/16)
  if (const char* e = std::getenv("RDD_CHOL_OUTER")) kOuter = std::max(1, std::atoi(e));  // tuning experiments only
  struct Step {
    size_t act0, nact, sd0, nsd, ud0, nud;
    long long stotal, utotal;
  };
  std::vector<Step> steps(nbmax);
  std::vector<int> act;
  std::vector<UpdDesc> sd, ud;
  long long tmax = 0;
  for (int k = 0; k < nbmax; ++k) {
    Step& st = steps[k];
    st.act0 = act.size();
    st.sd0 = sd.size();
    st.ud0 = ud.size();
    long long stotal = 0, utotal = 0;
    const int ostart = (k / kOuter) * kOuter;
    for (int i = 0; i < B; ++i) {
      const int nb = ceil_div(n[i], NB);
      if (k >= nb) continue;
      act.push_back(i);
      const int oend = std::min(nb, ostart + kOuter);
      const int* efh = c.env_first.data() + c.env_off[ids[i]];
      const int* efd = c.denv_first.p + c.env_off[ids[i]];
      // block rows whose envelope reaches column k (the step's panel solve and K = 64 updates)
      int nbk = k + 1;
      for (int ib = nb - 1; ib > k; --ib)
        if (efh[ib] <= k) {
          nbk = ib + 1;
          break;
        }
      if (nbk - k - 1 > 0) {  // panel solve
        sd.push_back({off[i], stotal, n[i], k, ostart, oend, 2, nbk,
                      Dinv + doff[i] + static_cast<long long>(k) * NB * NB, efd});
        stotal += nbk - k - 1;
      }
      long long cnt = 0;
      for (int jb = k + 1; jb < std::min(oend, nbk); ++jb) cnt += nbk - jb;
      if (cnt > 0) {
        ud.push_back({off[i], utotal, n[i], k, ostart, oend, 0, nbk, nullptr, efd});
        utotal += cnt;
      }
      if (k == oend - 1 && oend < nb) {  // the completed outer panel's K = 512 update of the trailing matrix
        int nbo = oend;
        for (int ib = nb - 1; ib >= oend; --ib)
          if (efh[ib] < oend) {
            nbo = ib + 1;
            break;
          }
        const long long T = nbo - oend;
        if (T > 0) {
          ud.push_back({off[i], utotal, n[i], k, ostart, oend, 1, nbo, nullptr, efd});
          utotal += T * (T + 1) / 2;
        }
      }
    }
    st.nact = act.size() - st.act0;
    st.nsd = sd.size() - st.sd0;
    st.nud = ud.size() - st.ud0;
    st.stotal = stotal;
    st.utotal = utotal;
    tmax = std::max(tmax, std::max(stotal, utotal));
  }
  DBuf<UpdDesc> dsd, dud;
  DBuf<GemmTask>& dtask = c.wsg;
  dact.upload(act, c.stream);
  dsd.upload(sd, c.stream);
  dud.upload(ud, c.stream);
  dtask.ensure(static_cast<size_t>(std::max<long long>(1, tmax)));
  for (int k = 0; k < nbmax; ++k) {
    const Step& st = steps[k];
    {
      ScopedKernelTimer tp(c, "potrf");
      k_potrf_diag<<<static_cast<int>(st.nact), 256, kPairSmem, c.stream>>>(A, dm.p, dact.p + st.act0, k, dfail.p,
                                                                             Dinv, ddoff.p);
      RDD_LAUNCH_CHECK();
    }
    if (st.stotal > 0) {  // panel: A[ib, k] <- A[ib, k] D_kᵀ on DMMA
      k_make_updates<<<ceil_div(st.stotal, 256), 256, 0, c.stream>>>(A, dsd.p + st.sd0, static_cast<int>(st.nsd),
                                                                      st.stotal, dtask.p);
      RDD_LAUNCH_CHECK();
      gemm_nt_dev(c, dtask.p, static_cast<int>(st.stotal));
    }
    if (st.utotal > 0) {
      k_make_updates<<<ceil_div(st.utotal, 256), 256, 0, c.stream>>>(A, dud.p + st.ud0, static_cast<int>(st.nud),
                                                                      st.utotal, dtask.p);
      RDD_LAUNCH_CHECK();
      gemm_nt_dev(c, dtask.p, static_cast<int>(st.utotal));
    }
  }
  DBuf<int2> drows;
  std::vector<int2> rows;
  for (int i = 0; i < B; ++i)
    for (int k = 0; k < ceil_div(n[i], NB); ++k) rows.push_back(make_int2(i, k));
  drows.upload(rows, c.stream);
  dpoff.upload(poff, c.stream);
  if (!inverse) {
    std::vector<int> eo(B);
    for (int i = 0; i < B; ++i) eo[i] = c.env_off[ids[i]];
    DBuf<int> deo;
    deo.upload(eo, c.stream);
    k_pack_row<<<static_cast<int>(rows.size()), 256, 0, c.stream>>>(A, dm.p, drows.p, P, dpoff.p, Dinv, ddoff.p, deo.p,
                                                                     c.denv_first.p, c.denv_base.p);
    RDD_LAUNCH_CHECK();
  } else {
    // explicit inverse for small blocks: M = L⁻¹ by block rows (M_kk = D_k,
    // M[ib, :ib] = -D_ib L[ib, :ib] M[:ib, :ib]), then A⁻¹ = MᵀM (lower tiles), packed
    const size_t tot = static_cast<size_t>(off[B - 1] + static_cast<long long>(n[B - 1]) * n[B - 1]);
    double* Mi = c.ws("chol.Minv", tot);
    double* Pf = c.ws("chol.Pfull", tot);
    RDD_CUDA(cudaMemsetAsync(Mi, 0, tot * sizeof(double), c.stream));
    k_set_diag<<<static_cast<int>(rows.size()), 256, 0, c.stream>>>(Mi, dm.p, drows.p, Dinv, ddoff.p);
    RDD_LAUNCH_CHECK();
    long long tmp_sz = 0;
    std::vector<long long> toff(B);
    for (int i = 0; i < B; ++i) {
      toff[i] = tmp_sz;
      tmp_sz += static_cast<long long>(NB) * n[i];
    }
    double* tmp = c.ws("chol.tmp", std::max<long long>(1, tmp_sz));
    for (int ib = 1; ib < nbmax; ++ib) {
      std::vector<GemmTask> g1, g2;
      for (int i = 0; i < B; ++i) {
        if (ib >= ceil_div(n[i], NB)) continue;
        const int bi = std::min(NB, n[i] - ib * NB), wd = ib * NB;
        double* L = A + off[i];
        double* Mm = Mi + off[i];
        for (int tn = 0; tn < ib; ++tn) {
          const int k0 = tn * NB;
          GemmTask t{};  // tmp[:, tn] = L[ib, k0:wd] M[k0:wd, tn]  (M lower triangular)
          t.A = L + ib * NB + static_cast<long long>(k0) * n[i];
          t.B = Mm + k0 + static_cast<long long>(k0) * n[i];
          t.Cm = tmp + toff[i] + static_cast<long long>(k0) * NB;
          t.M = bi;
          t.N = NB;
          t.K = wd - k0;
          t.lda = t.ldb = n[i];
          t.ldc = NB;
          t.alpha = 1.0;
          g1.push_back(t);
          GemmTask u{};  // M[ib, tn] = -D_ib tmp[:, tn]
          u.A = Mm + ib * NB + static_cast<long long>(ib * NB) * n[i];
          u.B = tmp + toff[i];
          u.Cm = Mm + ib * NB;
          u.M = bi;
          u.N = wd;
          u.K = bi;
          u.lda = n[i];
          u.ldb = NB;
          u.ldc = n[i];
          u.tn = tn;
          u.alpha = -1.0;
          g2.push_back(u);
        }
      }
      gemm_nn(c, g1);
      gemm_nn(c, g2);
    }
    std::vector<GemmTask> g;
    for (int i = 0; i < B; ++i)
      for (int tm = 0; tm < ceil_div(n[i], NB); ++tm)
        for (int tn = 0; tn <= tm; ++tn) {
          GemmTask t{};
          const int k0 = tm * NB;  // rows of M below the tile's first output row
          t.A = Mi + off[i] + k0;
          t.B = Mi + off[i] + k0;
          t.Cm = Pf + off[i];
          t.M = t.N = n[i];
          t.K = n[i] - k0;
          t.lda = t.ldb = t.ldc = n[i];
          t.tm = tm;
          t.tn = tn;
          t.alpha = 1.0;
          g.push_back(t);
        }
    gemm_tn(c, g);  // P = MᵀM, lower tiles
    k_pack_lower<<<static_cast<int>(rows.size()), 256, 0, c.stream>>>(Pf, dm.p, drows.p, P, dpoff.p);
    RDD_LAUNCH_CHECK();
    if (frob_P) {
      DBuf<double> fpart, dfp;
      fpart.ensure(static_cast<size_t>(B) * kFrobParts);
      dfp.ensure(B);
      k_frob_part<<<dim3(kFrobParts, B), 256, 0, c.stream>>>(Pf, dm.p, fpart.p);
      RDD_LAUNCH_CHECK();
      k_frob_sum<<<ceil_div(B, 128), 128, 0, c.stream>>>(fpart.p, B, dfp.p);
      RDD_LAUNCH_CHECK();
      frob_P->assign(B, 0.0);
      dfp.download(frob_P->data(), B, c.stream);
    }
    if (Pfull_out) *Pfull_out = Pf;
  }
  dfail.download(fail.data(), B, c.stream);
  dfa.download(frob_A.data(), B, c.stream);
  RDD_CUDA(cudaStreamSynchronize(c.stream));
}

long long packed_chol_size(int n) {
  const long long nb = ceil_div(n, NB);
  return nb * (nb + 1) / 2 * NB * NB;
}
long long packed_inverse_size(int n) {  // explicit-inverse layout: trimmed last block row
  const long long nb = ceil_div(n, NB);
  return (nb - 1) * nb / 2 * NB * NB + nb * NB * inv_last_ld(n);
}

size_t chol_solve_smem(int nmax, bool inverse) {
  const size_t len = static_cast<size_t>(ceil_div(nmax, NB)) * NB;
  return (len + (inverse ? kSolveWarps * len : kSolveWarps * NB)) * sizeof(double);
}

std::vector<double> batched_inv_power(Ctx& c, const double* P, const std::vector<int>& ids, const std::vector<int>& n,
                                      const std::vector<long long>& poff, int iters, bool inverse) {
  ScopedKernelTimer tk(c, "inv_power");
  const int B = static_cast<int>(n.size());
  std::vector<double> out(B, 0.0);
  if (B == 0) return out;
  const int nmax = *std::max_element(n.begin(), n.end());
  // largest blocks first (one CTA each, time ∝ n²): no big block starts in the last wave
  std::vector<int> perm(B);
  for (int b = 0; b < B; ++b) perm[b] = b;
  std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return n[a] > n[b]; });
  std::vector<int> ns(B), eo(B);
  std::vector<long long> ps(B);
  for (int b = 0; b < B; ++b) {
    ns[b] = n[perm[b]];
    ps[b] = poff[perm[b]];
    eo[b] = c.env_off[ids[perm[b]]];
  }
  DBuf<int> dn, deo;
  deo.upload(eo, c.stream);
  DBuf<long long> dp;
  DBuf<double> d;
  dn.upload(ns, c.stream);
  dp.upload(ps, c.stream);
  d.ensure(B);
  const size_t smem = chol_solve_smem(nmax, inverse);
  if (c.verbose) std::fprintf(stderr, "[inv_power] B=%d nmax=%d smem=%zu iters=%d\n", B, nmax, smem, iters);
  RDD_CUDA(cudaFuncSetAttribute(k_chol_power, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  k_chol_power<<<B, kSolveWarps * 32, smem, c.stream>>>(P, dp.p, dn.p, iters, ceil_div(nmax, NB), d.p,
                                                        inverse ? 1 : 0, deo.p, c.denv_first.p, c.denv_base.p);
  RDD_LAUNCH_CHECK();
  std::vector<double> sorted(B);
  d.download(sorted.data(), B, c.stream);
  RDD_CUDA(cudaStreamSynchronize(c.stream));
  for (int b = 0; b < B; ++b) out[perm[b]] = sorted[b];
  return out;
}

// Schwarz local apply, factor mode: z_i = A_i⁻¹ g_i, g_i = w(v)[S_i] (schwarz.hpp:153-215: SAS/RAS
// weights in front of the local solve for the transpose) through the envelope-packed Cholesky
// factor or, for eigen-fallback subdomains, the dense pseudo-inverse. One CTA per subdomain; CTAs
// take the subdomains largest first (order): the per-CTA streaming time grows with n_i², so the
// biggest local solves must not start in the last wave. (The explicit inverses of the small-block
// mode go through k_inv_apply_tma below.)
__global__ void __launch_bounds__(kSolveWarps * 32) k_chol_apply(
    const double* __restrict__ P, const long long* __restrict__ poff, const double* const* __restrict__ dense,
    const int* __restrict__ set_ptr, const int* __restrict__ set_idx, const double* __restrict__ v,
    const int* __restrict__ mult, const int* __restrict__ owner, int kind, int transpose, int nbmax,
    double* __restrict__ z, const int* __restrict__ live, const int* __restrict__ order,
    const int* __restrict__ eoff, const int* __restrict__ efirst, const int* __restrict__ ebase) {
  if (live && *live != 0) return;  // solver loop already stopped (speculative graph iteration)
  extern __shared__ double sm[];
  double* g = sm;
  double* red = sm + static_cast<size_t>(nbmax) * NB;
  const int i = order ? order[blockIdx.x] : blockIdx.x;
  const int s0 = set_ptr[i], n = set_ptr[i + 1] - s0, nb = (n + NB - 1) / NB;
  for (int q = threadIdx.x; q < nb * NB; q += blockDim.x) {
    double val = 0.0;
    if (q < n) {
      const int col = set_idx[s0 + q];
      val = v[col];
      if (transpose) {
        if (kind == RDD_PRECOND_SAS) val /= mult[col];
        else if (kind == RDD_PRECOND_RAS) val = owner[col] == i ? val : 0.0;
      }
    }
    g[q] = val;
  }
  __syncthreads();
  const double* D = dense[i];
  if (D) {
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
      double acc = 0.0;
      for (int q = 0; q < n; ++q) acc += D[r + static_cast<long long>(q) * n] * g[q];
      z[s0 + r] = acc;
    }
    return;
  }
  chol_solve(P + poff[i], nb, g, red, efirst + eoff[i], ebase + eoff[i]);
  for (int r = threadIdx.x; r < n; r += blockDim.x) z[s0 + r] = g[r];
}

// ---- explicit-inverse apply through a TMA ring (small blocks: C1, C2, C4). The packed lower tiles
// of A_i⁻¹ (64x64, 32 KB each, block row after block row) are streamed by one producer warp with
// 1-D bulk copies (cp.async.bulk, mbarrier completion) into a 2-stage shared-memory ring; eight
// consumer warps split every tile by columns (8 each): y_k += T_kj g_j accumulates per lane in
// registers along the block row, y_j += T_kjᵀ g_k is reduced per column (fold + butterfly) and added
// by its one owning lane. Memory latency is covered by the copies in flight, not by resident warps.
// Two CTAs per subdomain take alternate tiles (partials to z and z + zhalf, summed by k_reduce).
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT%=:\n\t"
      "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

constexpr int kTmaStages = 3;
constexpr int kTileBytes = NB * NB * sizeof(double);

__global__ void __launch_bounds__((kSolveWarps + 1) * 32) k_inv_apply_tma(
    const double* __restrict__ P, const long long* __restrict__ poff, const double* const* __restrict__ dense,
    const int* __restrict__ set_ptr, const int* __restrict__ set_idx, const double* __restrict__ v,
    const int* __restrict__ mult, const int* __restrict__ owner, int kind, int transpose, int nbmax,
    double* __restrict__ z, long long zhalf, const int* __restrict__ live, const int* __restrict__ order) {
  if (live && *live != 0) return;
  extern __shared__ __align__(128) double tsm[];
  double* ring = tsm;                                      // kTmaStages x 64 x 64
  double* g = ring + kTmaStages * NB * NB;                 // nbmax * 64
  double* y = g + static_cast<size_t>(nbmax) * NB;         // nbmax * 64
  double* scr = y + static_cast<size_t>(nbmax) * NB;       // kSolveWarps x 64 (block-row flush)
  __shared__ __align__(8) uint64_t full[kTmaStages], empty[kTmaStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bi = blockIdx.x >> 1, h = blockIdx.x & 1;
  const int i = order ? order[bi] : bi;
  const int s0 = set_ptr[i], n = set_ptr[i + 1] - s0, nb = (n + NB - 1) / NB;
  const double* D = dense[i];
  double* zo = z + static_cast<long long>(h) * zhalf;
  for (int q = threadIdx.x; q < nb * NB; q += blockDim.x) {
    double val = 0.0;
    if (q < n) {
      const int col = set_idx[s0 + q];
      val = v[col];
      if (transpose) {
        if (kind == RDD_PRECOND_SAS) val /= mult[col];
        else if (kind == RDD_PRECOND_RAS) val = owner[col] == i ? val : 0.0;
      }
    }
    g[q] = val;
    y[q] = 0.0;
  }
  if (threadIdx.x == 0) {
    for (int b = 0; b < kTmaStages; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], kSolveWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (D) {  // eigen-fallback block: dense pseudo-inverse, one CTA
    for (int r = threadIdx.x; r < n; r += blockDim.x) {
      double acc = 0.0;
      if (h == 0)
        for (int q = 0; q < n; ++q) acc += D[r + static_cast<long long>(q) * n] * g[q];
      zo[s0 + r] = acc;
    }
    return;
  }
  const int T = nb * (nb + 1) / 2;
  const double* Pi = P + poff[i];
  if (warp == kSolveWarps) {  // producer
    if (lane == 0) {
      int it = 0, pk = 0, pj = h;  // tile t = pk(pk+1)/2 + pj
      while (pj > pk) {
        pj -= pk + 1;
        ++pk;
      }
      for (int t = h; t < T; t += 2, ++it) {
        const int b = it % kTmaStages;
        if (it >= kTmaStages) mbar_wait(&empty[b], ((it / kTmaStages) - 1) & 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t bytes = static_cast<uint32_t>(NB * inv_tile_ld(n, pk) * sizeof(double));
        mbar_expect_tx(&full[b], bytes);
        bulk_load(ring + b * NB * NB, Pi + inv_tile_off(n, pk, pj), bytes, &full[b]);
        pj += 2;
        while (pj > pk && pk < nb) {
          pj -= pk + 1;
          ++pk;
        }
      }
    }
    return;
  }
  // consumers: warp takes columns [8w, 8w + 8) of every tile; lane holds rows 2l, 2l + 1
  int k = 0, j = h;
  while (j > k) {
    j -= k + 1;
    ++k;
  }
  double a0 = 0.0, a1 = 0.0;
  int it = 0;
  for (int t = h; t < T; t += 2, ++it) {
    const int b = it % kTmaStages;
    mbar_wait(&full[b], (it / kTmaStages) & 1);
    const double* tile = ring + b * NB * NB;
    const int ld = inv_tile_ld(n, k);      // rows stored per tile column (the last block row is trimmed)
    const bool rv = 2 * lane < ld;
    const double gk0 = g[k * NB + 2 * lane], gk1 = g[k * NB + 2 * lane + 1];
    double p[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int col = warp * 8 + c;
      double2 a = make_double2(0.0, 0.0);
      if (rv) a = reinterpret_cast<const double2*>(tile + col * ld)[lane];
      const double gc = g[j * NB + col];
      a0 += a.x * gc;
      a1 += a.y * gc;
      p[c] = a.x * gk0 + a.y * gk1;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[b]);  // the tile is in registers
    if (j < k) {  // y_j += T_kjᵀ g_k: fold 32 lanes to 8, then an 8-lane transpose butterfly
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        p[c] += __shfl_xor_sync(0xffffffffu, p[c], 16);
        p[c] += __shfl_xor_sync(0xffffffffu, p[c], 8);
      }
#pragma unroll
      for (int o = 4; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int q = 0; q < o; ++q) {
          const double send = up ? p[q] : p[q + o];
          const double keep = up ? p[q + o] : p[q];
          p[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      if (lane < 8) y[j * NB + warp * 8 + lane] += p[0];
    }
    // next tile of this CTA; flush the row partials when the block row changes
    int nk = k, nj = j + 2;
    while (nj > nk && nk < nb) {
      nj -= nk + 1;
      ++nk;
    }
    if (nk != k || t + 2 >= T) {
      scr[warp * NB + 2 * lane] = a0;
      scr[warp * NB + 2 * lane + 1] = a1;
      asm volatile("bar.sync 1, %0;" ::"r"(kSolveWarps * 32) : "memory");
      if (threadIdx.x < NB) {
        double s = 0.0;
        for (int w = 0; w < kSolveWarps; ++w) s += scr[w * NB + threadIdx.x];
        y[k * NB + threadIdx.x] += s;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(kSolveWarps * 32) : "memory");
      a0 = a1 = 0.0;
    }
    k = nk;
    j = nj;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(kSolveWarps * 32) : "memory");
  for (int r = threadIdx.x; r < n; r += kSolveWarps * 32) zo[s0 + r] = y[r];
}

size_t inv_apply_tma_smem(int nmax) {
  const size_t len = static_cast<size_t>(ceil_div(nmax, NB)) * NB;
  return (static_cast<size_t>(kTmaStages) * NB * NB + 2 * len + kSolveWarps * NB) * sizeof(double);
}

void chol_apply(Ctx& c, const double* v, bool transpose, double* zloc) {
  if (c.inv_mode) {
    const size_t tsm = inv_apply_tma_smem(c.nmax_local);
    ensure_smem_attr(reinterpret_cast<const void*>(k_inv_apply_tma), tsm);
    k_inv_apply_tma<<<2 * c.J, (kSolveWarps + 1) * 32, tsm, c.stream>>>(
        c.P.p, c.dP_off.p, c.dfb_ptr.p, c.dset_ptr.p, c.dset_idx.p, v, c.dmult.p, c.downer.p, c.pkind, transpose ? 1 : 0,
        ceil_div(c.nmax_local, NB), zloc, static_cast<long long>(c.set_idx.size()), c.live, c.apply_order.p);
    RDD_LAUNCH_CHECK();
    return;
  }
  const size_t smem = chol_solve_smem(c.nmax_local, false);
  ensure_smem_attr(reinterpret_cast<const void*>(k_chol_apply), smem);
  k_chol_apply<<<c.J, kSolveWarps * 32, smem, c.stream>>>(
      c.P.p, c.dP_off.p, c.dfb_ptr.p, c.dset_ptr.p, c.dset_idx.p, v, c.dmult.p, c.downer.p, c.pkind, transpose ? 1 : 0,
      ceil_div(c.nmax_local, NB), zloc, c.live, c.apply_order.p, c.denv_off.p, c.denv_first.p, c.denv_base.p);
  RDD_LAUNCH_CHECK();
}


// ---- RAS owner-row panels (schwarz.hpp:170-182): RAS adds only the entries of z_i = A_i⁻¹ g_i whose
// column subdomain i owns — block i's own p_i columns, a contiguous run (own_off, own_n) of S_i — so
// the apply needs only those p_i rows of A_i⁻¹: a p_i x n_i panel instead of the n_i² /2 inverse
// (2/9 of the bytes in 2-D, 2/27 in 3-D). The transpose needs the same panel: the RAS weights in
// front of the local solve zero every entry but the owned ones, and A_i⁻¹ is symmetric.
namespace {

__global__ void k_ras_panel(const double* __restrict__ P, const long long* __restrict__ poff,
                            const double* const* __restrict__ dense, const int* __restrict__ set_ptr,
                            const int* __restrict__ own_off, const int* __restrict__ own_n,
                            const long long* __restrict__ ras_off, double* __restrict__ R) {
  const int i = blockIdx.x;
  const int n = set_ptr[i + 1] - set_ptr[i], o = own_off[i], pr = own_n[i];
  const double* Pi = P + poff[i];
  const double* D = dense[i];
  double* Ri = R + ras_off[i];
  for (long long e = threadIdx.x; e < static_cast<long long>(pr) * n; e += blockDim.x) {
    const int r = static_cast<int>(e % pr), cc = static_cast<int>(e / pr);
    int a = o + r, b = cc;
    double v;
    if (D) {
      v = D[a + static_cast<long long>(b) * n];
    } else {
      if (a / NB < b / NB) {  // upper tiles are not stored: A_i⁻¹ is symmetric
        const int t = a;
        a = b;
        b = t;
      }
      const int tk = a / NB, tj = b / NB;  // packed explicit inverse (inv_tile_off / inv_tile_ld)
      v = (Pi + inv_tile_off(n, tk, tj))[(a % NB) + (b % NB) * inv_tile_ld(n, tk)];
    }
    Ri[e] = v;
  }
}

// factor mode: the panel is the transpose of X = A_i⁻¹ E_own (n_i x p_i, solved by ras_factor_solves):
// R[r, c] = X[c, r]; eigen-fallback blocks read their dense pseudo-inverse. 32 x 32 transposes
// through shared memory (both sides coalesced)
__global__ void k_ras_panel_x(const double* __restrict__ X, const long long* __restrict__ xoff,
                              const int* __restrict__ ldx, const double* const* __restrict__ dense,
                              const int* __restrict__ set_ptr, const int* __restrict__ own_off,
                              const int* __restrict__ own_n, const long long* __restrict__ ras_off,
                              double* __restrict__ R) {
  __shared__ double tile[32][33];
  const int i = blockIdx.y;
  const int n = set_ptr[i + 1] - set_ptr[i], o = own_off[i], pr = own_n[i];
  const double* D = dense[i];
  double* Ri = R + ras_off[i];
  const double* Xi = X + xoff[i];
  const int ld = ldx[i];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, ny = blockDim.x >> 5;
  const int ctiles = (n + 31) / 32, rtiles = (pr + 31) / 32;
  for (int t = blockIdx.x; t < ctiles * rtiles; t += gridDim.x) {
    const int c0 = (t % ctiles) * 32, r0 = (t / ctiles) * 32;
    for (int y = ty; y < 32; y += ny) {  // read X[c0 + tx, r0 + y] (or D[o + r, c])
      const int cc = c0 + tx, r = r0 + y;
      double v = 0.0;
      if (cc < n && r < pr) v = D ? D[(o + r) + static_cast<long long>(cc) * n] : Xi[cc + static_cast<long long>(r) * ld];
      tile[y][tx] = v;
    }
    __syncthreads();
    for (int y = ty; y < 32; y += ny) {  // write R[r0 + tx, c0 + y]
      const int r = r0 + tx, cc = c0 + y;
      if (r < pr && cc < n) Ri[r + static_cast<long long>(cc) * pr] = tile[tx][y];
    }
    __syncthreads();
  }
}
__global__ void k_ras_unit_rhs(double* __restrict__ X, const long long* __restrict__ xoff, const int* __restrict__ ldx,
                               const int* __restrict__ own_off, const int* __restrict__ own_n) {
  const int i = blockIdx.x;
  for (int r = threadIdx.x; r < own_n[i]; r += blockDim.x)
    X[xoff[i] + (own_off[i] + r) + static_cast<long long>(r) * ldx[i]] = 1.0;
}

constexpr int kRasRows = 4;  // row chunks of 32 per lane pass (128 rows; larger panels loop)

template <bool TR>
__global__ void __launch_bounds__(256) k_ras_apply(const double* __restrict__ R, const long long* __restrict__ ras_off,
                                                   const int* __restrict__ set_ptr, const int* __restrict__ set_idx,
                                                   const int* __restrict__ own_off, const int* __restrict__ own_n,
                                                   const double* __restrict__ v, double* __restrict__ z,
                                                   const int* __restrict__ live, const int* __restrict__ order) {
  if (live && *live != 0) return;
  extern __shared__ double sm[];
  const int i = order ? order[blockIdx.x] : blockIdx.x;
  const int s0 = set_ptr[i], n = set_ptr[i + 1] - s0, o = own_off[i], pr = own_n[i];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* Ri = R + ras_off[i];
  double* g = sm;
  if (!TR) {  // z_i[owned] = panel · v[S_i]: lanes over rows (coalesced columns), warps over columns
    for (int q = threadIdx.x; q < n; q += blockDim.x) g[q] = v[set_idx[s0 + q]];
    __syncthreads();
    double* part = g + n;  // 8 x pr per-warp partials
    for (int r0 = 0; r0 < pr; r0 += 32 * kRasRows) {
      double acc[kRasRows];
#pragma unroll
      for (int k = 0; k < kRasRows; ++k) acc[k] = 0.0;
#pragma unroll 4
      for (int cc = warp; cc < n; cc += 8) {
        const double gc = g[cc];
        const double* col = Ri + static_cast<long long>(cc) * pr;
#pragma unroll
        for (int k = 0; k < kRasRows; ++k) {
          const int r = r0 + lane + 32 * k;
          if (r < pr) acc[k] += col[r] * gc;
        }
      }
#pragma unroll
      for (int k = 0; k < kRasRows; ++k) {
        const int r = r0 + lane + 32 * k;
        if (r < pr) part[warp * pr + r] = acc[k];
      }
    }
    __syncthreads();
    for (int r = threadIdx.x; r < pr; r += blockDim.x) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += part[w * pr + r];
      z[s0 + o + r] = t;
    }
  } else {  // z_i = panelᵀ · v[owned] (the RAS transpose weights keep only the owned entries)
    for (int r = threadIdx.x; r < pr; r += blockDim.x) g[r] = v[set_idx[s0 + o + r]];
    __syncthreads();
    for (int cc = warp; cc < n; cc += 8) {
      double acc = 0.0;
      for (int r = lane; r < pr; r += 32) acc += Ri[r + static_cast<long long>(cc) * pr] * g[r];
      for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (lane == 0) z[s0 + cc] = acc;
    }
  }
}

}  // namespace

// X_i = A_i⁻¹ E_own for every factor-path subdomain, E_own the identity columns of the owned run:
// the forward and backward triangular solves of all p_i right-hand sides as batched DMMA products
// over the envelope-packed factor. A block row of the packing is a contiguous 64 x 64·(k − first_k)
// column-major matrix (lda = 64), so the forward step k is Y_k = D_k (E_k − L[k, first:k] Y[first:k])
// (one NN product per subdomain and step, then the in-place product with D_k = L_kk⁻¹), and the
// backward pass is row-wise like the apply's: X_i = D_iᵀ Y_i, then Y[first:i] −= L[i, first:i]ᵀ X_i
// (TN products). Rows above the owned run stay zero in the forward pass and are skipped.
static void ras_factor_solves(Ctx& c, const std::vector<int>& oo, const std::vector<int>& on, double* X,
                              const std::vector<long long>& xoff, const std::vector<int>& ldx,
                              const std::vector<double*>& dense) {
  const int J = static_cast<int>(oo.size());
  int nbmax = 0;
  for (int i = 0; i < J; ++i) nbmax = std::max(nbmax, ldx[i] / NB);
  auto tile = [&](int i, int k, int j) {  // tile (k, j) of subdomain i's packed factor
    return c.P.p + c.P_off[i] + static_cast<long long>(c.env_base[c.env_off[i] + k] + j) * (NB * NB);
  };
  std::vector<GemmTask> ta, tb;
  for (int k = 0; k < nbmax; ++k) {  // forward
    ta.clear();
    tb.clear();
    for (int i = 0; i < J; ++i) {
      if (dense[i] || k >= ldx[i] / NB || k < oo[i] / NB) continue;
      const int j0 = std::max(c.env_first[c.env_off[i] + k], oo[i] / NB);  // Y_j = 0 above the owned run
      double* Wk = X + xoff[i] + static_cast<long long>(k) * NB;
      for (int tn = 0; tn < ceil_div(on[i], NB); ++tn) {
        if (k > j0)
          ta.push_back({tile(i, k, j0), X + xoff[i] + static_cast<long long>(j0) * NB, Wk, nullptr, nullptr, NB, on[i],
                        NB * (k - j0), NB, ldx[i], ldx[i], 0, tn, 1.0, -1.0});
        tb.push_back({tile(i, k, k), Wk, Wk, nullptr, nullptr, NB, on[i], NB, NB, ldx[i], ldx[i], 0, tn, 0.0, 1.0});
      }
    }
    gemm_nn(c, ta);
    gemm_nn(c, tb);  // in place: a CTA reads its whole 64-row column tile before its epilogue writes it
  }
  for (int k = nbmax - 1; k >= 0; --k) {  // backward, row by row
    ta.clear();
    tb.clear();
    for (int i = 0; i < J; ++i) {
      if (dense[i] || k >= ldx[i] / NB) continue;
      const int j0 = c.env_first[c.env_off[i] + k];
      double* Wk = X + xoff[i] + static_cast<long long>(k) * NB;
      for (int tn = 0; tn < ceil_div(on[i], NB); ++tn) {
        tb.push_back({tile(i, k, k), Wk, Wk, nullptr, nullptr, NB, on[i], NB, NB, ldx[i], ldx[i], 0, tn, 0.0, 1.0});
        for (int tm = 0; tm < k - j0; ++tm)
          ta.push_back({tile(i, k, j0), Wk, X + xoff[i] + static_cast<long long>(j0) * NB, nullptr, nullptr, NB * (k - j0),
                        on[i], NB, NB, ldx[i], ldx[i], tm, tn, 1.0, -1.0});
      }
    }
    gemm_tn(c, tb);  // X_k = D_kᵀ Y_k, in place
    gemm_tn(c, ta);  // Y[first:k] -= L[k, first:k]ᵀ X_k
  }
}

void build_ras_panels(Ctx& c) {
  c.ras_panel = false;
  if (c.pkind != RDD_PRECOND_RAS) return;
  ScopedKernelTimer tk(c, "ras_panels");
  const int J = static_cast<int>(c.set_ptr.size()) - 1;
  std::vector<int> oo(J), on(J);
  c.ras_off.assign(J + 1, 0);
  for (int i = 0; i < J; ++i) {
    int first = -1, cnt = 0, last = -2;
    for (int q = c.set_ptr[i]; q < c.set_ptr[i + 1]; ++q)
      if (c.h_owner[c.set_idx[q]] == i) {
        const int pos = q - c.set_ptr[i];
        if (first < 0) first = pos;
        if (last >= 0 && pos != last + 1) return;  // not contiguous: keep the full local solves
        last = pos;
        ++cnt;
      }
    oo[i] = first < 0 ? 0 : first;
    on[i] = cnt;
    c.ras_off[i + 1] = c.ras_off[i] + static_cast<long long>(cnt) * (c.set_ptr[i + 1] - c.set_ptr[i]);
  }
  c.down_off.upload(oo, c.stream);
  c.down_n.upload(on, c.stream);
  c.dras_off.upload(c.ras_off, c.stream);
  c.Pras.ensure(static_cast<size_t>(std::max<long long>(1, c.ras_off[J])));
  if (c.inv_mode) {
    k_ras_panel<<<J, 256, 0, c.stream>>>(c.P.p, c.dP_off.p, c.dfb_ptr.p, c.dset_ptr.p, c.down_off.p, c.down_n.p,
                                         c.dras_off.p, c.Pras.p);
    RDD_LAUNCH_CHECK();
  } else {
    // factor mode (large blocks): solve for the owned right-hand sides once, keep the panel
    std::vector<long long> xoff(J + 1, 0);
    std::vector<int> ldx(J);
    std::vector<double*> dense(J, nullptr);
    for (int i = 0; i < J; ++i) {
      ldx[i] = ceil_div(c.local_n[i], NB) * NB;
      auto it = c.fb_store.find(i);
      if (it != c.fb_store.end()) dense[i] = it->second.p;
      xoff[i + 1] = xoff[i] + (dense[i] ? 0 : static_cast<long long>(ldx[i]) * on[i]);
    }
    double* X = c.ws("ras.X", static_cast<size_t>(std::max<long long>(1, xoff[J])));
    RDD_CUDA(cudaMemsetAsync(X, 0, sizeof(double) * static_cast<size_t>(xoff[J]), c.stream));
    DBuf<long long> dxoff;
    DBuf<int> dldx;
    dxoff.upload(xoff, c.stream);
    dldx.upload(ldx, c.stream);
    std::vector<int> on_f(on);
    for (int i = 0; i < J; ++i)
      if (dense[i]) on_f[i] = 0;  // no unit columns for the dense blocks (no X storage)
    DBuf<int> don_f;
    don_f.upload(on_f, c.stream);
    k_ras_unit_rhs<<<J, 256, 0, c.stream>>>(X, dxoff.p, dldx.p, c.down_off.p, don_f.p);
    RDD_LAUNCH_CHECK();
    ras_factor_solves(c, oo, on, X, xoff, ldx, dense);
    k_ras_panel_x<<<dim3(64, J), 256, 0, c.stream>>>(X, dxoff.p, dldx.p, c.dfb_ptr.p, c.dset_ptr.p, c.down_off.p,
                                                    c.down_n.p, c.dras_off.p, c.Pras.p);
    RDD_LAUNCH_CHECK();
  }
  RDD_CUDA(cudaStreamSynchronize(c.stream));
  c.ras_panel = true;
}

void ras_panel_apply(Ctx& c, const double* v, bool transpose, double* zloc) {
  int pmax = 0;
  for (int j = 0; j < c.J; ++j) pmax = std::max(pmax, c.h_p[j]);
  const size_t smem = static_cast<size_t>(c.nmax_local + 8 * pmax) * sizeof(double);
  if (transpose) {
    ensure_smem_attr(reinterpret_cast<const void*>(k_ras_apply<true>), smem);
    k_ras_apply<true><<<c.J, 256, smem, c.stream>>>(c.Pras.p, c.dras_off.p, c.dset_ptr.p, c.dset_idx.p, c.down_off.p,
                                                   c.down_n.p, v, zloc, c.live, c.apply_order.p);
  } else {
    ensure_smem_attr(reinterpret_cast<const void*>(k_ras_apply<false>), smem);
    k_ras_apply<false><<<c.J, 256, smem, c.stream>>>(c.Pras.p, c.dras_off.p, c.dset_ptr.p, c.dset_idx.p, c.down_off.p,
                                                    c.down_n.p, v, zloc, c.live, c.apply_order.p);
  }
  RDD_LAUNCH_CHECK();
}

}  // namespace rdd
