// matvec.cu — K6 column equilibration and K9/K10 block-sparse H·w, Hᵀ·r.
//
// H·w (assembly.hpp:110-121) scatter-adds each block's rows into y; here each global row is
// owned by one thread that gathers the ≤2^d covering blocks' rows (owner-computes, no atomics;
// the per-row sum visits blocks in ascending j like the reference). Hᵀ·r (assembly.hpp:123-133)
// is one warp per column: a contiguous column of a column-major block against r gathered through
// rows_j. Both are HBM-bound streams over H (8·nnz bytes each).
#include <algorithm>

#include "ctx.hpp"

namespace rdd {

namespace {

// one warp per column: 2-norm, zero -> 1 (runner.hpp:96-99), then H col /= s (assembly.hpp:197-204)
__global__ void k_colnorm_scale(double* __restrict__ H, const long long* __restrict__ H_off,
                                const int* __restrict__ row_ptr, const int* __restrict__ col_off,
                                const int* __restrict__ col_owner, int p, double* __restrict__ scales, int apply) {
  const int col = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (col >= p) return;
  const int j = col_owner[col];
  const int k = col - col_off[j];
  const int rows = row_ptr[j + 1] - row_ptr[j];
  double* h = H + H_off[j] + static_cast<long long>(k) * rows;
  double s = 0.0;
  for (int r = lane; r < rows; r += 32) s += h[r] * h[r];
  s = sqrt(warp_sum(s));
  if (s == 0.0) s = 1.0;
  if (!apply) s = 1.0;
  if (lane == 0) scales[col] = s;
  if (apply && s != 1.0)
    for (int r = lane; r < rows; r += 32) h[r] = h[r] / s;
}

__global__ void k_matvec(const double* __restrict__ H, const long long* __restrict__ H_off,
                         const int* __restrict__ row_ptr, const int* __restrict__ col_off,
                         const int* __restrict__ cov_n, const int* __restrict__ cov_j, const int* __restrict__ cov_r,
                         int maxcov, int N, const double* __restrict__ w, double* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  double acc = 0.0;
  const int nc = cov_n[i];
  for (int s = 0; s < nc; ++s) {
    const int j = cov_j[static_cast<size_t>(i) * maxcov + s];
    const int r = cov_r[static_cast<size_t>(i) * maxcov + s];
    const int rows = row_ptr[j + 1] - row_ptr[j];
    const int c0 = col_off[j], pj = col_off[j + 1] - c0;
    const double* h = H + H_off[j] + r;
    double t = 0.0;
    for (int k = 0; k < pj; ++k) t += h[static_cast<long long>(k) * rows] * w[c0 + k];
    acc += t;
  }
  y[i] = acc;
}

__global__ void k_matvec_t(const double* __restrict__ H, const long long* __restrict__ H_off,
                           const int* __restrict__ row_ptr, const int* __restrict__ row_idx,
                           const int* __restrict__ col_off, const int* __restrict__ col_owner, int p,
                           const double* __restrict__ r, double* __restrict__ out) {
  const int col = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (col >= p) return;
  const int j = col_owner[col];
  const int k = col - col_off[j];
  const int r0 = row_ptr[j], rows = row_ptr[j + 1] - r0;
  const double* h = H + H_off[j] + static_cast<long long>(k) * rows;
  double s = 0.0;
  for (int q = lane; q < rows; q += 32) s += h[q] * r[row_idx[r0 + q]];
  s = warp_sum(s);
  if (lane == 0) out[col] = s;
}

}  // namespace

void ensure_col_owner(Ctx& c) {
  std::vector<int> own(c.p);
  for (int j = 0; j < c.J; ++j)
    for (int k = c.h_col_off[j]; k < c.h_col_off[j + 1]; ++k) own[k] = j;
  c.h_owner = own;
  c.downer.upload(own, c.stream);
}

void column_norms_scale(Ctx& c, bool equilibrate) {
  ScopedKernelTimer tk(c, "equilibrate");
  c.scales.ensure(std::max(1, c.p));
  const int threads = 256;
  k_colnorm_scale<<<ceil_div(static_cast<long long>(c.p) * 32, threads), threads, 0, c.stream>>>(
      c.H, c.dH_off.p, c.row_ptr.p, c.dcol_off.p, c.downer.p, c.p, c.scales.p, equilibrate ? 1 : 0);
  RDD_LAUNCH_CHECK();
}

void matvec_dev(Ctx& c, const double* w, double* y) {
  ScopedKernelTimer tk(c, "matvec");
  k_matvec<<<ceil_div(c.N, 256), 256, 0, c.stream>>>(c.H, c.dH_off.p, c.row_ptr.p, c.dcol_off.p, c.cov_n.p, c.cov_j.p,
                                                     c.cov_r.p, c.maxcov, c.N, w, y);
  RDD_LAUNCH_CHECK();
}

void matvec_t_dev(Ctx& c, const double* r, double* out) {
  ScopedKernelTimer tk(c, "matvec_t");
  k_matvec_t<<<ceil_div(static_cast<long long>(c.p) * 32, 256), 256, 0, c.stream>>>(
      c.H, c.dH_off.p, c.row_ptr.p, c.row_idx.p, c.dcol_off.p, c.downer.p, c.p, r, out);
  RDD_LAUNCH_CHECK();
}

}  // namespace rdd

// ============================================================================================
// Fused single-pass normal operator out = Hᵀ(H·w) (runner.hpp:232-234 computes it as two passes,
// assembly.hpp:110-133). Global rows are cut into tiles of kFT consecutive points; a CTA gathers
// the rows of every covering block for its tile (each H element belongs to exactly one tile, so
// HBM reads H once), forms y = H·w for the tile in shared memory in the reference's per-row order
// (ascending covering block), then re-reads the same (now L2-resident) rows to accumulate
// Hᵀy per (tile, block) into a partial buffer. A second kernel sums the partials of each block in
// tile order: deterministic, no atomics.
// ============================================================================================
namespace rdd {
namespace {

constexpr int kFT = 128;     // points per tile
constexpr int kFSlots = 32;  // distinct blocks per tile (plan falls back to two passes beyond)

struct FusedArgs {
  const double* H;
  const long long* H_off;
  const int* row_ptr;
  const int* col_off;
  const int* cov_n;
  const int* cov_j;
  const int* cov_r;
  int maxcov, N;
  const int* tile_blk;        // ntiles x kFSlots block ids (-1 unused)
  const long long* tile_poff; // ntiles x kFSlots partial offsets
  const double* w;
  double* part;
};

__global__ void __launch_bounds__(256) k_fused_normal(FusedArgs A) {
  extern __shared__ double fsm[];
  const int MC = A.maxcov;
  double* yparts = fsm;                          // MC x kFT (cover-major)
  double* y = yparts + kFT * MC;                 // kFT
  int* pslot = reinterpret_cast<int*>(y + kFT);  // MC x kFT slot of each cover (-1 none)
  int* prow = pslot + kFT * MC;                  // MC x kFT local row
  int* lst = prow + kFT * MC;                    // per-slot compact lists: packed (t | c << 16), kFT*MC total
  __shared__ int s_blk[kFSlots], s_c0[kFSlots], s_pj[kFSlots], s_rows[kFSlots], s_lo[kFSlots], s_len[kFSlots];
  __shared__ long long s_hoff[kFSlots], s_poff[kFSlots];
  __shared__ int s_ns;
  const int tile = blockIdx.x;
  const int i0 = tile * kFT;
  if (threadIdx.x == 0) s_ns = 0;
  __syncthreads();
  if (threadIdx.x < kFSlots) {
    const int b = A.tile_blk[static_cast<long long>(tile) * kFSlots + threadIdx.x];
    s_blk[threadIdx.x] = b;
    if (b >= 0) {
      s_c0[threadIdx.x] = A.col_off[b];
      s_pj[threadIdx.x] = A.col_off[b + 1] - A.col_off[b];
      s_rows[threadIdx.x] = A.row_ptr[b + 1] - A.row_ptr[b];
      s_hoff[threadIdx.x] = A.H_off[b];
      s_poff[threadIdx.x] = A.tile_poff[static_cast<long long>(tile) * kFSlots + threadIdx.x];
      atomicMax(&s_ns, threadIdx.x + 1);
    }
  }
  __syncthreads();
  const int ns = s_ns;
  // covers of the tile's points -> (slot, local row); cover-major so a warp walks consecutive points
  for (int e = threadIdx.x; e < kFT * MC; e += blockDim.x) {
    const int c = e / kFT, t = e % kFT;
    const int i = i0 + t;
    int slot = -1, r = 0;
    if (i < A.N && c < A.cov_n[i]) {
      const int b = A.cov_j[static_cast<long long>(i) * MC + c];
      r = A.cov_r[static_cast<long long>(i) * MC + c];
      for (int s = 0; s < ns; ++s)
        if (s_blk[s] == b) slot = s;
    }
    pslot[e] = slot;
    prow[e] = r;
  }
  __syncthreads();
  // y partials, one thread per (cover, point): coalesced along consecutive points
  for (int e = threadIdx.x; e < kFT * MC; e += blockDim.x) {
    const int s = pslot[e];
    double acc = 0.0;
    if (s >= 0) {
      const double* h = A.H + s_hoff[s] + prow[e];
      const double* ww = A.w + s_c0[s];
      const int rows = s_rows[s], pj = s_pj[s];
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int k = 0;
      for (; k + 4 <= pj; k += 4) {
        a0 += __ldg(h + static_cast<long long>(k) * rows) * ww[k];
        a1 += __ldg(h + static_cast<long long>(k + 1) * rows) * ww[k + 1];
        a2 += __ldg(h + static_cast<long long>(k + 2) * rows) * ww[k + 2];
        a3 += __ldg(h + static_cast<long long>(k + 3) * rows) * ww[k + 3];
      }
      for (; k < pj; ++k) a0 += __ldg(h + static_cast<long long>(k) * rows) * ww[k];
      acc = (a0 + a1) + (a2 + a3);
    }
    yparts[e] = acc;
  }
  // per-slot compact (point, cover) lists in ascending point order (warp ballot: deterministic)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (threadIdx.x < kFT) {
    double acc = 0.0;
    for (int c = 0; c < MC; ++c) acc += yparts[c * kFT + threadIdx.x];  // covers in ascending block order
    y[threadIdx.x] = acc;
  }
  for (int s = warp; s < ns; s += nw) {  // per-slot counts
    int cnt = 0;
    for (int e = lane; e < kFT * MC; e += 32) cnt += __popc(__ballot_sync(0xffffffffu, pslot[e] == s)) * (lane == 0);
    if (lane == 0) s_len[s] = cnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int lo = 0;
    for (int s = 0; s < ns; ++s) {
      s_lo[s] = lo;
      lo += s_len[s];
    }
  }
  __syncthreads();
  for (int s = warp; s < ns; s += nw) {
    int pos = s_lo[s];
    for (int t0 = 0; t0 < kFT; t0 += 32) {
      for (int c = 0; c < MC; ++c) {
        const int e = c * kFT + t0 + lane;
        const bool hit = pslot[e] == s;
        const unsigned m = __ballot_sync(0xffffffffu, hit);
        if (hit) lst[pos + __popc(m & ((1u << lane) - 1u))] = (t0 + lane) | (c << 16);
        pos += __popc(m);
      }
    }
  }
  __syncthreads();
  // Hᵀy partials: warp per (slot, column); lanes walk the slot's list (coalesced, L2-resident)
  int total = 0;
  for (int s = 0; s < ns; ++s) total += s_pj[s];
  for (int q = warp; q < total; q += nw) {
    int s = 0, k = q;
    while (k >= s_pj[s]) {
      k -= s_pj[s];
      ++s;
    }
    const double* hcol = A.H + s_hoff[s] + static_cast<long long>(k) * s_rows[s];
    const int* L = lst + s_lo[s];
    const int len = s_len[s];
    double acc = 0.0;
    for (int l = lane; l < len; l += 32) {
      const int v = L[l];
      const int t = v & 0xffff, c = v >> 16;
      acc += __ldg(hcol + prow[c * kFT + t]) * y[t];
    }
    acc = warp_sum(acc);
    if (lane == 0) A.part[s_poff[s] + k] = acc;
  }
}

// out[col] = Σ_tiles partial(tile, owner(col))[k], tiles in ascending order
__global__ void k_fused_reduce(const double* __restrict__ part, const int* __restrict__ bptr,
                               const long long* __restrict__ bparts, const int* __restrict__ col_off,
                               const int* __restrict__ col_owner, int p, double* __restrict__ out) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= p) return;
  const int j = col_owner[col];
  const int k = col - col_off[j];
  double s = 0.0;
  for (int q = bptr[j]; q < bptr[j + 1]; ++q) s += part[bparts[q] + k];
  out[col] = s;
}

}  // namespace

// Tile plan for the fused operator (once per assembled system): distinct covering blocks per
// tile, partial-buffer offsets, and per-block partial lists in tile order.
bool build_fused_plan(Ctx& c) {
  const int N = c.N, MC = c.maxcov, J = c.J;
  const int ntiles = ceil_div(N, kFT);
  std::vector<int> cn(N), cj(static_cast<size_t>(N) * MC);
  c.cov_n.download(cn.data(), N, c.stream);
  c.cov_j.download(cj.data(), cj.size(), c.stream);
  RDD_CUDA(cudaStreamSynchronize(c.stream));
  std::vector<int> tb(static_cast<size_t>(ntiles) * kFSlots, -1);
  std::vector<long long> tp(static_cast<size_t>(ntiles) * kFSlots, -1);
  std::vector<std::vector<long long>> per_block(J);
  long long off = 0;
  for (int t = 0; t < ntiles; ++t) {
    int ns = 0;
    int* slots = &tb[static_cast<size_t>(t) * kFSlots];
    for (int i = t * kFT; i < std::min(N, (t + 1) * kFT); ++i)
      for (int q = 0; q < cn[i]; ++q) {
        const int b = cj[static_cast<size_t>(i) * MC + q];
        bool found = false;
        for (int s = 0; s < ns; ++s) found |= slots[s] == b;
        if (!found) {
          if (ns == kFSlots) return false;
          slots[ns++] = b;
        }
      }
    std::sort(slots, slots + ns);
    for (int s = 0; s < ns; ++s) {
      tp[static_cast<size_t>(t) * kFSlots + s] = off;
      per_block[slots[s]].push_back(off);
      off += c.h_p[slots[s]];
    }
  }
  std::vector<int> bptr(J + 1, 0);
  std::vector<long long> bparts;
  for (int j = 0; j < J; ++j) {
    bparts.insert(bparts.end(), per_block[j].begin(), per_block[j].end());
    bptr[j + 1] = static_cast<int>(bparts.size());
  }
  c.f_tile_blk.upload(tb, c.stream);
  c.f_tile_poff.upload(tp, c.stream);
  c.f_bptr.upload(bptr, c.stream);
  c.f_bparts.upload(bparts, c.stream);
  c.f_part.ensure(std::max<long long>(1, off));
  c.f_ntiles = ntiles;
  c.f_part_size = off;
  c.fused_ready = true;
  return true;
}

void fused_normal_apply_dev(Ctx& c, const double* w, double* out) {
  ScopedKernelTimer tk(c, "fused_normal");
  FusedArgs A{};
  A.H = c.H;
  A.H_off = c.dH_off.p;
  A.row_ptr = c.row_ptr.p;
  A.col_off = c.dcol_off.p;
  A.cov_n = c.cov_n.p;
  A.cov_j = c.cov_j.p;
  A.cov_r = c.cov_r.p;
  A.maxcov = c.maxcov;
  A.N = c.N;
  A.tile_blk = c.f_tile_blk.p;
  A.tile_poff = c.f_tile_poff.p;
  A.w = w;
  A.part = c.f_part.p;
  const size_t smem = static_cast<size_t>(kFT) * c.maxcov * (sizeof(double) + 3 * sizeof(int)) + kFT * sizeof(double);
  if (smem > 48 * 1024)
    RDD_CUDA(cudaFuncSetAttribute(k_fused_normal, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  k_fused_normal<<<c.f_ntiles, 256, smem, c.stream>>>(A);
  RDD_LAUNCH_CHECK();
  k_fused_reduce<<<ceil_div(c.p, 256), 256, 0, c.stream>>>(c.f_part.p, c.f_bptr.p, c.f_bparts.p, c.dcol_off.p,
                                                           c.downer.p, c.p, out);
  RDD_LAUNCH_CHECK();
}

}  // namespace rdd
