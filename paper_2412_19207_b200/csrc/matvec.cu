// matvec.cu — K6 column equilibration and K9/K10 block-sparse H·w, Hᵀ·r.
//
// H·w (assembly.hpp:110-121) scatter-adds each block's rows into y; here per-block partial rows
// z_j = H_j w_j are formed tile by tile and each global row then sums its ≤2^d covering blocks'
// partials in ascending j like the reference (owner-computes, no atomics). Hᵀ·r
// (assembly.hpp:123-133) reduces contiguous columns of a column-major block against r gathered
// through rows_j, staged once per (block, column group). Both are HBM-bound streams over H
// (8·nnz bytes each).
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

// H·w in two steps, both in the reference's summation order: (1) per (block j, tile of kMvRows
// local rows), z_j[r] = Σ_k H_j[r, k] w_j[k] (ascending k) with w_j in shared memory and kMvUnroll
// independent column loads in flight per thread; (2) y_i = Σ over the covering blocks of i in
// ascending j of z_j[r_i]. Every warp of step 1 runs the same block: uniform trip counts.
constexpr int kMvRows = 256, kMvUnroll = 8;
__global__ void __launch_bounds__(kMvRows) k_block_gemv(const double* __restrict__ H, const long long* __restrict__ H_off,
                                                         const int* __restrict__ row_ptr, const int* __restrict__ col_off,
                                                         const int2* __restrict__ tiles, const double* __restrict__ w,
                                                         double* __restrict__ z, const int* __restrict__ live) {
  if (live && *live != 0) return;  // solver loop already stopped (speculative graph iteration)
  extern __shared__ double wsm[];
  const int2 t = tiles[blockIdx.x];
  const int j = t.x;
  const int rows = row_ptr[j + 1] - row_ptr[j];
  const int c0 = col_off[j], pj = col_off[j + 1] - c0;
  for (int k = threadIdx.x; k < pj; k += blockDim.x) wsm[k] = w[c0 + k];
  __syncthreads();
  const int r = t.y + threadIdx.x;
  if (r >= rows) return;
  const double* h = H + H_off[j] + r;
  double acc = 0.0;
  int k = 0;
  for (; k + kMvUnroll <= pj; k += kMvUnroll) {
    double v[kMvUnroll];
#pragma unroll
    for (int u = 0; u < kMvUnroll; ++u) v[u] = __ldcs(h + static_cast<long long>(k + u) * rows);
#pragma unroll
    for (int u = 0; u < kMvUnroll; ++u) acc += v[u] * wsm[k + u];
  }
  for (; k < pj; ++k) acc += __ldcs(h + static_cast<long long>(k) * rows) * wsm[k];
  z[row_ptr[j] + r] = acc;
}

__global__ void k_cover_sum(const double* __restrict__ z, const int* __restrict__ row_ptr,
                            const int* __restrict__ cov_n, const int* __restrict__ cov_j, const int* __restrict__ cov_r,
                            int maxcov, int N, double* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  double acc = 0.0;
  const int nc = cov_n[i];
  for (int s = 0; s < nc; ++s) {
    const size_t e = static_cast<size_t>(i) * maxcov + s;
    acc += z[row_ptr[cov_j[e]] + cov_r[e]];
  }
  y[i] = acc;
}

// Hᵀ·r in two steps: (1) per (block j, chunk of kMtRows local rows) the gathered r chunk is staged
// in shared memory and every column of H_j is reduced over the chunk (warps take columns; lanes
// stride the rows, then the butterfly) into a partial; (2) each column sums its chunk partials in
// chunk order. Deterministic, no atomics; the tile count does not depend on p_j, so the grid fills
// the GPU even when blocks are narrow.
// FROM_Z (the normal operator Hᵀ(H·w)): the staged r = (H·w)[rows_j] is formed here from the
// per-block partials z of k_block_gemv through the per-entry cover lists (ascending j, the
// reference's summation order, so identical to k_cover_sum's y) — no y round trip, one launch less.
constexpr int kMtRows = 512, kMtWarps = 8, kMtUnroll = 8;
template <bool FROM_Z, int W>
__global__ void __launch_bounds__(kMtWarps * 32) k_block_gemv_t(const double* __restrict__ H,
                                                                 const long long* __restrict__ H_off,
                                                                 const int* __restrict__ row_ptr,
                                                                 const int* __restrict__ row_idx,
                                                                 const int* __restrict__ col_off,
                                                                 const int2* __restrict__ tiles,
                                                                 const int* __restrict__ part_off,
                                                                 const double* __restrict__ r, double* __restrict__ part,
                                                                 const int* __restrict__ ent_flat,
                                                                 const int* __restrict__ live) {
  if (live && *live != 0) return;
  __shared__ double rsm[kMtRows];
  const int2 t = tiles[blockIdx.x];
  const int j = t.x;
  const int r0 = row_ptr[j], rows = row_ptr[j + 1] - r0;
  const int q0 = t.y, nq = min(kMtRows, rows - q0);
  const int pj = col_off[j + 1] - col_off[j];
  for (int q = threadIdx.x; q < nq; q += blockDim.x) {
    if constexpr (FROM_Z) {
      const int4* f = reinterpret_cast<const int4*>(ent_flat + static_cast<size_t>(r0 + q0 + q) * W);
      int idx[W];
#pragma unroll
      for (int u = 0; u < W / 4; ++u) {
        const int4 v = f[u];
        idx[4 * u] = v.x;
        idx[4 * u + 1] = v.y;
        idx[4 * u + 2] = v.z;
        idx[4 * u + 3] = v.w;
      }
      double zv[W];
#pragma unroll
      for (int u = 0; u < W; ++u) zv[u] = idx[u] >= 0 ? r[idx[u]] : 0.0;
      double s = 0.0;
#pragma unroll
      for (int u = 0; u < W; ++u)
        if (idx[u] >= 0) s += zv[u];
      rsm[q] = s;
    } else {
      rsm[q] = r[row_idx[r0 + q0 + q]];
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* out = part + part_off[blockIdx.x];
  for (int k = warp; k < pj; k += 2 * kMtWarps) {  // two columns per warp: 2·kMtUnroll loads in flight
    const int kb = k + kMtWarps;
    const bool hb = kb < pj;
    const double* ha = H + H_off[j] + static_cast<long long>(k) * rows + q0;
    const double* hbp = H + H_off[j] + static_cast<long long>(hb ? kb : k) * rows + q0;
    double sa = 0.0, sb = 0.0;
    int q = lane;
    for (; q + 32 * (kMtUnroll - 1) < nq; q += 32 * kMtUnroll) {
      double a[kMtUnroll], b[kMtUnroll];
#pragma unroll
      for (int u = 0; u < kMtUnroll; ++u) {
        a[u] = __ldcs(ha + q + 32 * u);
        b[u] = hb ? __ldcs(hbp + q + 32 * u) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kMtUnroll; ++u) {
        sa += a[u] * rsm[q + 32 * u];
        sb += b[u] * rsm[q + 32 * u];
      }
    }
    for (; q < nq; q += 32) {
      sa += ha[q] * rsm[q];
      if (hb) sb += hbp[q] * rsm[q];
    }
    sa = warp_sum(sa);
    sb = warp_sum(sb);
    if (lane == 0) {
      out[k] = sa;
      if (hb) out[kb] = sb;
    }
  }
}

// out[col] = Σ over the row chunks of its block (ascending) of the partials
// (optional) dw/dpart: per-CTA partial of dw·out (the CG's pᵀAp), fixed order
__global__ void __launch_bounds__(256) k_chunk_sum(const double* __restrict__ part, const int* __restrict__ col_owner,
                                                   const int* __restrict__ col_off, const int* __restrict__ blk_tile0,
                                                   const int* __restrict__ part_off, int p, double* __restrict__ out,
                                                   const double* __restrict__ dw, double* __restrict__ dpart,
                                                   const int* __restrict__ live) {
  if (live && *live != 0) return;
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  double s = 0.0;
  if (col < p) {
    const int j = col_owner[col], k = col - col_off[j];
    for (int tt = blk_tile0[j]; tt < blk_tile0[j + 1]; ++tt) s += part[part_off[tt] + k];
    out[col] = s;
  }
  if (dpart) {
    double d = col < p ? dw[col] * s : 0.0;
    d = block_sum_256(d);
    if (threadIdx.x == 0) dpart[blockIdx.x] = d;
  }
}

}  // namespace

// per (block, local row) entry: flat indices into the per-block partials z of the entry's point's
// covering (block, row) pairs, ascending block, padded with -1 to the width W (4 or 8)
__global__ void k_entry_covers(const int* __restrict__ row_idx, const int* __restrict__ row_ptr,
                               const int* __restrict__ cov_n, const int* __restrict__ cov_j,
                               const int* __restrict__ cov_r, int maxcov, long long nent, int W,
                               int* __restrict__ ent_flat) {
  const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (e >= nent) return;
  const int i = row_idx[e], nc = cov_n[i];
  for (int s = 0; s < W; ++s) {
    int v = -1;
    if (s < nc) {
      const size_t q = static_cast<size_t>(i) * maxcov + s;
      v = row_ptr[cov_j[q]] + cov_r[q];
    }
    ent_flat[e * W + s] = v;
  }
}

void ensure_col_owner(Ctx& c) {
  std::vector<int> own(c.p);
  for (int j = 0; j < c.J; ++j)
    for (int k = c.h_col_off[j]; k < c.h_col_off[j + 1]; ++k) own[k] = j;
  c.h_owner = own;
  c.downer.upload(own, c.stream);
  // tile lists of the block-tiled H·w / Hᵀ·r
  std::vector<int2> mv, mt;
  std::vector<int> poff, t0(c.J + 1, 0);
  int rmax = 0, pacc = 0;
  for (int j = 0; j < c.J; ++j) {
    const int rows = c.h_row_ptr[j + 1] - c.h_row_ptr[j];
    rmax = std::max(rmax, rows);
    for (int r = 0; r < rows; r += kMvRows) mv.push_back(make_int2(j, r));
    t0[j] = static_cast<int>(mt.size());
    for (int r = 0; r < rows; r += kMtRows) {
      mt.push_back(make_int2(j, r));
      poff.push_back(pacc);
      pacc += c.h_p[j];
    }
  }
  t0[c.J] = static_cast<int>(mt.size());
  c.mv_ntiles = static_cast<int>(mv.size());
  c.mt_ntiles = static_cast<int>(mt.size());
  c.mv_rmax = rmax;
  c.mv_tiles.upload(mv, c.stream);
  c.mt_tiles.upload(mt, c.stream);
  c.mt_part_off.upload(poff, c.stream);
  c.mt_blk_tile0.upload(t0, c.stream);
  c.mt_part.ensure(std::max(1, pacc));
  c.zrows.ensure(std::max(1, c.h_row_ptr[c.J]));
  // cover lists per entry for the normal operator's fused staging (built once per instance,
  // outside any graph capture)
  c.ent_w = c.maxcov <= 4 ? 4 : 8;
  const long long nent = c.h_row_ptr[c.J];
  if (c.maxcov <= 8 && nent > 0) {
    c.ent_flat.ensure(static_cast<size_t>(nent) * c.ent_w);
    k_entry_covers<<<ceil_div(nent, 256), 256, 0, c.stream>>>(c.row_idx.p, c.row_ptr.p, c.cov_n.p, c.cov_j.p, c.cov_r.p,
                                                              c.maxcov, nent, c.ent_w, c.ent_flat.p);
    RDD_LAUNCH_CHECK();
  } else {
    c.ent_w = 0;
  }
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
  if (c.mv_ntiles > 0) {
    const size_t sm = static_cast<size_t>(c.m) * sizeof(double);
    k_block_gemv<<<c.mv_ntiles, kMvRows, sm, c.stream>>>(c.H, c.dH_off.p, c.row_ptr.p, c.dcol_off.p, c.mv_tiles.p, w,
                                                         c.zrows.p, c.live);
    RDD_LAUNCH_CHECK();
  }
  k_cover_sum<<<ceil_div(c.N, 256), 256, 0, c.stream>>>(c.zrows.p, c.row_ptr.p, c.cov_n.p, c.cov_j.p, c.cov_r.p,
                                                        c.maxcov, c.N, y);
  RDD_LAUNCH_CHECK();
}

void matvec_t_dev(Ctx& c, const double* r, double* out, const double* dot_with, double* dot_part) {
  ScopedKernelTimer tk(c, "matvec_t");
  if (c.mt_ntiles == 0) return;
  k_block_gemv_t<false, 4><<<c.mt_ntiles, kMtWarps * 32, 0, c.stream>>>(
      c.H, c.dH_off.p, c.row_ptr.p, c.row_idx.p, c.dcol_off.p, c.mt_tiles.p, c.mt_part_off.p, r, c.mt_part.p, nullptr, c.live);
  RDD_LAUNCH_CHECK();
  k_chunk_sum<<<ceil_div(c.p, 256), 256, 0, c.stream>>>(c.mt_part.p, c.downer.p, c.dcol_off.p, c.mt_blk_tile0.p,
                                                        c.mt_part_off.p, c.p, out, dot_with, dot_part, c.live);
  RDD_LAUNCH_CHECK();
}

// out = Hᵀ(H·w) in the reference's two passes over H, y = H·w formed inside the Hᵀ staging
void normal_two_pass_dev(Ctx& c, const double* w, double* out, double* dot_part) {
  if (c.ent_w == 0 || c.mt_ntiles == 0) {
    matvec_dev(c, w, c.ytmp.ensure(c.N));
    matvec_t_dev(c, c.ytmp.p, out, dot_part ? w : nullptr, dot_part);
    return;
  }
  ScopedKernelTimer tk(c, "normal_two_pass");
  if (c.mv_ntiles > 0) {
    const size_t sm = static_cast<size_t>(c.m) * sizeof(double);
    k_block_gemv<<<c.mv_ntiles, kMvRows, sm, c.stream>>>(c.H, c.dH_off.p, c.row_ptr.p, c.dcol_off.p, c.mv_tiles.p, w,
                                                         c.zrows.p, c.live);
    RDD_LAUNCH_CHECK();
  }
  if (c.ent_w == 4)
    k_block_gemv_t<true, 4><<<c.mt_ntiles, kMtWarps * 32, 0, c.stream>>>(
        c.H, c.dH_off.p, c.row_ptr.p, c.row_idx.p, c.dcol_off.p, c.mt_tiles.p, c.mt_part_off.p, c.zrows.p, c.mt_part.p,
        c.ent_flat.p, c.live);
  else
    k_block_gemv_t<true, 8><<<c.mt_ntiles, kMtWarps * 32, 0, c.stream>>>(
        c.H, c.dH_off.p, c.row_ptr.p, c.row_idx.p, c.dcol_off.p, c.mt_tiles.p, c.mt_part_off.p, c.zrows.p, c.mt_part.p,
        c.ent_flat.p, c.live);
  RDD_LAUNCH_CHECK();
  k_chunk_sum<<<ceil_div(c.p, 256), 256, 0, c.stream>>>(c.mt_part.p, c.downer.p, c.dcol_off.p, c.mt_blk_tile0.p,
                                                        c.mt_part_off.p, c.p, out, dot_part ? w : nullptr, dot_part, c.live);
  RDD_LAUNCH_CHECK();
}

}  // namespace rdd
