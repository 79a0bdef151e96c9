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

// ============================================================================================
// Fused single-pass normal operator out = Hᵀ(H·w) (runner.hpp:232-234 computes it as two passes
// over H, assembly.hpp:110-133). Global rows are cut into tiles of consecutive points such that,
// for every covering block j ("slot"), the tile's points inside box j are one contiguous range of
// the tile with contiguous local rows of H_j. Each slot column segment is then one contiguous run
// of a column-major block, streamed into shared memory by a 1-D TMA bulk copy (cp.async.bulk,
// mbarrier completion) — H is read from HBM exactly once. A persistent CTA double-buffers tiles:
// while tile t is reduced from shared memory, tile t+grid is in flight. y = H·w is formed per
// point in the reference's order (ascending covering block), then Hᵀy per (tile, slot) goes to a
// partial buffer that a second kernel sums in tile order: deterministic, no atomics.
// ============================================================================================
namespace rdd {
namespace {

constexpr int kFT = 128;                // max points per tile
constexpr int kFSlots = 16;             // max covering blocks per tile
constexpr int kFBuf = 96 * 1024;        // bytes per tile buffer (two buffers per CTA)
constexpr int kFThreads = 512;

struct TileSlot {
  int blk, ta, len, ra;   // block, first point in tile, #points, first local row
  int pj, rows, c0, base; // block width, block rows, first column, offset in the tile buffer
  long long src;          // element index of H_j[ra, 0]
};
struct Tile {
  int i0, npts, ns, tx_bytes;
  long long poff;         // partial offset of slot 0 (slots follow, p_j each)
  TileSlot s[kFSlots];
};

struct FusedArgs {
  const double* H;
  const long long* H_off;
  const int* row_ptr;
  const int* col_off;
  const Tile* tiles;
  int ntiles;
  const double* w;
  double* part;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT%=:\n\t"
      "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// layout of one slot inside a tile buffer: p_j column segments, pitch = len + 2 (even), each
// segment starts on a 16-byte boundary and holds the 16-byte aligned superset of the rows
__device__ __forceinline__ int seg_pitch(int len) { return (len + 3) & ~1; }

__device__ __forceinline__ int col_parity(const TileSlot& S, int k) {
  return static_cast<int>((S.src + static_cast<long long>(k) * S.rows) & 1);
}

// producer warp: arm the barrier with the tile's byte count, then one bulk copy per column segment
__device__ void issue_tile(const FusedArgs& A, const Tile* T, double* buf, uint64_t* bar, int lane) {
  const int ns = T->ns;
  if (lane == 0) mbar_expect_tx(bar, static_cast<uint32_t>(T->tx_bytes));
  __syncwarp();
  for (int s = 0; s < ns; ++s) {
    const TileSlot S = T->s[s];
    const int pitch = seg_pitch(S.len);
    for (int k = lane; k < S.pj; k += 32) {
      const long long idx = S.src + static_cast<long long>(k) * S.rows;
      const int a = static_cast<int>(idx & 1);
      tma_load_1d(buf + S.base + k * pitch, A.H + (idx - a),
                  static_cast<uint32_t>(((S.len + a + 1) & ~1) * sizeof(double)), bar);
    }
  }
}

__global__ void __launch_bounds__(kFThreads) k_fused_normal(FusedArgs A) {
  extern __shared__ __align__(128) double fsm[];
  double* bufs[2] = {fsm, fsm + kFBuf / sizeof(double)};
  __shared__ __align__(8) uint64_t full[2], empty[2];
  __shared__ double y[kFT];
  __shared__ double ypart[kFSlots][kFT];
  __shared__ Tile cur;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncw = (blockDim.x >> 5) - 1;  // compute warps (warp 0 produces)
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], ncw);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    // ---- producer: keep up to two tiles in flight
    int it = 0;
    for (int tile = blockIdx.x; tile < A.ntiles; tile += gridDim.x, ++it) {
      const int b = it & 1;
      if (it >= 2) mbar_wait(&empty[b], ((it >> 1) - 1) & 1);  // consumers released this buffer
      if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      issue_tile(A, A.tiles + tile, bufs[b], &full[b], lane);
    }
    return;
  }
  // ---- consumers (warps 1..ncw), named barrier 1 among them
  const int ctid = threadIdx.x - 32, cthr = ncw * 32;
  int it = 0;
  for (int tile = blockIdx.x; tile < A.ntiles; tile += gridDim.x, ++it) {
    const int b = it & 1;
    for (int q = ctid; q < static_cast<int>(sizeof(Tile) / sizeof(int)); q += cthr)
      reinterpret_cast<int*>(&cur)[q] = reinterpret_cast<const int*>(A.tiles + tile)[q];
    mbar_wait(&full[b], (it >> 1) & 1);
    asm volatile("bar.sync 1, %0;" ::"r"(cthr) : "memory");
    const double* buf = bufs[b];
    const int ns = cur.ns;
    // y partials: thread per (slot, point in slot)
    for (int e = ctid; e < ns * kFT; e += cthr) {
      const int s = e / kFT, tt = e % kFT;
      const TileSlot& S = cur.s[s];
      if (tt >= S.len) continue;
      const int pitch = seg_pitch(S.len), pj = S.pj;
      const int par0 = static_cast<int>(S.src & 1), rodd = S.rows & 1;
      const double* seg = buf + S.base + tt;
      const double* ww = A.w + S.c0;
      double a0 = 0.0, a1 = 0.0;
      int k = 0;
      for (; k + 2 <= pj; k += 2) {
        a0 += seg[k * pitch + par0] * ww[k];
        a1 += seg[(k + 1) * pitch + (par0 ^ rodd)] * ww[k + 1];
      }
      if (k < pj) a0 += seg[k * pitch + (par0 ^ (k & rodd))] * ww[k];
      ypart[s][S.ta + tt] = a0 + a1;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(cthr) : "memory");
    for (int t = ctid; t < cur.npts; t += cthr) {
      double acc = 0.0;
      for (int s = 0; s < ns; ++s)  // slots ascend by block: the reference's per-row order
        if (t >= cur.s[s].ta && t < cur.s[s].ta + cur.s[s].len) acc += ypart[s][t];
      y[t] = acc;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(cthr) : "memory");
    // Hᵀy partials: warp per (slot, column), lanes over the slot's points
    const int cw = warp - 1;
    long long po = cur.poff;
    for (int s = 0; s < ns; ++s) {
      const TileSlot& S = cur.s[s];
      const int pitch = seg_pitch(S.len);
      const int par0 = static_cast<int>(S.src & 1), rodd = S.rows & 1;
      for (int k = cw; k < S.pj; k += ncw) {
        const double* seg = buf + S.base + k * pitch + (par0 ^ (k & rodd));
        double acc = 0.0;
        for (int tt = lane; tt < S.len; tt += 32) acc += seg[tt] * y[S.ta + tt];
        acc = warp_sum(acc);
        if (lane == 0) A.part[po + k] = acc;
      }
      po += S.pj;
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(smem_u32(&empty[b])) : "memory");
    asm volatile("bar.sync 1, %0;" ::"r"(cthr) : "memory");  // `cur`, y, ypart reusable
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

// Tile plan (once per assembled system): greedy runs of consecutive points in which every
// covering block's rows stay contiguous, bounded by kFT points, kFSlots blocks and kFBuf bytes.
bool build_fused_plan(Ctx& c) {
  const int N = c.N, MC = c.maxcov, J = c.J;
  std::vector<int> cn(N), cj(static_cast<size_t>(N) * MC), cr(static_cast<size_t>(N) * MC);
  c.cov_n.download(cn.data(), N, c.stream);
  c.cov_j.download(cj.data(), cj.size(), c.stream);
  c.cov_r.download(cr.data(), cr.size(), c.stream);
  RDD_CUDA(cudaStreamSynchronize(c.stream));
  std::vector<Tile> tiles;
  std::vector<std::vector<long long>> per_block(J);
  long long poff = 0;
  auto seg_pitch_h = [](int len) { return (len + 3) & ~1; };
  int i = 0;
  while (i < N) {
    Tile T{};
    T.i0 = i;
    T.ns = 0;
    int t = 0;
    for (; i < N && t < kFT; ++i, ++t) {
      // tentative extension by point i
      Tile U = T;
      bool ok = true;
      for (int q = 0; q < cn[i] && ok; ++q) {
        const int b = cj[static_cast<size_t>(i) * MC + q], r = cr[static_cast<size_t>(i) * MC + q];
        int s = -1;
        for (int z = 0; z < U.ns; ++z)
          if (U.s[z].blk == b) s = z;
        if (s < 0) {
          if (U.ns == kFSlots) {
            ok = false;
            break;
          }
          U.s[U.ns++] = TileSlot{b, t, 1, r, 0, 0, 0, 0, 0};
        } else {
          TileSlot& S = U.s[s];
          if (S.ta + S.len != t || S.ra + S.len != r) ok = false;  // contiguity in tile and rows
          else ++S.len;
        }
      }
      long long bytes = 0;
      for (int z = 0; z < U.ns && ok; ++z) bytes += static_cast<long long>(c.h_p[U.s[z].blk]) * seg_pitch_h(U.s[z].len) * 8;
      if (!ok || bytes > kFBuf) {
        if (t == 0) return false;  // a single point does not fit
        break;
      }
      T = U;
    }
    T.npts = t;
    // slots in ascending block order (the reference's per-row summation order)
    std::sort(T.s, T.s + T.ns, [](const TileSlot& a, const TileSlot& b) { return a.blk < b.blk; });
    T.poff = poff;
    long long tx = 0;
    int base = 0;
    for (int z = 0; z < T.ns; ++z) {
      TileSlot& S = T.s[z];
      const int j = S.blk;
      S.pj = c.h_p[j];
      S.rows = c.h_row_ptr[j + 1] - c.h_row_ptr[j];
      S.c0 = c.h_col_off[j];
      S.base = base;
      S.src = c.H_off[j] + S.ra;
      base += S.pj * seg_pitch_h(S.len);
      for (int k = 0; k < S.pj; ++k) {
        const int a = static_cast<int>((S.src + static_cast<long long>(k) * S.rows) & 1);
        tx += ((S.len + a + 1) & ~1) * 8;
      }
    }
    T.tx_bytes = static_cast<int>(tx);
    for (int z = 0; z < T.ns; ++z) {
      per_block[T.s[z].blk].push_back(poff);
      poff += c.h_p[T.s[z].blk];
    }
    tiles.push_back(T);
  }
  std::vector<int> bptr(J + 1, 0);
  std::vector<long long> bparts;
  for (int j = 0; j < J; ++j) {
    bparts.insert(bparts.end(), per_block[j].begin(), per_block[j].end());
    bptr[j + 1] = static_cast<int>(bparts.size());
  }
  c.f_tiles.ensure(tiles.size() * sizeof(Tile));
  RDD_CUDA(cudaMemcpyAsync(c.f_tiles.p, tiles.data(), tiles.size() * sizeof(Tile), cudaMemcpyHostToDevice, c.stream));
  c.f_bptr.upload(bptr, c.stream);
  c.f_bparts.upload(bparts, c.stream);
  c.f_part.ensure(std::max<long long>(1, poff));
  c.f_ntiles = static_cast<int>(tiles.size());
  c.f_part_size = poff;
  RDD_CUDA(cudaStreamSynchronize(c.stream));
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
  A.tiles = reinterpret_cast<const Tile*>(c.f_tiles.p);
  A.ntiles = c.f_ntiles;
  A.w = w;
  A.part = c.f_part.p;
  const size_t smem = 2 * static_cast<size_t>(kFBuf);
  static bool attr = false;
  if (!attr) {
    RDD_CUDA(cudaFuncSetAttribute(k_fused_normal, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    attr = true;
  }
  const int grid = std::min(c.f_ntiles, c.prop.multiProcessorCount);
  k_fused_normal<<<grid, kFThreads, smem, c.stream>>>(A);
  RDD_LAUNCH_CHECK();
  k_fused_reduce<<<ceil_div(c.p, 256), 256, 0, c.stream>>>(c.f_part.p, c.f_bptr.p, c.f_bparts.p, c.dcol_off.p,
                                                           c.downer.p, c.p, out);
  RDD_LAUNCH_CHECK();
}

}  // namespace rdd
