// index.cu — K1: point -> subdomain indexing (bit-exact).
//
// Replaces the O(J·N) scans of assembly.hpp:58-64 (rows_j) / reduction.hpp:36-37 and the
// covering_subdomains loop (geometry.hpp:180-185). The decomposition is a tensor product of
// per-axis intervals, so contains(box_j, x) (geometry.hpp:51-57, closed) is evaluated as the
// same per-axis comparisons against the uploaded interval bounds — identical doubles, identical
// comparisons, hence identical sets. rows_j lists global ids in ascending order; the stable
// two-pass counting sort below (per 256-point chunk: warp ballots for in-warp ranks, per-warp
// box lists for in-CTA offsets, a column scan over chunks) preserves that order without atomics.
#include "ctx.hpp"

namespace rdd {

namespace {

constexpr int kChunk = 256;      // points per CTA
constexpr int kWarps = kChunk / 32;
constexpr int kMaxCov = 64;      // covering boxes per point (3^d worst case for delta=2 is 27)
constexpr int kMaxDistinct = 64; // distinct boxes per warp

struct AxisInfo {
  int d;
  int counts[kMaxDim];
  int stride[kMaxDim];  // flat index stride per axis (axis 0 slowest)
  int off[kMaxDim];     // offsets into the interval arrays
};

// Covering boxes of point i in ascending flat order; returns count (or -1 on overflow).
__device__ int covering(const double* __restrict__ pts, int N, int i, const double* __restrict__ ax_lo,
                        const double* __restrict__ ax_hi, const AxisInfo& A, int* out) {
  int cand[kMaxDim][8];
  int nc[kMaxDim];
  for (int a = 0; a < A.d; ++a) {
    const double x = pts[static_cast<size_t>(a) * N + i];
    nc[a] = 0;
    for (int k = 0; k < A.counts[a]; ++k) {
      const double lo = ax_lo[A.off[a] + k], hi = ax_hi[A.off[a] + k];
      if (!(x < lo || x > hi)) {  // geometry.hpp:54 closed test, same comparisons
        if (nc[a] >= 8) return -1;
        cand[a][nc[a]++] = k;
      }
    }
    if (nc[a] == 0) return 0;
  }
  // lexicographic product (axis 0 slowest) = ascending flat index
  int n = 0;
  int it[kMaxDim] = {0, 0, 0, 0};
  while (true) {
    int flat = 0;
    for (int a = 0; a < A.d; ++a) flat += cand[a][it[a]] * A.stride[a];
    if (n >= kMaxCov) return -1;
    out[n++] = flat;
    int a = A.d - 1;
    for (; a >= 0; --a) {
      if (++it[a] < nc[a]) break;
      it[a] = 0;
    }
    if (a < 0) break;
  }
  return n;
}

struct WarpLists {
  int box[kWarps][kMaxDistinct];
  int cnt[kWarps][kMaxDistinct];
  int n[kWarps];
};

// In-warp pass: for each distinct box among the warp's covers (ascending), ballot the lanes
// that cover it; lane rank = popc(ballot & lanemask_lt). Records (box, count) per warp.
__device__ void warp_rank(const int* cov, int ncov, int* rank, WarpLists& L, int warp, int lane, int* overflow) {
  int done = 0;  // bitmask over cov slots already ranked (ncov <= 64)
  unsigned long long donemask = 0ull;
  int nd = 0;
  while (true) {
    int mine = INT32_MAX;
    for (int s = 0; s < ncov; ++s)
      if (!((donemask >> s) & 1ull)) mine = min(mine, cov[s]);
    const int jmin = warp_min(mine);
    if (jmin == INT32_MAX) break;
    int slot = -1;
    for (int s = 0; s < ncov; ++s)
      if (cov[s] == jmin) slot = s;
    const unsigned ball = __ballot_sync(0xffffffffu, slot >= 0);
    if (slot >= 0) {
      rank[slot] = __popc(ball & ((1u << lane) - 1u));
      donemask |= (1ull << slot);
    }
    if (lane == 0) {
      if (nd < kMaxDistinct) {
        L.box[warp][nd] = jmin;
        L.cnt[warp][nd] = __popc(ball);
      } else {
        *overflow = 1;
      }
    }
    ++nd;
  }
  (void)done;
  if (lane == 0) L.n[warp] = min(nd, kMaxDistinct);
}

__device__ int warp_offset(const WarpLists& L, int warp, int box) {
  int off = 0;
  for (int w = 0; w < warp; ++w)
    for (int t = 0; t < L.n[w]; ++t)
      if (L.box[w][t] == box) off += L.cnt[w][t];
  return off;
}

__global__ void k_index_count(const double* __restrict__ pts, int N, const double* __restrict__ ax_lo,
                              const double* __restrict__ ax_hi, AxisInfo A, int J, int* __restrict__ chunk_cnt,
                              int* __restrict__ cov_n, int* __restrict__ err) {
  __shared__ WarpLists L;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * kChunk + threadIdx.x;
  int cov[kMaxCov], rank[kMaxCov];
  int ncov = 0;
  if (i < N) {
    ncov = covering(pts, N, i, ax_lo, ax_hi, A, cov);
    if (ncov < 0) {
      atomicExch(err, 1);
      ncov = 0;
    }
    cov_n[i] = ncov;
  }
  warp_rank(cov, ncov, rank, L, warp, lane, err);
  __syncthreads();
  // chunk totals: the first warp holding a box sums all warps' counts for it
  if (lane == 0) {
    for (int t = 0; t < L.n[warp]; ++t) {
      const int b = L.box[warp][t];
      bool first = true;
      for (int w = 0; w < warp && first; ++w)
        for (int u = 0; u < L.n[w]; ++u)
          if (L.box[w][u] == b) first = false;
      if (!first) continue;
      int tot = 0;
      for (int w = 0; w < kWarps; ++w)
        for (int u = 0; u < L.n[w]; ++u)
          if (L.box[w][u] == b) tot += L.cnt[w][u];
      chunk_cnt[static_cast<size_t>(blockIdx.x) * J + b] = tot;
    }
  }
}

// exclusive scan over chunks, per box (column scan); totals out
__global__ void k_chunk_scan(int* __restrict__ chunk_cnt, int nchunks, int J, int* __restrict__ totals) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= J) return;
  int run = 0;
  int c = 0;
  for (; c + 8 <= nchunks; c += 8) {  // independent loads in flight, serial running sum
    int v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = chunk_cnt[static_cast<size_t>(c + u) * J + j];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      chunk_cnt[static_cast<size_t>(c + u) * J + j] = run;
      run += v[u];
    }
  }
  for (; c < nchunks; ++c) {
    const size_t k = static_cast<size_t>(c) * J + j;
    const int v = chunk_cnt[k];
    chunk_cnt[k] = run;
    run += v;
  }
  totals[j] = run;
}

__global__ void k_index_fill(const double* __restrict__ pts, int N, const double* __restrict__ ax_lo,
                             const double* __restrict__ ax_hi, AxisInfo A, int J,
                             const int* __restrict__ chunk_off, const int* __restrict__ row_ptr,
                             int* __restrict__ row_idx, int* __restrict__ cov_j, int* __restrict__ cov_r, int maxcov,
                             int* __restrict__ err) {
  __shared__ WarpLists L;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * kChunk + threadIdx.x;
  int cov[kMaxCov], rank[kMaxCov];
  int ncov = 0;
  if (i < N) {
    ncov = covering(pts, N, i, ax_lo, ax_hi, A, cov);
    if (ncov < 0) ncov = 0;
  }
  warp_rank(cov, ncov, rank, L, warp, lane, err);
  __syncthreads();
  for (int s = 0; s < ncov; ++s) {
    const int b = cov[s];
    const int local = chunk_off[static_cast<size_t>(blockIdx.x) * J + b] + warp_offset(L, warp, b) + rank[s];
    const int pos = row_ptr[b] + local;
    row_idx[pos] = i;
    if (s < maxcov) {
      cov_j[static_cast<size_t>(i) * maxcov + s] = b;
      cov_r[static_cast<size_t>(i) * maxcov + s] = local;
    }
  }
}

__global__ void k_max(const int* __restrict__ v, int n, int* __restrict__ out) {
  int m = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) m = max(m, v[i]);
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

}  // namespace

void build_index(Ctx& c) {
  ScopedKernelTimer tk(c, "index");
  const int N = c.N, J = c.J;
  AxisInfo A{};
  A.d = c.d;
  std::vector<double> alo, ahi;
  int stride = 1;
  for (int a = c.d - 1; a >= 0; --a) {
    A.stride[a] = stride;
    stride *= c.counts[a];
  }
  for (int a = 0; a < c.d; ++a) {
    A.counts[a] = c.counts[a];
    A.off[a] = static_cast<int>(alo.size());
    for (int k = 0; k < c.counts[a]; ++k) {
      alo.push_back(c.axis_lo[a][k]);
      ahi.push_back(c.axis_hi[a][k]);
    }
  }
  DBuf<double>& dlo = c.ax_lo;  // kept: the evaluation finds test-point covers the same way
  DBuf<double>& dhi = c.ax_hi;
  dlo.upload(alo, c.stream);
  dhi.upload(ahi, c.stream);
  for (int a = 0; a < kMaxDim; ++a) {
    c.ax_counts[a] = a < c.d ? A.counts[a] : 1;
    c.ax_stride[a] = a < c.d ? A.stride[a] : 0;
    c.ax_off[a] = a < c.d ? A.off[a] : 0;
  }
  const int nchunks = ceil_div(N, kChunk);
  DBuf<int> chunk, totals, err, mx;
  chunk.zero(static_cast<size_t>(nchunks) * J, c.stream);
  totals.ensure(J);
  err.zero(1, c.stream);
  mx.zero(1, c.stream);
  c.cov_n.ensure(N);
  k_index_count<<<nchunks, kChunk, 0, c.stream>>>(c.pts.p, N, dlo.p, dhi.p, A, J, chunk.p, c.cov_n.p, err.p);
  RDD_LAUNCH_CHECK();
  k_chunk_scan<<<ceil_div(J, 128), 128, 0, c.stream>>>(chunk.p, nchunks, J, totals.p);
  RDD_LAUNCH_CHECK();
  k_max<<<std::min(1024, ceil_div(N, 256)), 256, 0, c.stream>>>(c.cov_n.p, N, mx.p);
  RDD_LAUNCH_CHECK();
  std::vector<int> h_tot(J);
  int h_err = 0, h_max = 0;
  totals.download(h_tot.data(), J, c.stream);
  err.download(&h_err, 1, c.stream);
  mx.download(&h_max, 1, c.stream);
  RDD_CUDA(cudaStreamSynchronize(c.stream));
  if (h_err) throw std::runtime_error("indexing: too many covering subdomains per point");
  c.h_row_ptr.assign(J + 1, 0);
  for (int j = 0; j < J; ++j) c.h_row_ptr[j + 1] = c.h_row_ptr[j] + h_tot[j];
  c.sum_rows = c.h_row_ptr[J];
  c.maxcov = std::max(1, h_max);
  c.row_ptr.upload(c.h_row_ptr, c.stream);
  c.row_idx.ensure(std::max<long long>(1, c.sum_rows));
  c.cov_j.ensure(static_cast<size_t>(N) * c.maxcov);
  c.cov_r.ensure(static_cast<size_t>(N) * c.maxcov);
  k_index_fill<<<nchunks, kChunk, 0, c.stream>>>(c.pts.p, N, dlo.p, dhi.p, A, J, chunk.p, c.row_ptr.p, c.row_idx.p,
                                                 c.cov_j.p, c.cov_r.p, c.maxcov, err.p);
  RDD_LAUNCH_CHECK();
  err.download(&h_err, 1, c.stream);
  RDD_CUDA(cudaStreamSynchronize(c.stream));
  if (h_err) throw std::runtime_error("indexing: too many distinct subdomains per warp");
}

}  // namespace rdd
