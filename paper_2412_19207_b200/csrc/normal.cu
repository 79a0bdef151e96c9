// normal.cu — K7: normal blocks H_j1ᵀH_j2 over the row intersection (assembly.hpp:148-183),
// and the block-sparse HᵀH operator built from them.
//
// For every neighbour pair j1 <= j2 (neighbour sets are symmetric and sorted), the sorted row
// lists are intersected on the device (one CTA per pair: binary search of rows_j1 in rows_j2,
// block-wide stable compaction), then one TN DMMA GEMM over all pairs gathers the intersecting
// rows straight from the column-major blocks. Pairs with an empty intersection are omitted,
// exactly like the reference (`if (i1.empty()) continue;`).
#include <algorithm>

#include "ctx.hpp"

namespace rdd {

namespace {

constexpr int kT = 256;

__device__ __forceinline__ int lower_bound(const int* a, int n, int key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// mode 0: count only; mode 1: write (i1, i2) local-row pairs at out_off[pair]
__global__ void k_intersect(const int* __restrict__ row_ptr, const int* __restrict__ row_idx,
                            const int* __restrict__ pj1, const int* __restrict__ pj2, int* __restrict__ counts,
                            const long long* __restrict__ out_off, int* __restrict__ o1, int* __restrict__ o2,
                            int mode) {
  __shared__ int warp_tot[kT / 32];
  __shared__ int base;
  const int pr = blockIdx.x;
  const int j1 = pj1[pr], j2 = pj2[pr];
  const int* r1 = row_idx + row_ptr[j1];
  const int* r2 = row_idx + row_ptr[j2];
  const int n1 = row_ptr[j1 + 1] - row_ptr[j1], n2 = row_ptr[j2 + 1] - row_ptr[j2];
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int s = 0; s < n1; s += kT) {
    const int a = s + threadIdx.x;
    int pos = -1;
    if (a < n1) {
      const int b = lower_bound(r2, n2, r1[a]);
      if (b < n2 && r2[b] == r1[a]) pos = b;
    }
    const unsigned ball = __ballot_sync(0xffffffffu, pos >= 0);
    if (lane == 0) warp_tot[warp] = __popc(ball);
    __syncthreads();
    int off = base;
    for (int w = 0; w < warp; ++w) off += warp_tot[w];
    off += __popc(ball & ((1u << lane) - 1u));
    if (mode == 1 && pos >= 0) {
      o1[out_off[pr] + off] = a;
      o2[out_off[pr] + off] = pos;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int w = 0; w < kT / 32; ++w) t += warp_tot[w];
      base += t;
    }
    __syncthreads();
  }
  if (mode == 0 && threadIdx.x == 0) counts[pr] = base;
}

// out[col] = Σ_{pairs} NB-block products: y_j1 += B w_j2, y_j2 += Bᵀ w_j1 (j1 != j2).
// One warp per (block row j, local row k): walks the neighbour list of j.
__global__ void k_normal_apply(const double* __restrict__ NB, const long long* __restrict__ nb_lookup_off,
                               const int* __restrict__ nbr_ptr, const int* __restrict__ nbr_idx,
                               const int* __restrict__ col_off, const int* __restrict__ col_owner, int p,
                               const double* __restrict__ w, double* __restrict__ out) {
  const int col = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (col >= p) return;
  const int j = col_owner[col];
  const int k = col - col_off[j];
  const int pj = col_off[j + 1] - col_off[j];
  double s = 0.0;
  for (int q = nbr_ptr[j]; q < nbr_ptr[j + 1]; ++q) {
    const int j2 = nbr_idx[q];
    const long long off = nb_lookup_off[q];  // -1 when the pair has no rows in common
    if (off < 0) continue;
    const int c2 = col_off[j2], p2 = col_off[j2 + 1] - c2;
    if (j <= j2) {  // block (j, j2) is pj x p2 column-major: row k = NB[off + k + c*pj]
      for (int cc = lane; cc < p2; cc += 32) s += NB[off + k + static_cast<long long>(cc) * pj] * w[c2 + cc];
    } else {        // block (j2, j) is p2 x pj: use its column k
      for (int cc = lane; cc < p2; cc += 32) s += NB[off + cc + static_cast<long long>(k) * p2] * w[c2 + cc];
    }
  }
  s = warp_sum(s);
  if (lane == 0) out[col] = s;
}

}  // namespace

void build_normal_blocks(Ctx& c) {
  ScopedKernelTimer tk(c, "normal_blocks");
  const int J = c.J;
  std::vector<int> a1, a2;
  for (int j1 = 0; j1 < J; ++j1)
    for (int q = c.nbr_ptr[j1]; q < c.nbr_ptr[j1 + 1]; ++q)
      if (c.nbr_idx[q] >= j1) {
        a1.push_back(j1);
        a2.push_back(c.nbr_idx[q]);
      }
  const int P = static_cast<int>(a1.size());
  DBuf<int> d1, d2, cnt, o1, o2;
  DBuf<long long> ooff;
  d1.upload(a1, c.stream);
  d2.upload(a2, c.stream);
  cnt.ensure(std::max(P, 1));
  if (P > 0) {
    k_intersect<<<P, kT, 0, c.stream>>>(c.row_ptr.p, c.row_idx.p, d1.p, d2.p, cnt.p, nullptr, nullptr, nullptr, 0);
    RDD_LAUNCH_CHECK();
  }
  std::vector<int> hc(P);
  cnt.download(hc.data(), P, c.stream);
  RDD_CUDA(cudaStreamSynchronize(c.stream));
  std::vector<long long> off(P + 1, 0);
  for (int i = 0; i < P; ++i) off[i + 1] = off[i] + hc[i];
  ooff.upload(off, c.stream);
  o1.ensure(std::max<long long>(1, off[P]));
  o2.ensure(std::max<long long>(1, off[P]));
  if (P > 0) {
    k_intersect<<<P, kT, 0, c.stream>>>(c.row_ptr.p, c.row_idx.p, d1.p, d2.p, cnt.p, ooff.p, o1.p, o2.p, 1);
    RDD_LAUNCH_CHECK();
  }
  // keep non-empty pairs, allocate blocks, one batched TN GEMM with row gathers
  c.nb_j1.clear();
  c.nb_j2.clear();
  c.nb_off.assign(1, 0);
  c.nb_index.clear();
  std::vector<GemmTask> tasks;
  std::vector<int> kept;
  for (int i = 0; i < P; ++i) {
    if (hc[i] == 0) continue;
    const int j1 = a1[i], j2 = a2[i];
    const int p1 = c.h_p[j1], p2 = c.h_p[j2];
    c.nb_index[{j1, j2}] = static_cast<int>(c.nb_j1.size());
    c.nb_j1.push_back(j1);
    c.nb_j2.push_back(j2);
    c.nb_off.push_back(c.nb_off.back() + static_cast<long long>(p1) * p2);
    kept.push_back(i);
  }
  c.NB.ensure(std::max<long long>(1, c.nb_off.back()));
  for (size_t q = 0; q < kept.size(); ++q) {
    const int i = kept[q];
    const int j1 = a1[i], j2 = a2[i];
    const int p1 = c.h_p[j1], p2 = c.h_p[j2];
    const int rows1 = c.h_row_ptr[j1 + 1] - c.h_row_ptr[j1], rows2 = c.h_row_ptr[j2 + 1] - c.h_row_ptr[j2];
    for (int tm = 0; tm < ceil_div(p1, 64); ++tm)
      for (int tn = 0; tn < ceil_div(p2, 64); ++tn)
        tasks.push_back({c.H + c.H_off[j1], c.H + c.H_off[j2], c.NB.p + c.nb_off[q], o1.p + off[i], o2.p + off[i], p1,
                         p2, hc[i], rows1, rows2, p1, tm, tn, 0.0});
  }
  gemm_tn(c, tasks);
  // lookup table aligned with the neighbour CSR for the block-sparse operator
  std::vector<long long> look(c.nbr_idx.size(), -1);
  for (int j = 0; j < J; ++j)
    for (int q = c.nbr_ptr[j]; q < c.nbr_ptr[j + 1]; ++q) {
      const int j2 = c.nbr_idx[q];
      auto it = c.nb_index.find({std::min(j, j2), std::max(j, j2)});
      if (it != c.nb_index.end()) look[q] = c.nb_off[it->second];
    }
  c.nb_look.upload(look, c.stream);
  c.h_nb_look = look;
  RDD_CUDA(cudaStreamSynchronize(c.stream));
}

void normal_apply_dev(Ctx& c, const double* w, double* out) {
  ScopedKernelTimer tk(c, "normal_apply");
  k_normal_apply<<<ceil_div(static_cast<long long>(c.p) * 32, 256), 256, 0, c.stream>>>(
      c.NB.p, c.nb_look.p, c.dnbr_ptr.p, c.dnbr_idx.p, c.dcol_off.p, c.downer.p, c.p, w, out);
  RDD_LAUNCH_CHECK();
}

}  // namespace rdd
