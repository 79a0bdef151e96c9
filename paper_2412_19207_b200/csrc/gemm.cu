// gemm.cu — batched, variable-shape FP64 GEMM on the FP64 tensor cores (DMMA).
//
// tcgen05 has no f64 kind (ptxas rejects `.kind::f64` for sm_100a), so FP64
// tensor-core work on B200 is `mma.sync.aligned.m8n8k4.row.col.f64` (SASS: DMMA). One CTA
// computes a 64x64 tile of one task with 4 warps (32x32 warp tiles = 4x4 DMMA fragments),
// K staged 16 at a time through padded shared memory with register prefetch of the next
// stage. Used for: Gram SᵀS and TᵀT (PCA, feeds reduction.hpp:91), T = S·V and H = S·V
// (reduction.hpp:133 by linearity), normal blocks H_j1[I]ᵀH_j2[I] with row gathers
// (assembly.hpp:148-183), local-inverse products (schwarz.hpp:76-79).
#include "ctx.hpp"

namespace rdd {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, PAD = 8, NT = 128;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <bool AT, bool BT>
__global__ void __launch_bounds__(NT) k_gemm(const GemmTask* __restrict__ tasks) {
  __shared__ double As[2][BK][BM + PAD];
  __shared__ double Bs[2][BK][BN + PAD];
  const GemmTask T = tasks[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m0 = T.tm * BM, n0 = T.tn * BN;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  double ra[8], rb[8];
  auto load = [&](int k0) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (AT) {  // A(k, m) = A[k + m*lda]
        const int k = k0 + (tid & 15), m = m0 + (tid >> 4) + 8 * i;
        double v = 0.0;
        if (k < T.K && m < T.M) {
          const long long kk = T.gA ? T.gA[k] : k;
          v = T.A[kk + static_cast<long long>(m) * T.lda];
        }
        ra[i] = v;
      } else {  // A(m, k) = A[m + k*lda]
        const int m = m0 + (tid & 63), k = k0 + (tid >> 6) + 2 * i;
        ra[i] = (k < T.K && m < T.M) ? T.A[m + static_cast<long long>(k) * T.lda] : 0.0;
      }
      if (!BT) {  // B(k, n) = B[k + n*ldb]
        const int k = k0 + (tid & 15), n = n0 + (tid >> 4) + 8 * i;
        double v = 0.0;
        if (k < T.K && n < T.N) {
          const long long kk = T.gB ? T.gB[k] : k;
          v = T.B[kk + static_cast<long long>(n) * T.ldb];
        }
        rb[i] = v;
      } else {  // B(k, n) = Bt[n + k*ldb]
        const int n = n0 + (tid & 63), k = k0 + (tid >> 6) + 2 * i;
        rb[i] = (k < T.K && n < T.N) ? T.B[n + static_cast<long long>(k) * T.ldb] : 0.0;
      }
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (AT) As[buf][tid & 15][(tid >> 4) + 8 * i] = ra[i];
      else As[buf][(tid >> 6) + 2 * i][tid & 63] = ra[i];
      if (!BT) Bs[buf][tid & 15][(tid >> 4) + 8 * i] = rb[i];
      else Bs[buf][(tid >> 6) + 2 * i][tid & 63] = rb[i];
    }
  };

  const int nk = (T.K + BK - 1) / BK;
  if (nk > 0) {
    load(0);
    store(0);
  }
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) load((kt + 1) * BK);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[buf][kk + (lane & 3)][wm + 8 * i + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bs[buf][kk + (lane & 3)][wn + 8 * j + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
    if (kt + 1 < nk) store(buf ^ 1);
    __syncthreads();
  }
  // epilogue: fragment (row = lane>>2, cols 2*(lane&3) + {0,1})
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m = m0 + wm + 8 * i + (lane >> 2);
        const int n = n0 + wn + 8 * j + 2 * (lane & 3) + e;
        if (m < T.M && n < T.N) {
          double* p = T.Cm + m + static_cast<long long>(n) * T.ldc;
          *p = (T.beta != 0.0 ? T.beta * *p : 0.0) + T.alpha * acc[i][j][e];
        }
      }
}

template <bool AT, bool BT>
void launch(Ctx& c, const std::vector<GemmTask>& tasks, const char* fam) {
  if (tasks.empty()) return;
  ScopedKernelTimer tk(c, fam);
  DBuf<GemmTask> d;
  d.upload(tasks, c.stream);
  // grid.x limit is 2^31-1; tasks are far fewer
  k_gemm<AT, BT><<<static_cast<unsigned>(tasks.size()), NT, 0, c.stream>>>(d.p);
  RDD_LAUNCH_CHECK();
  if (!alloc_stream()) RDD_CUDA(cudaStreamSynchronize(c.stream));  // task buffer lifetime (non-pooled)
}

}  // namespace

void gemm_tn(Ctx& c, const std::vector<GemmTask>& tasks) { launch<true, false>(c, tasks, "gemm_tn"); }
void gemm_nn(Ctx& c, const std::vector<GemmTask>& tasks) { launch<false, false>(c, tasks, "gemm_nn"); }
void gemm_nt(Ctx& c, const std::vector<GemmTask>& tasks) { launch<false, true>(c, tasks, "gemm_nt"); }

}  // namespace rdd
