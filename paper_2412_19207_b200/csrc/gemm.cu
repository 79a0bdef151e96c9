// gemm.cu — batched, variable-shape FP64 GEMM on the FP64 tensor cores (DMMA).
//
// tcgen05 has no f64 kind (ptxas rejects `.kind::f64` for sm_100a), so FP64
// tensor-core work on B200 is `mma.sync.aligned.m8n8k4.row.col.f64` (SASS: DMMA). One CTA
// computes a 64x64 tile of one task with 4 warps (32x32 warp tiles = 4x4 DMMA fragments),
// K staged 16 at a time through a 3-deep cp.async ring in padded shared memory. Used for: Gram SᵀS and TᵀT (PCA, feeds reduction.hpp:91), T = S·V and H = S·V
// (reduction.hpp:133 by linearity), normal blocks H_j1[I]ᵀH_j2[I] with row gathers
// (assembly.hpp:148-183), local-inverse products (schwarz.hpp:76-79).
#include "ctx.hpp"

namespace rdd {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 128;
constexpr int KP = BK + 4;   // k-contiguous tiles: [tile][BK+4] (row stride ≡ 4 banks mod 16)
constexpr int MP = BM + 4;   // m/n-contiguous tiles: [BK][tile+4] (64- and 80-wide: stride ≡ 4 mod 16)
// doubles per operand per stage for a TB-wide square CTA tile (TB = 64 or 80)
constexpr int stage_doubles(int tb) { return tb * KP > BK * (tb + 4) ? tb * KP : BK * (tb + 4); }
constexpr int kStageA = stage_doubles(BM);
constexpr size_t gemm_smem(int stages, int tb = BM) {
  return static_cast<size_t>(stages) * 2 * stage_doubles(tb) * sizeof(double);
}
// pipeline depth / residency per mode (tools/gemm_bench.py): the NN and NT products (projections,
// Cholesky panel and trailing updates) run best with a 2-deep ring and 4 CTAs per SM (+5-10% on
// the K = 64 and K = 512 update shapes), the TN Gram products with a 3-deep ring and 3 CTAs
template <bool AT>
struct GemmCfg {
  static constexpr int stages = AT ? 3 : 2;
  static constexpr int minb = AT ? 3 : 4;
};

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
// 8-byte asynchronous global->shared copy; src_size 0 zero-fills (out-of-range elements)
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// One CTA: a TB x TB tile of one task (TB = 16·FR: 64 by default, 80 for operands whose edges
// are multiples of 80 — m = 400 pads to 448 in 64-wide tiles, a quarter more work), 4 warps
// (8·FR-square warp tiles = FR x FR DMMA fragments). K streams through a STAGES-deep cp.async
// ring; each operand tile keeps its global contiguous direction in shared memory (k-contiguous
// for Aᵀ / B, m-contiguous for A / Bᵀ) so the copies coalesce, and the padded strides make the
// fragment reads bank-conflict free.
template <bool AT, bool BT, int STAGES = GemmCfg<AT>::stages, int FR = 4, int MINB = GemmCfg<AT>::minb, int FRN = FR>
__global__ void __launch_bounds__(NT, MINB) k_gemm(const GemmTask* __restrict__ tasks) {
  // TB x TBN CTA tile (rows x columns of C); the square tiles have FRN = FR
  constexpr int TB = 16 * FR, WT = 8 * FR, MPt = TB + 4, kStageA_ = stage_doubles(TB);
  constexpr int TBN = 16 * FRN, WTN = 8 * FRN, NPt = TBN + 4, kStageB_ = stage_doubles(TBN);
  constexpr int kStage2 = kStageA_ + kStageB_;
  extern __shared__ __align__(16) double gsm[];
  const GemmTask T = tasks[blockIdx.x];
  if (T.M <= 0) return;  // empty task (a structurally zero tile of a device-generated list)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m0 = T.tm * TB, n0 = T.tn * TBN;
  const int wm = (warp >> 1) * WT, wn = (warp & 1) * WTN;

  // C = beta·C + alpha·op(A)op(B). With alpha = ±1 the accumulators start from (beta/alpha)·C,
  // loaded here so the C read overlaps the operand prologue instead of trailing the main loop
  const bool pre = T.beta != 0.0 && (T.alpha == 1.0 || T.alpha == -1.0);
  const double cf = T.beta * T.alpha;  // beta/alpha for alpha = ±1
  double acc[FR][FRN][2];
#pragma unroll
  for (int i = 0; i < FR; ++i)
#pragma unroll
    for (int j = 0; j < FRN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m = m0 + wm + 8 * i + (lane >> 2);
        const int n = n0 + wn + 8 * j + 2 * (lane & 3) + e;
        acc[i][j][e] = (pre && m < T.M && n < T.N) ? cf * T.Cm[m + static_cast<long long>(n) * T.ldc] : 0.0;
      }

  auto As = [&](int s) { return gsm + static_cast<size_t>(s) * kStage2; };
  auto Bs = [&](int s) { return gsm + static_cast<size_t>(s) * kStage2 + kStageA_; };
  // row-gather indices (TN normal blocks) for the stage issued next are loaded one issue ahead, so
  // the dependent index read does not stall the cp.async issue of every stage
  int gia = 0, gib = 0;
  auto gidx = [&](int kt) {
    const int k = kt * BK + (tid & 15);
    gia = (AT && T.gA && k < T.K) ? __ldg(T.gA + k) : k;
    gib = (!BT && T.gB && k < T.K) ? __ldg(T.gB + k) : k;
  };
  gidx(0);
  auto issue = [&](int kt, int s) {
    const int k0 = kt * BK;
    double* a = As(s);
    double* bsm = Bs(s);
    const int ga = gia, gb = gib;
    // the wide tiles keep these loops rolled: unrolled, their hoisted row addresses spill
#pragma unroll(FR == 4 && FRN == 4 ? TB / 8 : 1)
    for (int i = 0; i < TB / 8; ++i) {
      if (AT) {  // A(k, m) = A[k + m*lda] -> a[m][k]
        const int k = k0 + (tid & 15), ml = (tid >> 4) + 8 * i, m = m0 + ml;
        const bool v = k < T.K && m < T.M;
        const long long kk = v ? ga : 0;
        cp_async8(a + ml * KP + (tid & 15), v ? T.A + kk + static_cast<long long>(m) * T.lda : T.A, v);
      } else {  // A(m, k) = A[m + k*lda] -> a[k][m]
        const int e = tid + NT * i, ml = e % TB, m = m0 + ml, kl = e / TB, k = k0 + kl;
        const bool v = k < T.K && m < T.M;
        cp_async8(a + kl * MPt + ml, v ? T.A + m + static_cast<long long>(k) * T.lda : T.A, v);
      }
      if (FRN == FR) {
        if (!BT) {  // B(k, n) = B[k + n*ldb] -> b[n][k]
          const int k = k0 + (tid & 15), nl = (tid >> 4) + 8 * i, n = n0 + nl;
          const bool v = k < T.K && n < T.N;
          const long long kk = v ? gb : 0;
          cp_async8(bsm + nl * KP + (tid & 15), v ? T.B + kk + static_cast<long long>(n) * T.ldb : T.B, v);
        } else {  // B(k, n) = Bt[n + k*ldb] -> b[k][n]
          const int e = tid + NT * i, nl = e % TBN, n = n0 + nl, kl = e / TBN, k = k0 + kl;
          const bool v = k < T.K && n < T.N;
          cp_async8(bsm + kl * NPt + nl, v ? T.B + n + static_cast<long long>(k) * T.ldb : T.B, v);
        }
      }
    }
    if (FRN != FR) {
#pragma unroll 1
      for (int i = 0; i < TBN / 8; ++i) {
        if (!BT) {
          const int k = k0 + (tid & 15), nl = (tid >> 4) + 8 * i, n = n0 + nl;
          const bool v = k < T.K && n < T.N;
          const long long kk = v ? gb : 0;
          cp_async8(bsm + nl * KP + (tid & 15), v ? T.B + kk + static_cast<long long>(n) * T.ldb : T.B, v);
        } else {
          const int e = tid + NT * i, nl = e % TBN, n = n0 + nl, kl = e / TBN, k = k0 + kl;
          const bool v = k < T.K && n < T.N;
          cp_async8(bsm + kl * NPt + nl, v ? T.B + n + static_cast<long long>(k) * T.ldb : T.B, v);
        }
      }
    }
    gidx(kt + 1);
  };

  const int nk = (T.K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) issue(s, s);
    cp_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();  // stage kt visible to all; stage kt-1's buffer free for reuse
    if (kt + STAGES - 1 < nk) issue(kt + STAGES - 1, (kt + STAGES - 1) % STAGES);
    cp_commit();
    const double* a = As(kt % STAGES);
    const double* bsm = Bs(kt % STAGES);
    // fragments double-buffered across the four k-steps of the stage: the loads of step kk+4 are
    // issued before the FR² DMMAs of step kk, so no DMMA waits on its own shared-memory load
    constexpr int NBUF = FR == 4 ? 2 : 1;  // the 80 x 80 tile has no registers left for a second set
    double af[NBUF][FR], bf[NBUF][FRN];
    auto frag = [&](int kk, int b) {
      const int k = kk + (lane & 3);
#pragma unroll
      for (int i = 0; i < FR; ++i) {
        const int ml = wm + 8 * i + (lane >> 2);
        af[b][i] = AT ? a[ml * KP + k] : a[k * MPt + ml];
      }
#pragma unroll
      for (int j = 0; j < FRN; ++j) {
        const int nl = wn + 8 * j + (lane >> 2);
        bf[b][j] = BT ? bsm[k * NPt + nl] : bsm[nl * KP + k];
      }
    };
    if (NBUF == 2) frag(0, 0);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      const int b = NBUF == 2 ? (kk >> 2) & 1 : 0;
      if (NBUF == 2) {
        if (kk + 4 < BK) frag(kk + 4, b ^ 1);
      } else {
        frag(kk, 0);
      }
#pragma unroll
      for (int i = 0; i < FR; ++i)
#pragma unroll
        for (int j = 0; j < FRN; ++j) dmma(acc[i][j], af[b][i], bf[b][j]);
    }
  }
  cp_wait<0>();
  // epilogue: fragment (row = lane>>2, cols 2*(lane&3) + {0,1})
#pragma unroll
  for (int i = 0; i < FR; ++i)
#pragma unroll
    for (int j = 0; j < FRN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m = m0 + wm + 8 * i + (lane >> 2);
        const int n = n0 + wn + 8 * j + 2 * (lane & 3) + e;
        if (m < T.M && n < T.N) {
          double* p = T.Cm + m + static_cast<long long>(n) * T.ldc;
          *p = pre ? T.alpha * acc[i][j][e] : (T.beta != 0.0 ? T.beta * *p : 0.0) + T.alpha * acc[i][j][e];
        }
      }
}

// NN product with a 64 x 128 CTA tile (8 warps, 32x32 warp tiles): for C = A·B with N <= 128 (the
// PCA's S·V_r, S·Q and S·V on blocks with r_j, p_j <= 128) one CTA covers every column, so the
// large A = S is streamed once per row tile instead of once per 64-column tile. Tasks index tiles
// in units of (64, 128).
constexpr int WBN = 128, WNT = 256, WSTAGES = 3;
constexpr int kStageWA = BK * MP, kStageWB = WBN * KP;
constexpr size_t kWideSmem = static_cast<size_t>(WSTAGES) * (kStageWA + kStageWB) * sizeof(double);

__global__ void __launch_bounds__(WNT, 2) k_gemm_nn_wide(const GemmTask* __restrict__ tasks) {
  extern __shared__ __align__(16) double gsm[];
  const GemmTask T = tasks[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m0 = T.tm * BM, n0 = T.tn * WBN;
  const int wm = (warp >> 2) * 32, wn = (warp & 3) * 32;
  const bool pre = T.beta != 0.0 && (T.alpha == 1.0 || T.alpha == -1.0);
  const double cf = T.beta * T.alpha;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m = m0 + wm + 8 * i + (lane >> 2);
        const int n = n0 + wn + 8 * j + 2 * (lane & 3) + e;
        acc[i][j][e] = (pre && m < T.M && n < T.N) ? cf * T.Cm[m + static_cast<long long>(n) * T.ldc] : 0.0;
      }
  auto As = [&](int st) { return gsm + static_cast<size_t>(st) * (kStageWA + kStageWB); };
  auto Bs = [&](int st) { return gsm + static_cast<size_t>(st) * (kStageWA + kStageWB) + kStageWA; };
  auto issue = [&](int kt, int st) {
    const int k0 = kt * BK;
    double* a = As(st);
    double* bsm = Bs(st);
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // A(m, k) = A[m + k*lda] -> a[k][m]
      const int ml = tid & 63, m = m0 + ml, kl = (tid >> 6) + 4 * i, k = k0 + kl;
      const bool v = k < T.K && m < T.M;
      cp_async8(a + kl * MP + ml, v ? T.A + m + static_cast<long long>(k) * T.lda : T.A, v);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {  // B(k, n) = B[k + n*ldb] -> b[n][k]
      const int kl = tid & 15, k = k0 + kl, nl = (tid >> 4) + 16 * i, n = n0 + nl;
      const bool v = k < T.K && n < T.N;
      cp_async8(bsm + nl * KP + kl, v ? T.B + k + static_cast<long long>(n) * T.ldb : T.B, v);
    }
  };
  const int nk = (T.K + BK - 1) / BK;
#pragma unroll
  for (int st = 0; st < WSTAGES - 1; ++st) {
    if (st < nk) issue(st, st);
    cp_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_wait<WSTAGES - 2>();
    __syncthreads();
    if (kt + WSTAGES - 1 < nk) issue(kt + WSTAGES - 1, (kt + WSTAGES - 1) % WSTAGES);
    cp_commit();
    const double* a = As(kt % WSTAGES);
    const double* bsm = Bs(kt % WSTAGES);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      const int k = kk + (lane & 3);
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = a[k * MP + wm + 8 * i + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = bsm[(wn + 8 * j + (lane >> 2)) * KP + k];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_wait<0>();
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int m = m0 + wm + 8 * i + (lane >> 2);
        const int n = n0 + wn + 8 * j + 2 * (lane & 3) + e;
        if (m < T.M && n < T.N) {
          double* pp = T.Cm + m + static_cast<long long>(n) * T.ldc;
          *pp = pre ? T.alpha * acc[i][j][e] : (T.beta != 0.0 ? T.beta * *pp : 0.0) + T.alpha * acc[i][j][e];
        }
      }
}

template <bool AT, bool BT>
void launch(Ctx& c, const std::vector<GemmTask>& tasks, const char* fam, int tile = BM) {
  if (tasks.empty()) return;
  ScopedKernelTimer tk(c, fam);
  DBuf<GemmTask> d;
  d.ensure(tasks.size());
  c.stage.upload(d.p, tasks.data(), tasks.size() * sizeof(GemmTask), c.stream);
  // grid.x limit is 2^31-1; tasks are far fewer
  if (tile == 6480) {  // 64 x 80 (rows x columns): 2-deep ring, 3 CTAs per SM
    constexpr size_t smem = static_cast<size_t>(2) * (stage_doubles(64) + stage_doubles(80)) * sizeof(double);
    ensure_smem_attr(reinterpret_cast<const void*>(k_gemm<AT, BT, 2, 4, 3, 5>), smem);
    k_gemm<AT, BT, 2, 4, 3, 5><<<static_cast<unsigned>(tasks.size()), NT, smem, c.stream>>>(d.p);
  } else if (tile == 80) {  // 2-deep ring, 3 CTAs per SM (100 accumulator registers per thread)
    constexpr size_t smem = gemm_smem(2, 80);
    ensure_smem_attr(reinterpret_cast<const void*>(k_gemm<AT, BT, 2, 5, 3>), smem);
    k_gemm<AT, BT, 2, 5, 3><<<static_cast<unsigned>(tasks.size()), NT, smem, c.stream>>>(d.p);
  } else {
    constexpr size_t smem = gemm_smem(GemmCfg<AT>::stages);
    ensure_smem_attr(reinterpret_cast<const void*>(k_gemm<AT, BT>), smem);
    k_gemm<AT, BT><<<static_cast<unsigned>(tasks.size()), NT, smem, c.stream>>>(d.p);
  }
  RDD_LAUNCH_CHECK();
  if (!alloc_stream()) RDD_CUDA(cudaStreamSynchronize(c.stream));  // task buffer lifetime (non-pooled)
}

}  // namespace

void gemm_nn_wide(Ctx& c, const std::vector<GemmTask>& tasks) {
  if (tasks.empty()) return;
  ScopedKernelTimer tk(c, "gemm_nn");
  DBuf<GemmTask> d;
  d.ensure(tasks.size());
  c.stage.upload(d.p, tasks.data(), tasks.size() * sizeof(GemmTask), c.stream);
  ensure_smem_attr(reinterpret_cast<const void*>(k_gemm_nn_wide), kWideSmem);
  k_gemm_nn_wide<<<static_cast<unsigned>(tasks.size()), WNT, kWideSmem, c.stream>>>(d.p);
  RDD_LAUNCH_CHECK();
  if (!alloc_stream()) RDD_CUDA(cudaStreamSynchronize(c.stream));
}
void gemm_tn(Ctx& c, const std::vector<GemmTask>& tasks, int tile) { launch<true, false>(c, tasks, "gemm_tn", tile); }
void gemm_nn(Ctx& c, const std::vector<GemmTask>& tasks, int tile) { launch<false, false>(c, tasks, "gemm_nn", tile); }
void gemm_nt(Ctx& c, const std::vector<GemmTask>& tasks) { launch<false, true>(c, tasks, "gemm_nt"); }

// tasks already in device memory (generated by a kernel)
void gemm_nt_dev(Ctx& c, const GemmTask* tasks, int count) {
  if (count <= 0) return;
  ScopedKernelTimer tk(c, "gemm_nt");
  constexpr size_t smem = gemm_smem(GemmCfg<false>::stages);
  ensure_smem_attr(reinterpret_cast<const void*>(k_gemm<false, true>), smem);
  k_gemm<false, true><<<static_cast<unsigned>(count), NT, smem, c.stream>>>(tasks);
  RDD_LAUNCH_CHECK();
}

}  // namespace rdd
