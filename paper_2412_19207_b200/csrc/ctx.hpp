// ctx.hpp — the solver context behind the C ABI: host geometry + device-resident state.
//
// HBM layout (DESIGN.md §Data layout):
//   pts        d x N doubles, axis-major (SoA)           collocation points (uploaded, bit-exact)
//   row_ptr    J+1 ints; row_idx Σrows ints              rows_j: ascending global ids (assembly.hpp:58-64)
//   cov_j/r    N x maxcov ints                           per-point covering (block, local row)
//   Ljet       N x jet_len doubles                       L(x) jets; F  N x C (column-major)
//   S          Σ_j rows_j*m doubles, per-block column-major   unreduced (op_applied/psi) blocks
//   H          Σ_j rows_j*p_j doubles, per-block column-major reduced, equilibrated blocks
//   NB         Σ_pairs p_j1*p_j2 doubles                  normal blocks H_j1ᵀH_j2 (j1 <= j2)
//   P          Σ_i n_i*n_i doubles                        local (pseudo-)inverses (Schwarz)
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/rdd.h"
#include "common.cuh"

namespace rdd {

// Problem on the device: id + operator coefficients over the jet (operators.hpp as c·jet).
struct ProblemDesc {
  int id = 0;
  int d = 2;
  int C = 1;
  int n = 2;          // example1 complexity
  double lo[kMaxDim] = {0, 0, 0, 0}, hi[kMaxDim] = {1, 1, 1, 1};
  double coef[kMaxJet] = {0};
  bool has_exact = true;
};

inline double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct KernelStat {
  double ms = 0.0;
  int64_t launches = 0;
};

struct GemmTask {
  const double* A;
  const double* B;
  double* Cm;
  const int* gA;   // optional row gather for op(A)'s K index (TN mode)
  const int* gB;
  int M, N, K, lda, ldb, ldc;
  int tm, tn;      // tile indices
  double beta;     // C = alpha * op(A) op(B) + beta * C
  double alpha = 1.0;
};

// Caller-supplied inputs (rdd_set_decomposition / points / bases / problem): the reference's
// CartesianDecomposition, PointSet, RandomBasis and a ProblemSpec evaluated at the points.
struct CustomInputs {
  bool has_dec = false, has_pts = false, has_bases = false, has_problem = false;
  int d = 0;
  std::vector<int> counts;
  std::vector<double> dom_lo, dom_hi;           // d
  std::vector<double> lo, hi, ctr, half;        // J x d (geometry.hpp:84-97 sub, centers, half)
  std::vector<int> nbr_ptr, nbr_idx;            // neighbour sets (CSR)
  std::vector<double> pts;                      // N x d, point after point
  int m = 0, act = 0;
  std::vector<double> R, b;                     // J x m x d, J x m
  int C = 1;
  std::vector<double> coef, Ljet, F;            // jet_len(d); N x jet_len(d); N x C (column-major)
};

// Pinned staging for host-built task lists: the H2D copy of a pageable vector blocks the host
// until the stream reaches it (so the GPU idles while the next list is built); two pinned slots
// alternate, each reused only after its previous copy has executed.
struct PinnedStage {
  void* buf[2] = {nullptr, nullptr};
  size_t cap[2] = {0, 0};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  bool used[2] = {false, false};
  int next = 0;
  ~PinnedStage() {
    for (int i = 0; i < 2; ++i) {
      if (buf[i]) cudaFreeHost(buf[i]);
      if (ev[i]) cudaEventDestroy(ev[i]);
    }
  }
  // copies `bytes` from host `src` to device `dst` on `s` through a pinned slot
  void upload(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (!bytes) return;
    const int k = next;
    next ^= 1;
    if (!ev[k]) RDD_CUDA(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
    if (used[k]) RDD_CUDA(cudaEventSynchronize(ev[k]));
    if (cap[k] < bytes) {
      if (buf[k]) RDD_CUDA(cudaFreeHost(buf[k]));
      cap[k] = std::max(bytes, cap[k] * 2);
      RDD_CUDA(cudaHostAlloc(&buf[k], cap[k], cudaHostAllocDefault));
    }
    std::memcpy(buf[k], src, bytes);
    RDD_CUDA(cudaMemcpyAsync(dst, buf[k], bytes, cudaMemcpyHostToDevice, s));
    RDD_CUDA(cudaEventRecord(ev[k], s));
    used[k] = true;
    h2d_counter() += static_cast<int64_t>(bytes);
  }
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  cudaDeviceProp prop{};

  // ---- configuration
  rdd_config cfg{};
  uint64_t seed = 0;
  ProblemDesc prob;                 // id 0 = caller-supplied problem (CustomInputs)
  int d = 2, J = 0, N = 0, m = 0, C = 1, jl = 6;
  CustomInputs custom;

  // ---- host geometry (geometry.hpp:84-185)
  std::vector<double> box_lo, box_hi, box_c, box_h;  // J x 4
  std::vector<int> counts;
  std::vector<std::vector<double>> axis_lo, axis_hi;  // per axis, per index
  std::vector<int> nbr_ptr, nbr_idx;                  // CSR, ascending, includes self
  pinned_vector<double> h_pts;                        // d x N (axis-major), pinned staging
  pinned_vector<double> h_R, h_b;                     // J*m*d (k-major, then axis), J*m

  // ---- device: inputs
  DBuf<double> pts, dbox;  // dbox: J x 16 (lo[4], hi[4], center[4], half[4])
  DBuf<double> daxis;      // per axis: lo/hi interval arrays (offsets in axis_off)
  std::vector<int> axis_off;
  DBuf<int> dnbr_ptr, dnbr_idx;
  DBuf<double> R, bvec;
  DBuf<double> Ljet, Fpt;  // N x jl, N x C

  // ---- device: indexing (K1)
  std::vector<int> h_row_ptr;
  DBuf<int> row_ptr, row_idx;
  int maxcov = 0;
  DBuf<int> cov_j, cov_r, cov_n;
  DBuf<double> ax_lo, ax_hi;          // per-axis box intervals (axis-major), for cover searches
  int ax_counts[kMaxDim] = {1, 1, 1, 1}, ax_stride[kMaxDim] = {0, 0, 0, 0}, ax_off[kMaxDim] = {0, 0, 0, 0};
  long long sum_rows = 0;

  // ---- PCA (K2-K5)
  bool identity_V = true;
  std::vector<int> h_p;            // p_j
  std::vector<int> h_col_off;      // J+1
  int p = 0;
  DBuf<double> S;                  // unreduced sample blocks (Σ rows_j*m)
  std::vector<long long> S_off;    // J+1 (elements)
  DBuf<double> Vred;               // J x m x m (columns 0..p_j-1 used)
  DBuf<double> sigma;              // J x m
  DBuf<int> dp_j;

  // ---- assembled system
  DBuf<double> Hbuf;               // reduced blocks (or alias of S when identity)
  double* H = nullptr;
  std::vector<long long> H_off;    // J+1 (elements)
  DBuf<long long> dH_off;
  DBuf<int> dcol_off;
  DBuf<double> scales;             // p
  DBuf<double> F;                  // N x C (column-major)
  bool assembled = false;
  bool equilibrated = false;

  // ---- normal blocks (assembly.hpp:137-183)
  std::vector<int> nb_j1, nb_j2;   // pairs j1 <= j2 with non-empty row intersection
  std::vector<long long> nb_off;   // element offsets into NB
  DBuf<double> NB;
  std::map<std::pair<int, int>, int> nb_index;
  DBuf<long long> nb_look;         // per neighbour-CSR entry: NB offset or -1
  std::vector<long long> h_nb_look;  // host copy

  // ---- Schwarz (schwarz.hpp)
  int pkind = RDD_PRECOND_NONE;
  std::vector<int> set_ptr, set_idx;  // S_i (CSR)
  std::vector<int> h_owner, h_mult;
  std::vector<int> local_rank;
  std::vector<double> local_cond;
  std::vector<long long> P_off;       // per i: offset of the tile-packed Cholesky factor of A_i
  DBuf<double> P;
  DBuf<int> dset_ptr, dset_idx, dmult, downer;
  DBuf<long long> dP_off;
  // envelope (skyline) of the tile-packed factors: block row k of A_i's factor holds the tiles
  // env_first[k]..k. The blocks of A_i that pair two neighbours of i which do not overlap each
  // other are exact zeros, and Cholesky does not fill in left of a row's first nonzero, so those
  // tiles are neither computed, stored nor read. Tile (k, j) of subdomain i lives at
  // P_off[i] + (env_base[k] + j)·64²; both arrays are indexed at env_off[i] + k. The packed
  // explicit inverses (inv_mode) are dense: first = 0, base = k(k+1)/2.
  std::vector<int> env_off, env_first, env_base;
  DBuf<int> denv_off, denv_first, denv_base;
  double env_entries = 0.0;           // Σ_i scalar entries inside the envelopes of the lower triangles
  int inv_max = 1024;                 // largest local order kept as an explicit inverse ("inv_max" parameter)
  // owner-gather map for the AS/SAS reduction: per column c, list of (i, position)
  DBuf<int> gat_ptr, gat_pos, gat_owner_pos;
  int nmax_local = 0;
  int n_fallback = 0;                 // local blocks that took the eigen pseudo-inverse
  std::vector<int> fallback, local_n;
  size_t schwarz_budget = 0;
  bool inv_mode = false;              // small blocks: packed explicit A_i⁻¹ (one SYMV per apply)
  int qr_rank = 0;                    // numerical rank of the dense QR path          // bytes of gathered A_i per chunk (fixed per context)
  std::map<int, DBuf<double>> fb_store;  // eigen-fallback subdomains: dense pseudo-inverse
  DBuf<double*> dfb_ptr;              // per i: dense pseudo-inverse or nullptr (factor path)
  bool local_cond_exact = false;
  struct GatherTask {
    int i, j1, j2, o1, o2;
    long long nb;
  };
  std::vector<GatherTask> gat_tasks;
  int pca_refine = 0;                 // subspace-refinement steps of the PCA (0 = automatic)
  double pca_stop = 1e-17;            // pivoted-Cholesky stop of PCA stage 1, relative to the first pivot (λ scale)
  double full_rank_cond = 1e9;        // Cholesky path when cond_est(A_i) is below this (DESIGN §4 K8)
  DBuf<double> zloc;                  // Σ n_i
  // RAS owner-row panels (small blocks): per i the rows of A_i⁻¹ that subdomain i owns
  // (p_i x n_i, column-major), the only rows the restricted apply keeps (schwarz.hpp:170-182)
  bool ras_panel = false;
  DBuf<double> Pras;
  DBuf<long long> dras_off;
  DBuf<int> down_off, down_n;
  std::vector<long long> ras_off;
  DBuf<int> apply_order;              // subdomains by local size, largest first (apply CTA order)

  // ---- Krylov
  DBuf<double> work;                  // vectors
  DBuf<double> scal;                  // device scalars
  std::vector<std::vector<double>> hist, true_hist;
  std::vector<int> iters, conv, brk;
  DBuf<double> W;                     // p x C (unscaled)
  DBuf<double> ytmp;                  // N
  DBuf<int2> mv_tiles, mt_tiles;      // (block, first row) / (block, first column) tiles of H·w / Hᵀ·r
  int mv_ntiles = 0, mt_ntiles = 0, mv_rmax = 0;
  DBuf<double> zrows;                 // per-block partial H_j·w_j (row_ptr layout)
  const int* live = nullptr;          // solver status word (0 = running) while a solver graph is captured:
                                      // operator/preconditioner kernels of speculative iterations exit early
  DBuf<int> ent_flat;                 // per (block, local row): flat z indices of the point's covers (-1 pad)
  int ent_w = 0;                      // its width (4 or 8; 0 = not built)
  DBuf<int> mt_part_off, mt_blk_tile0;  // Hᵀ·r row-chunk partials: offset per tile, first tile per block
  DBuf<double> mt_part;
  DBuf<GemmTask> wsg;                 // device-generated GEMM task lists
  int mt_groups = 0;
  size_t mt_smem = 0;

  // ---- evaluation
  std::vector<double> approx, exact;  // M x C (host copies)
  DBuf<double> ref2;                  // example2 reference field (res x res, level-major)
  int ref2_res = 0;
  rdd_summary sum{};

  // ---- instrumentation
  std::map<std::string, KernelStat> stats;
  bool timing = false;
  bool verbose = false;
  size_t cg_graph_kernels = 0;

  double* wk(size_t count) { return work.ensure(count); }
  // persistent grow-only workspaces for large temporaries (no per-call pool traffic)
  std::map<std::string, DBuf<double>> wsd;
  double* ws(const std::string& name, size_t count) { return wsd[name].ensure(count > 0 ? count : 1); }
  cudaEvent_t ev[8] = {nullptr};
  PinnedStage stage;                  // task-list uploads (gemm.cu)
};

// timing helper: records device time of a kernel family when ctx.timing is on
struct ScopedKernelTimer {
  Ctx& c;
  const char* fam;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  ScopedKernelTimer(Ctx& ctx, const char* family) : c(ctx), fam(family) {
    if (c.timing) {
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, c.stream);
    }
  }
  ~ScopedKernelTimer() {
    if (c.timing) {
      cudaEventRecord(e1, c.stream);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      auto& s = c.stats[fam];
      s.ms += ms;
      s.launches += 1;
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    }
  }
};

// ---- module entry points (one per reference function family) -----------------------
// host_setup.cpp
void setup_problem(Ctx& c, const rdd_config& cfg, uint64_t seed);  // problems + geometry + bases + points
void reference_example2_grid(int res, std::vector<double>& v);     // problems.hpp:219-264
void upload_inputs(Ctx& c);
void setup_custom(Ctx& c, const rdd_config& cfg);                  // the same from CustomInputs
// index.cu (K1)
void build_index(Ctx& c);
// problem.cu
void eval_problem(Ctx& c);
void upload_custom_problem(Ctx& c);  // caller L jets and F instead of eval_problem
// assemble.cu (K2)
void assemble_samples(Ctx& c, int kind, double* out, const std::vector<long long>& off);
// pca.cu (K3-K5)
void run_pca(Ctx& c);
// equil.cu (K6) + matvec.cu (K9/K10)
void column_norms_scale(Ctx& c, bool equilibrate);
void matvec_dev(Ctx& c, const double* w, double* y);
// dot_with/dot_part: per-CTA partials (ceil(p/256)) of dot_with·out, fused into the last kernel
void matvec_t_dev(Ctx& c, const double* r, double* out, const double* dot_with = nullptr, double* dot_part = nullptr);
// normal.cu (K7)
void build_normal_blocks(Ctx& c);
void normal_apply_dev(Ctx& c, const double* w, double* out);
void normal_operator(Ctx& c, const double* w, double* out);  // runner.hpp:232-234
bool normal_operator_dot(Ctx& c, const double* w, double* out, double* dot_part);
void normal_two_pass_dev(Ctx& c, const double* w, double* out, double* dot_part);
// schwarz.cu (K8/K11)
struct SchwarzIndex {  // host side of build_index_sets (schwarz.hpp:39-61) + the column gather map
  std::vector<int> set_ptr, set_idx, mult, n, gp, gpos, owner_pos;
};
SchwarzIndex prepare_schwarz_index(const Ctx& c);
void build_schwarz(Ctx& c, int kind, SchwarzIndex* pre = nullptr);
// pzz/pzv: per-CTA partials (ceil(p/256)) of z·z and z·v, fused into the reduction kernel
void precond_apply_dev(Ctx& c, const double* v, double* z, bool transpose, double* pzz = nullptr, double* pzv = nullptr);
void gather_locals(Ctx& c, const std::vector<int>& which, DBuf<double>& out, const std::vector<long long>& off,
                   bool lower_only = false);
void refresh_local_cond(Ctx& c);
size_t device_available(Ctx& c);
void release_scratch(Ctx& c);
// krylov.cu (K12/K13)
void qr_solve_dev(Ctx& c);
void solve_all(Ctx& c, int solver, double tol, int max_iter, int restart);
// evaluate.cu (K14)
void evaluate(Ctx& c, const int* test_res);
// runner.hpp:105-127 evaluate_solution at caller points (M x d, point after point) with caller W
// (p x C, column-major, unscaled) or the solved one (W = nullptr), caller L values (M) and G
// values (M x C, column-major; nullptr = 0); out M x C column-major
void evaluate_at(Ctx& c, long long M, const double* pts, const double* W, const double* Lv, const double* Gv,
                 double* out);
// gemm.cu
// tile = CTA tile edge, 64 or 80 (the tasks' (tm, tn) count tiles of that size), or 6480 = 64 rows x 80 columns
void gemm_tn(Ctx& c, const std::vector<GemmTask>& tasks, int tile = 64);  // C = Aᵀ B (A: K x M, B: K x N col-major)
void gemm_nn(Ctx& c, const std::vector<GemmTask>& tasks, int tile = 64);  // C = A B  (A: M x K, B: K x N col-major)
void gemm_nn_wide(Ctx& c, const std::vector<GemmTask>& tasks);  // same, 64 x 128 tiles (tn in units of 128)
void gemm_nt(Ctx& c, const std::vector<GemmTask>& tasks);
void gemm_nt_dev(Ctx& c, const GemmTask* tasks, int count);  // C = A Bᵀ (A: M x K, B: N x K col-major)
void project_blocks(Ctx& c);
void ensure_col_owner(Ctx& c);
// cholesky.cu
// ids: the subdomain of every batch entry (its envelope: c.env_*)
void batched_cholesky_pack(Ctx& c, double* A, const std::vector<int>& ids, const std::vector<int>& n,
                           const std::vector<long long>& off, double* P, const std::vector<long long>& poff,
                           std::vector<int>& fail, std::vector<double>& frob_A, bool inverse = false,
                           std::vector<double>* frob_P = nullptr, double** Pfull_out = nullptr);
long long packed_chol_size(int n);
long long packed_inverse_size(int n);
size_t chol_solve_smem(int nmax, bool inverse);
std::vector<double> batched_inv_power(Ctx& c, const double* P, const std::vector<int>& ids, const std::vector<int>& n,
                                      const std::vector<long long>& poff, int iters, bool inverse);
void chol_apply(Ctx& c, const double* v, bool transpose, double* zloc);
void build_ras_panels(Ctx& c);                                        // after build_schwarz (RAS, inverse mode)
void ras_panel_apply(Ctx& c, const double* v, bool transpose, double* zloc);
std::vector<double> batched_power(Ctx& c, const double* A, const std::vector<int>& n,
                                  const std::vector<long long>& off, int iters);
// diag.cu (§8f row 4: krylov.hpp:403-440 dense diagnostics)
void check_dense_cap(long long n, int cap);
void dense_eigenvalues_dev(Ctx& c, double* A, int n, std::vector<double>& wr, std::vector<double>& wi);
void symmetric_eigenvalues_dev(Ctx& c, double* A, int n, std::vector<double>& ev);
void singular_values_dev(Ctx& c, double* A, int m, int n, std::vector<double>& sv);
double condition_from(const std::vector<double>& sv);
void spectra(Ctx& c, int cap, std::vector<double>& nre, std::vector<double>& nim, std::vector<double>* pre,
             std::vector<double>* pim, double* cond_n, double* cond_p);
// jacobi.cu
struct EigOpts {
  int absolute = 0;       // 1: |a_pq| > tol·max|a_ii| (backward stable); 0: |a_pq| > tol·sqrt|a_pp a_qq| (graded)
  double tol = 1e-14;
  double floor_rel = 0.0, floor_abs = 0.0;  // no rotation between two directions both below the floor
  double conv_rel = 0.0, conv_abs = 0.0;    // convergence judged on directions above this level only
  double conv_angle = 0.0;                  // ... and on rotations with |tan θ| above this
  int max_sweeps = 40;
};
double bench_syevj(Ctx& c, int n, int B, int sweeps);
void batched_syevj(Ctx& c, double* A, double* V, double* evals, const std::vector<int>& n,
                   const std::vector<long long>& offA, const EigOpts& o);

}  // namespace rdd
