// krylov.cu — K12/K13: PCG and GMRES(m) drivers (krylov.hpp:106-156, 275-389).
//
// All scalars live on the device. Reductions are deterministic two-stage (fixed-size grid of
// per-CTA partials, summed in order by the consumer), so reruns are bit-identical like the
// reference's (test_runner.cpp:109-117). CG keeps its control state (iteration, status, rz,
// histories) on the device: every kernel of an iteration is a no-op once the status leaves
// RUNNING, so an iteration is a fixed sequence of launches, captured once into a CUDA graph of
// eight iterations that the host replays, reading the status word once per replay.
// GMRES uses classical Gram–Schmidt applied twice (CGS2) — orthogonality equivalent to the
// reference's MGS twice, but as two batched projections instead of 2(k+1) sequential ones. The
// Hessenberg column, the Givens rotations, the residual estimate and the small triangular solve
// for the diagnostic true residual run in one warp on the device (k_gm_step); Arnoldi steps are
// launched in chunks with one status read per chunk.
#include <cmath>
#include <cstring>
#include <map>
#include <utility>

#include "ctx.hpp"

namespace rdd {

namespace {

constexpr int kRB = 120;   // reduction grid (CTAs)
constexpr int kRT = 256;

enum { ST_RUNNING = 0, ST_CONVERGED = 1, ST_BREAKDOWN = 2, ST_MAXITER = 3 };

// device control block for CG
struct CgState {
  int status;
  int it;
  int max_iter;
  int pad;
  double tol, z0, bnorm, rz, beta;
};

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[kRT / 32];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < kRT / 32 ? sh[threadIdx.x] : 0.0;
    t = warp_sum(t);
  }
  __syncthreads();
  return t;  // valid in thread 0
}

// partial sums are reduced by one warp in a fixed order (warp_sum_parts): deterministic, and
// every warp that needs the scalar computes the identical value


__global__ void k_dot_part(const double* __restrict__ x, const double* __restrict__ y, int n,
                           double* __restrict__ part, const int* __restrict__ live = nullptr) {
  if (live && *live) return;
  double s = 0.0;
  for (int i = blockIdx.x * kRT + threadIdx.x; i < n; i += kRB * kRT) s += x[i] * y[i];
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_dot2_part(const double* __restrict__ a, const double* __restrict__ b, const double* __restrict__ c,
                            int n, double* __restrict__ part_ab, double* __restrict__ part_ac) {
  double s1 = 0.0, s2 = 0.0;
  for (int i = blockIdx.x * kRT + threadIdx.x; i < n; i += kRB * kRT) {
    s1 += a[i] * b[i];
    s2 += a[i] * c[i];
  }
  s1 = block_sum(s1);
  s2 = block_sum(s2);
  if (threadIdx.x == 0) {
    part_ab[blockIdx.x] = s1;
    part_ac[blockIdx.x] = s2;
  }
}

// CG setup after z = M b: z0 = ‖z‖, rz = r·z, p = z
__global__ void k_cg_init(CgState* st, const double* __restrict__ pz, const double* __restrict__ prz,
                          const double* __restrict__ pbb, double* hist, double* thist, int npz, int npb) {
  const double zz = warp_sum_parts(pz, npz), rz = warp_sum_parts(prz, npz), bb = warp_sum_parts(pbb, npb);
  if (threadIdx.x != 0) return;
  st->z0 = sqrt(zz);
  st->bnorm = sqrt(bb);
  st->rz = rz;
  st->it = 0;
  if (st->z0 == 0.0) {
    st->status = ST_CONVERGED;
    hist[0] = 0.0;
    thist[0] = 0.0;
  } else {
    st->status = st->max_iter > 0 ? ST_RUNNING : ST_MAXITER;
    hist[0] = 1.0;
    thist[0] = st->bnorm > 0.0 ? 1.0 : 0.0;
  }
}

// alpha = rz / pAp; breakdown check (krylov.hpp:132-135); x += αp; r -= αAp; partial ‖r‖²
__global__ void k_cg_update(CgState* st, const double* __restrict__ ppap, double* __restrict__ x,
                            double* __restrict__ r, const double* __restrict__ p, const double* __restrict__ Ap, int n,
                            double* __restrict__ prr, int* brk_flag, int npap) {
  if (st->status != ST_RUNNING) return;
  const double pAp = warp_sum_parts(ppap, npap);
  const double rz = st->rz;
  if (pAp <= 0.0 || rz == 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *brk_flag = 1;
    return;
  }
  const double alpha = rz / pAp;
  double s = 0.0;
  for (int i = blockIdx.x * kRT + threadIdx.x; i < n; i += kRB * kRT) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * Ap[i];
    r[i] = ri;
    s += ri * ri;
  }
  s = block_sum(s);
  if (threadIdx.x == 0) prr[blockIdx.x] = s;
}

// rel = ‖z‖/‖z0‖, histories, convergence, beta (krylov.hpp:139-151)
__global__ void k_cg_finish(CgState* st, const double* __restrict__ pzz, const double* __restrict__ prz,
                            const double* __restrict__ prr, double* hist, double* thist, int* brk_flag, int npz) {
  if (st->status != ST_RUNNING) return;
  if (*brk_flag) {
    if (threadIdx.x == 0) st->status = ST_BREAKDOWN;
    return;
  }
  const double zz = warp_sum_parts(pzz, npz), rzn = warp_sum_parts(prz, npz), rr = warp_sum_parts(prr, kRB);
  if (threadIdx.x != 0) return;
  const double rel = sqrt(zz) / st->z0;
  const int it = st->it + 1;
  hist[it] = rel;
  thist[it] = st->bnorm > 0.0 ? sqrt(rr) / st->bnorm : sqrt(rr);
  st->it = it;
  if (rel <= st->tol) {
    st->status = ST_CONVERGED;
    return;
  }
  st->beta = rzn / st->rz;
  st->rz = rzn;
  if (it >= st->max_iter) st->status = ST_MAXITER;
}

__global__ void k_cg_p(const CgState* st, double* __restrict__ p, const double* __restrict__ z, int n) {
  if (st->status != ST_RUNNING) return;
  const double beta = st->beta;
  for (int i = blockIdx.x * kRT + threadIdx.x; i < n; i += kRB * kRT) p[i] = z[i] + beta * p[i];
}

__global__ void k_copy(double* __restrict__ dst, const double* __restrict__ src, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[i];
}
__global__ void k_fill(double* __restrict__ dst, double v, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = v;
}
__global__ void k_sub(double* __restrict__ out, const double* __restrict__ a, const double* __restrict__ b, int n,
                      const int* __restrict__ live = nullptr) {
  if (live && *live) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = a[i] - b[i];
}
__global__ void k_scale_to(double* __restrict__ out, const double* __restrict__ in, const double* s, int n,
                           int invert) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = invert ? in[i] / s[i] : in[i];
}

// GMRES: h[k] = V[:,k]ᵀ w for k < nk, one CTA per basis vector (fixed-order reduction)
__global__ void k_multidot(const double* __restrict__ V, long long ldv, const double* __restrict__ w, int n,
                           double* __restrict__ h, const int* __restrict__ live = nullptr) {
  if (live && *live) return;
  const int k = blockIdx.x;
  const double* v = V + k * ldv;
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += kRT) s += v[i] * w[i];
  s = block_sum(s);
  if (threadIdx.x == 0) h[k] = s;
}
// w -= V h (nk columns); optionally accumulate h into hacc
__global__ void k_multiaxpy(const double* __restrict__ V, long long ldv, double* __restrict__ w, int n,
                            const double* __restrict__ h, int nk, const int* __restrict__ live = nullptr) {
  if (live && *live) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double s = w[i];
    for (int k = 0; k < nk; ++k) s -= h[k] * V[k * ldv + i];
    w[i] = s;
  }
}
// x += V y
__global__ void k_combine(const double* __restrict__ V, long long ldv, const double* __restrict__ y, int nk,
                          const double* __restrict__ x0, double* __restrict__ x, int n,
                          const int* __restrict__ live = nullptr) {
  if (live && *live) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double s = x0[i];
    for (int k = 0; k < nk; ++k) s += y[k] * V[k * ldv + i];
    x[i] = s;
  }
}
__global__ void k_scal_div(double* __restrict__ out, const double* __restrict__ in, double s, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = in[i] / s;
}


// ---- GMRES(m) cycle on the device (krylov.hpp:275-389): the Hessenberg column, the Givens
// rotations, the residual estimate and the stopping tests of each Arnoldi step run in one warp, so
// the host launches whole chunks of steps without reading anything back; steps launched after the
// stop exit on the status word (Arnoldi is append-only, so the stopped state is exact).
enum { GM_RUN = 0, GM_CONV = 1, GM_BREAK = 2, GM_MAXIT = 3, GM_CYCLE = 4 };
struct GmState {
  int stop;   // GM_*
  int tr;     // 0 while the true residual of the latest step is pending
  int it;     // iterations so far (all cycles)
  int k;      // steps done in this cycle
  int max_it, len, ident, true_res;
  double gnorm0, bnorm, tol, hnext;
};

// step k: H[:, k] = hA + hB (CGS2), hnext = ‖w‖; previous rotations, new rotation, g; residual
// estimate; stopping tests in the reference's order (breakdown, converged/lucky, cap, cycle end)
__global__ void k_gm_step(GmState* st, const double* __restrict__ hA, const double* __restrict__ hB,
                          const double* __restrict__ part, int k, double* __restrict__ H, int ldh,
                          double* __restrict__ cs, double* __restrict__ sn, double* __restrict__ g,
                          double* __restrict__ y, double* __restrict__ hist, double* __restrict__ thist) {
  if (st->stop != GM_RUN) return;
  const double hnext = sqrt(warp_sum_parts(part, kRB));
  if (threadIdx.x != 0) return;
  double* col = H + static_cast<long long>(k) * ldh;
  for (int i = 0; i <= k; ++i) col[i] = hA[i] + hB[i];
  col[k + 1] = hnext;
  for (int i = 0; i < k; ++i) {
    const double t = cs[i] * col[i] + sn[i] * col[i + 1];
    col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1];
    col[i] = t;
  }
  const double denom = hypot(col[k], col[k + 1]);
  if (denom == 0.0) {
    st->stop = GM_BREAK;
    return;
  }
  cs[k] = col[k] / denom;
  sn[k] = col[k + 1] / denom;
  col[k] = denom;
  col[k + 1] = 0.0;
  g[k + 1] = -sn[k] * g[k];
  g[k] *= cs[k];
  const double rel = fabs(g[k + 1]) / st->gnorm0;
  const int it = ++st->it;
  st->k = k + 1;
  st->hnext = hnext;
  hist[it] = rel;
  if (st->ident) {
    thist[it] = rel;
  } else if (st->true_res) {  // y for the diagnostic true residual (krylov.hpp:360-367)
    for (int i = k; i >= 0; --i) {
      double s = g[i];
      for (int j = i + 1; j <= k; ++j) s -= H[i + static_cast<long long>(j) * ldh] * y[j];
      y[i] = s / H[i + static_cast<long long>(i) * ldh];
    }
    st->tr = 0;
  } else {
    thist[it] = -1.0;
  }
  if (rel <= st->tol || hnext == 0.0) st->stop = GM_CONV;
  else if (it >= st->max_it) st->stop = GM_MAXIT;
  else if (k + 1 == st->len) st->stop = GM_CYCLE;
}
// w /= hnext (skipped once stopped, and for hnext = 0)
__global__ void k_gm_scale(GmState* st, double* __restrict__ w, int n) {
  if (st->stop != GM_RUN) return;
  const double h = st->hnext;
  if (h == 0.0) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) w[i] = w[i] / h;
}
__global__ void k_gm_thist(GmState* st, const double* __restrict__ part, double* __restrict__ thist) {
  if (st->tr != 0) return;
  const double rn = sqrt(warp_sum_parts(part, kRB));
  if (threadIdx.x != 0) return;
  thist[st->it] = st->bnorm > 0.0 ? rn / st->bnorm : 0.0;
  st->tr = 1;
}
// y = R⁻¹ g for the kk steps of the cycle (back substitution on the rotated Hessenberg)
__global__ void k_gm_ysolve(const double* __restrict__ H, int ldh, const double* __restrict__ g, int kk,
                            double* __restrict__ y) {
  if (threadIdx.x != 0) return;
  for (int i = kk - 1; i >= 0; --i) {
    double s = g[i];
    for (int j = i + 1; j < kk; ++j) s -= H[i + static_cast<long long>(j) * ldh] * y[j];
    y[i] = s / H[i + static_cast<long long>(i) * ldh];
  }
}

struct Vecs {
  int n;
  Ctx* c;
  void copy(double* d, const double* s) {
    k_copy<<<kRB, kRT, 0, c->stream>>>(d, s, n);
    RDD_LAUNCH_CHECK();
  }
  void fill(double* d, double v) {
    k_fill<<<kRB, kRT, 0, c->stream>>>(d, v, n);
    RDD_LAUNCH_CHECK();
  }
};

}  // namespace

// A(w) = Hᵀ(H w) (runner.hpp:232-234) or the block-sparse HᵀH
void normal_operator(Ctx& c, const double* w, double* out) { normal_operator_dot(c, w, out, nullptr); }

// the normal operator; with dot_part, also per-CTA partials (ceil(p/256)) of w·out when the
// formulation produces them in its last kernel (returns whether it did)
bool normal_operator_dot(Ctx& c, const double* w, double* out, double* dot_part) {
  if (c.cfg.op_form == RDD_OPERATOR_NORMAL && c.NB.p) {
    normal_apply_dev(c, w, out);
    return false;
  }
  normal_two_pass_dev(c, w, out, dot_part);
  return dot_part != nullptr;
}

// z = M v; with pzz/pzv, also per-CTA partials (ceil(p/256)) of z·z and z·v (returns whether)
static bool precond(Ctx& c, const double* v, double* z, double* pzz = nullptr, double* pzv = nullptr) {
  if (c.pkind == RDD_PRECOND_NONE) {
    k_copy<<<kRB, kRT, 0, c.stream>>>(z, v, c.p);
    RDD_LAUNCH_CHECK();
    return false;
  }
  precond_apply_dev(c, v, z, false, pzz, pzv);
  return pzz != nullptr;
}

static double dot_host(Ctx& c, const double* x, const double* y, int n, double* part) {
  k_dot_part<<<kRB, kRT, 0, c.stream>>>(x, y, n, part);
  RDD_LAUNCH_CHECK();
  double h[kRB];
  RDD_CUDA(cudaMemcpyAsync(h, part, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
  RDD_CUDA(cudaStreamSynchronize(c.stream));
  double s = 0.0;
  for (int i = 0; i < kRB; ++i) s += h[i];
  return s;
}

// ---------------------------------------------------------------- CG (krylov.hpp:106-156)
struct CgGraph {
  cudaGraphExec_t exec = nullptr;
  ~CgGraph() {
    if (exec) cudaGraphExecDestroy(exec);
  }
};

static void cg_solve(Ctx& c, const double* b, double* x, double tol, int max_iter, int comp) {
  const int n = c.p;
  double* r = c.wk(static_cast<size_t>(n) * 8);
  double* z = r + n;
  double* pv = z + n;
  double* Ap = pv + n;
  const int ps = std::max(kRB, ceil_div(n, 256));  // partial slots: kRB dot CTAs or fused ceil(p/256)
  double* sc = c.wsd["cg.part"].ensure(5 * static_cast<size_t>(ps));
  double *P0 = sc, *P1 = sc + ps, *P2 = sc + 2 * ps, *P3 = sc + 3 * ps, *P4 = sc + 4 * ps;
  DBuf<CgState> st;
  DBuf<int> brk;
  DBuf<double> hist, thist;
  hist.ensure(max_iter + 2);
  thist.ensure(max_iter + 2);
  brk.zero(1, c.stream);
  CgState h0{};
  h0.status = ST_RUNNING;
  h0.max_iter = max_iter;
  h0.tol = tol;
  st.upload(&h0, 1, c.stream);
  Vecs V{n, &c};
  V.fill(x, 0.0);
  V.copy(r, b);
  // dot partials: fused into the operator's / preconditioner's last kernel where they exist
  // (ceil(p/256) partials), else the kRB-CTA dot kernels
  const int npf = ceil_div(n, 256);
  int npz = npf;
  if (!precond(c, r, z, P0, P1)) {
    k_dot2_part<<<kRB, kRT, 0, c.stream>>>(z, z, r, n, P0, P1);  // (z·z, z·r)
    RDD_LAUNCH_CHECK();
    npz = kRB;
  }
  k_dot_part<<<kRB, kRT, 0, c.stream>>>(b, b, n, P2);
  RDD_LAUNCH_CHECK();
  k_cg_init<<<1, 32, 0, c.stream>>>(st.p, P0, P1, P2, hist.p, thist.p, npz, kRB);
  RDD_LAUNCH_CHECK();
  V.copy(pv, z);

  // one iteration = fixed launch sequence; capture once, replay in chunks with a device status
  auto iteration = [&]() {
    int npap = npf;
    if (!normal_operator_dot(c, pv, Ap, P0)) {
      k_dot_part<<<kRB, kRT, 0, c.stream>>>(pv, Ap, n, P0);
      RDD_LAUNCH_CHECK();
      npap = kRB;
    }
    k_cg_update<<<kRB, kRT, 0, c.stream>>>(st.p, P0, x, r, pv, Ap, n, P4, brk.p, npap);
    RDD_LAUNCH_CHECK();
    int npzz = npf;
    if (!precond(c, r, z, P2, P3)) {
      k_dot2_part<<<kRB, kRT, 0, c.stream>>>(z, z, r, n, P2, P3);
      RDD_LAUNCH_CHECK();
      npzz = kRB;
    }
    k_cg_finish<<<1, 32, 0, c.stream>>>(st.p, P2, P3, P4, hist.p, thist.p, brk.p, npzz);
    RDD_LAUNCH_CHECK();
    k_cg_p<<<kRB, kRT, 0, c.stream>>>(st.p, pv, z, n);
    RDD_LAUNCH_CHECK();
  };
  const int chunk = 8;
  c.ytmp.ensure(c.N);  // no allocations inside the capture
  CgGraph g;
  const bool timing = c.timing;
  c.timing = false;  // no event records inside capture
  // the operator/preconditioner kernels of iterations after the stop exit early
  struct LiveScope {
    Ctx& c;
    LiveScope(Ctx& cc, const int* p) : c(cc) { c.live = p; }
    ~LiveScope() { c.live = nullptr; }
  };
  {
    LiveScope ls(c, &st.p->status);
    cudaGraph_t graph;
    const int64_t before = launch_counter();
    RDD_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    for (int k = 0; k < chunk; ++k) iteration();
    RDD_CUDA(cudaStreamEndCapture(c.stream, &graph));
    c.cg_graph_kernels = static_cast<size_t>(launch_counter() - before);  // captured, not launched
    launch_counter() = before;
    RDD_CUDA(cudaGraphInstantiate(&g.exec, graph, 0));
    cudaGraphDestroy(graph);
  }
  c.timing = timing;
  const size_t graph_nodes = c.cg_graph_kernels;
  CgState hs{};
  for (int done = 0;;) {
    RDD_CUDA(cudaGraphLaunch(g.exec, c.stream));
    launch_counter() += static_cast<int64_t>(graph_nodes);
    done += chunk;
    RDD_CUDA(cudaMemcpyAsync(&hs, st.p, sizeof(CgState), cudaMemcpyDeviceToHost, c.stream));
    RDD_CUDA(cudaStreamSynchronize(c.stream));
    if (hs.status != ST_RUNNING) break;
    if (done > max_iter + chunk) break;
  }
  const int it = hs.it;
  c.hist[comp].resize(it + 1);
  c.true_hist[comp].resize(it + 1);
  hist.download(c.hist[comp].data(), it + 1, c.stream);
  thist.download(c.true_hist[comp].data(), it + 1, c.stream);
  RDD_CUDA(cudaStreamSynchronize(c.stream));
  if (hs.status == ST_CONVERGED && hs.z0 == 0.0) {
    c.hist[comp] = {0.0};
    c.true_hist[comp] = {0.0};
  }
  c.iters[comp] = it;
  c.conv[comp] = hs.status == ST_CONVERGED;
  c.brk[comp] = hs.status == ST_BREAKDOWN;
}

// ---------------------------------------------------------------- GMRES (krylov.hpp:275-389)
static void gmres_solve(Ctx& c, const double* b, double* x, double tol, int max_iter, int restart, int comp) {
  const int n = c.p;
  const bool ident = c.pkind == RDD_PRECOND_NONE;
  const bool true_res = c.cfg.true_residual != 0;
  double* part = c.scal.ensure(8 * kRB + 64);
  double* part2 = part + 2 * kRB;
  auto& hist = c.hist[comp];
  auto& thist = c.true_hist[comp];
  hist.clear();
  thist.clear();
  double* t1 = c.wk(static_cast<size_t>(n) * 4);
  double* t2 = t1 + n;
  double* xk = t2 + n;
  double* rr = xk + n;
  Vecs Vv{n, &c};
  const double bnorm = std::sqrt(dot_host(c, b, b, n, part));
  precond(c, b, t1);
  const double gnorm0 = std::sqrt(dot_host(c, t1, t1, n, part));
  Vv.fill(x, 0.0);
  c.iters[comp] = 0;
  c.conv[comp] = 0;
  c.brk[comp] = 0;
  if (gnorm0 == 0.0) {
    hist = {0.0};
    thist = {0.0};
    c.conv[comp] = 1;
    return;
  }
  const int cycle_len = restart > 0 ? restart : std::min(max_iter, n);
  if (restart == 0 && cycle_len > 4096)
    throw std::runtime_error("full GMRES basis of " + std::to_string(cycle_len) +
                             " vectors exceeds the cap; configure gmres_restart");
  const int ldh = cycle_len + 1;
  DBuf<double> Vb, hv, Hd, dhist, dthist;
  Vb.ensure(static_cast<size_t>(cycle_len + 1) * n);
  hv.ensure(static_cast<size_t>(5 * (cycle_len + 2)));  // hA, hB, cs, sn, g / y
  double *hA = hv.p, *hB = hA + (cycle_len + 2), *cs = hB + (cycle_len + 2), *sn = cs + (cycle_len + 2),
         *g = sn + (cycle_len + 2);
  DBuf<double> yv;
  yv.ensure(cycle_len + 2);
  Hd.ensure(static_cast<size_t>(ldh) * cycle_len);
  dhist.ensure(static_cast<size_t>(max_iter) + 2);
  dthist.ensure(static_cast<size_t>(max_iter) + 2);
  DBuf<GmState> st;
  st.ensure(1);
  GmState hs{};
  double one = 1.0, tb = bnorm > 0.0 ? 1.0 : 0.0;
  RDD_CUDA(cudaMemcpyAsync(dhist.p, &one, sizeof(double), cudaMemcpyHostToDevice, c.stream));
  RDD_CUDA(cudaMemcpyAsync(dthist.p, &tb, sizeof(double), cudaMemcpyHostToDevice, c.stream));
  int it = 0;
  bool converged = false, breakdown = false;
  struct LiveScope {
    Ctx& c;
    explicit LiveScope(Ctx& cc) : c(cc) {}
    ~LiveScope() { c.live = nullptr; }
  } ls(c);
  constexpr int kChunk = 8;  // Arnoldi steps per captured graph, one status read per replay
  // one Arnoldi step k (krylov.hpp:317-350): every kernel is a no-op once the status word stops
  // the cycle, so a chunk of steps is a fixed launch sequence, captured once per (k0, k1) and
  // replayed in every cycle
  auto step = [&](int k) {
    double* vk = Vb.p + static_cast<size_t>(k) * n;
    double* w = Vb.p + static_cast<size_t>(k + 1) * n;
    c.live = &st.p->stop;
    if (ident) {
      normal_operator(c, vk, w);
    } else {
      normal_operator(c, vk, t1);
      precond(c, t1, w);
    }
    // CGS2: h = Vᵀw; w -= V h (twice)
    k_multidot<<<k + 1, kRT, 0, c.stream>>>(Vb.p, n, w, n, hA, c.live);
    k_multiaxpy<<<kRB, kRT, 0, c.stream>>>(Vb.p, n, w, n, hA, k + 1, c.live);
    k_multidot<<<k + 1, kRT, 0, c.stream>>>(Vb.p, n, w, n, hB, c.live);
    k_multiaxpy<<<kRB, kRT, 0, c.stream>>>(Vb.p, n, w, n, hB, k + 1, c.live);
    k_dot_part<<<kRB, kRT, 0, c.stream>>>(w, w, n, part, c.live);
    RDD_LAUNCH_CHECK();
    k_gm_step<<<1, 32, 0, c.stream>>>(st.p, hA, hB, part, k, Hd.p, ldh, cs, sn, g, yv.p, dhist.p, dthist.p);
    RDD_LAUNCH_CHECK();
    k_gm_scale<<<kRB, kRT, 0, c.stream>>>(st.p, w, n);
    RDD_LAUNCH_CHECK();
    if (!ident && true_res) {  // diagnostic true residual ‖b − A x_k‖ (krylov.hpp:360-367)
      c.live = &st.p->tr;
      k_combine<<<kRB, kRT, 0, c.stream>>>(Vb.p, n, yv.p, k + 1, x, xk, n, c.live);
      RDD_LAUNCH_CHECK();
      normal_operator(c, xk, t1);
      k_sub<<<kRB, kRT, 0, c.stream>>>(rr, b, t1, n, c.live);
      k_dot_part<<<kRB, kRT, 0, c.stream>>>(rr, rr, n, part2, c.live);
      RDD_LAUNCH_CHECK();
      k_gm_thist<<<1, 32, 0, c.stream>>>(st.p, part2, dthist.p);
      RDD_LAUNCH_CHECK();
    }
    c.live = nullptr;
  };
  struct GraphCache {
    std::map<std::pair<int, int>, std::pair<cudaGraphExec_t, size_t>> g;
    ~GraphCache() {
      for (auto& kv : g) cudaGraphExecDestroy(kv.second.first);
    }
  } graphs;
  while (it < max_iter && !converged && !breakdown) {
    normal_operator(c, x, t1);
    k_sub<<<kRB, kRT, 0, c.stream>>>(t2, b, t1, n);  // b - A x
    RDD_LAUNCH_CHECK();
    if (ident) Vv.copy(t1, t2);
    else precond(c, t2, t1);
    const double beta = std::sqrt(dot_host(c, t1, t1, n, part));
    if (beta / gnorm0 <= tol) {
      converged = true;
      break;
    }
    const int len = std::min(cycle_len, max_iter - it);
    k_scal_div<<<kRB, kRT, 0, c.stream>>>(Vb.p, t1, beta, n);
    RDD_LAUNCH_CHECK();
    GmState s0{};
    s0.stop = GM_RUN;
    s0.tr = 1;
    s0.it = it;
    s0.max_it = max_iter;
    s0.len = len;
    s0.ident = ident ? 1 : 0;
    s0.true_res = true_res ? 1 : 0;
    s0.gnorm0 = gnorm0;
    s0.bnorm = bnorm;
    s0.tol = tol;
    st.upload(&s0, 1, c.stream);
    RDD_CUDA(cudaMemcpyAsync(g, &beta, sizeof(double), cudaMemcpyHostToDevice, c.stream));
    for (int k0 = 0; k0 < len; k0 += kChunk) {
      const int k1 = std::min(len, k0 + kChunk);
      auto key = std::make_pair(k0, k1);
      auto gi = graphs.g.find(key);
      if (gi == graphs.g.end()) {  // first use of this chunk shape: capture its launches once
        const bool timing = c.timing;
        c.timing = false;
        const int64_t before = launch_counter();
        cudaGraph_t graph;
        RDD_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
        for (int k = k0; k < k1; ++k) step(k);
        RDD_CUDA(cudaStreamEndCapture(c.stream, &graph));
        const size_t nodes = static_cast<size_t>(launch_counter() - before);
        launch_counter() = before;
        cudaGraphExec_t exec = nullptr;
        RDD_CUDA(cudaGraphInstantiate(&exec, graph, 0));
        cudaGraphDestroy(graph);
        c.timing = timing;
        gi = graphs.g.emplace(key, std::make_pair(exec, nodes)).first;
      }
      RDD_CUDA(cudaGraphLaunch(gi->second.first, c.stream));
      launch_counter() += static_cast<int64_t>(gi->second.second);
      st.download(&hs, 1, c.stream);
      RDD_CUDA(cudaStreamSynchronize(c.stream));
      if (hs.stop != GM_RUN) break;
    }
    it = hs.it;
    if (hs.k > 0) {  // x += V y
      k_gm_ysolve<<<1, 32, 0, c.stream>>>(Hd.p, ldh, g, hs.k, yv.p);
      RDD_LAUNCH_CHECK();
      k_combine<<<kRB, kRT, 0, c.stream>>>(Vb.p, n, yv.p, hs.k, x, x, n);
      RDD_LAUNCH_CHECK();
    }
    if (hs.stop == GM_CONV) converged = true;
    if (hs.stop == GM_BREAK) breakdown = true;
    if (restart == 0 && !converged && !breakdown && it < max_iter && hs.k == cycle_len) break;
  }
  c.iters[comp] = it;
  hist.resize(it + 1);
  thist.resize(it + 1);
  dhist.download(hist.data(), it + 1, c.stream);
  dthist.download(thist.data(), it + 1, c.stream);
  RDD_CUDA(cudaStreamSynchronize(c.stream));
  c.conv[comp] = converged;
  c.brk[comp] = breakdown;
}


static void precond_t(Ctx& c, const double* v, double* z) {
  if (c.pkind == RDD_PRECOND_NONE) {
    k_copy<<<kRB, kRT, 0, c.stream>>>(z, v, c.p);
    RDD_LAUNCH_CHECK();
  } else {
    precond_apply_dev(c, v, z, true);
  }
}


// ---------------------------------------------------------------- CGS / BiCG (krylov.hpp:159-270)
// The reference's recurrences with every scalar on the device: a dot writes kRB partials, one
// thread sums them in index order (the order the host sum used, so the iterates are unchanged) and
// derives α, the relative residual, the stop decision and β. Every kernel of an iteration is a no-op
// once the status leaves RUNNING, so a chunk of iterations is a fixed launch sequence, captured once
// as a CUDA graph and replayed with one status read per replay (as the CG and GMRES drivers).
namespace {

struct SsState {
  int status;
  int it;
  int max_iter;
  int ident;
  double rho, alpha, beta, gnorm, bnorm, tol, rel, one;
};

__device__ __forceinline__ double seq_sum(const double* p, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += p[i];
  return s;
}
// σ = Σ partials; breakdown when σ = 0 or ρ = 0 (krylov.hpp:184-187, 240-243); α = ρ/σ
__global__ void k_ss_alpha(SsState* st, const double* __restrict__ part) {
  if (threadIdx.x != 0 || st->status != ST_RUNNING) return;
  const double sigma = seq_sum(part, kRB);
  if (sigma == 0.0 || st->rho == 0.0) {
    st->status = ST_BREAKDOWN;
    return;
  }
  st->alpha = st->rho / sigma;
}
// out = a + (sgn·coef)·b with coef a device scalar (α or β)
__global__ void k_axpy_dev(double* out, const double* a, const double* b, const double* coef, double sgn, int n,
                           const int* __restrict__ live) {
  if (*live != ST_RUNNING) return;
  const double cb = sgn * *coef;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = 1.0 * a[i] + cb * b[i];
}
// rel = ‖r‖/‖g‖ into the history (the preconditioned residual; with no preconditioner also the true one)
__global__ void k_ss_rel(SsState* st, const double* __restrict__ part, double* hist, double* thist) {
  if (threadIdx.x != 0 || st->status != ST_RUNNING) return;
  const double rel = sqrt(seq_sum(part, kRB)) / st->gnorm;
  st->rel = rel;
  hist[st->it + 1] = rel;
  if (st->ident) thist[st->it + 1] = rel;
}
__global__ void k_ss_thist(const SsState* st, const double* __restrict__ part, double* thist) {
  if (threadIdx.x != 0 || st->status != ST_RUNNING) return;
  thist[st->it + 1] = st->bnorm > 0.0 ? sqrt(seq_sum(part, kRB)) / st->bnorm : 0.0;
}
// one iteration done: converged (rel <= tol) or out of iterations
__global__ void k_ss_finish(SsState* st) {
  if (threadIdx.x != 0 || st->status != ST_RUNNING) return;
  st->it += 1;
  if (st->rel <= st->tol) st->status = ST_CONVERGED;
  else if (st->it >= st->max_iter) st->status = ST_MAXITER;
}
// ρ_new = Σ partials, β = ρ_new/ρ
__global__ void k_ss_beta(SsState* st, const double* __restrict__ part) {
  if (threadIdx.x != 0 || st->status != ST_RUNNING) return;
  const double rn = seq_sum(part, kRB);
  st->beta = rn / st->rho;
  st->rho = rn;
}

struct GraphExec {
  cudaGraphExec_t exec = nullptr;
  size_t nodes = 0;
  ~GraphExec() {
    if (exec) cudaGraphExecDestroy(exec);
  }
};

}  // namespace

// shared driver: init on the host (one-time dots), then captured iterations until the status stops
template <class Iter>
static void ss_solve(Ctx& c, const double* b, double* x, double* r, double tol, int max_iter, int comp,
                     double rho, double gnorm, double bnorm, Iter iteration, DBuf<SsState>& st) {
  const bool ident = c.pkind == RDD_PRECOND_NONE;
  auto& hist = c.hist[comp];
  auto& thist = c.true_hist[comp];
  DBuf<double> dh, dth;
  dh.ensure(static_cast<size_t>(max_iter) + 2);
  dth.ensure(static_cast<size_t>(max_iter) + 2);
  const double h0 = 1.0, t0 = bnorm > 0.0 ? 1.0 : 0.0;
  RDD_CUDA(cudaMemcpyAsync(dh.p, &h0, sizeof(double), cudaMemcpyHostToDevice, c.stream));
  RDD_CUDA(cudaMemcpyAsync(dth.p, &t0, sizeof(double), cudaMemcpyHostToDevice, c.stream));
  SsState s0{};
  s0.status = max_iter > 0 ? ST_RUNNING : ST_MAXITER;
  s0.max_iter = max_iter;
  s0.ident = ident ? 1 : 0;
  s0.rho = rho;
  s0.gnorm = gnorm;
  s0.bnorm = bnorm;
  s0.tol = tol;
  s0.one = 1.0;
  st.upload(&s0, 1, c.stream);
  struct LiveScope {
    Ctx& c;
    LiveScope(Ctx& cc, const int* p) : c(cc) { c.live = p; }
    ~LiveScope() { c.live = nullptr; }
  } ls(c, &st.p->status);
  constexpr int kChunk = 8;
  GraphExec g;
  {
    const bool timing = c.timing;
    c.timing = false;
    const int64_t before = launch_counter();
    cudaGraph_t graph;
    RDD_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    for (int k = 0; k < kChunk; ++k) iteration(dh.p, dth.p);
    RDD_CUDA(cudaStreamEndCapture(c.stream, &graph));
    g.nodes = static_cast<size_t>(launch_counter() - before);
    launch_counter() = before;
    RDD_CUDA(cudaGraphInstantiate(&g.exec, graph, 0));
    cudaGraphDestroy(graph);
    c.timing = timing;
  }
  SsState hs{};
  for (;;) {
    RDD_CUDA(cudaGraphLaunch(g.exec, c.stream));
    launch_counter() += static_cast<int64_t>(g.nodes);
    RDD_CUDA(cudaMemcpyAsync(&hs, st.p, sizeof(SsState), cudaMemcpyDeviceToHost, c.stream));
    RDD_CUDA(cudaStreamSynchronize(c.stream));
    if (hs.status != ST_RUNNING) break;
  }
  c.iters[comp] = hs.it;
  c.conv[comp] = hs.status == ST_CONVERGED;
  c.brk[comp] = hs.status == ST_BREAKDOWN;
  hist.resize(hs.it + 1);
  thist.resize(hs.it + 1);
  dh.download(hist.data(), hs.it + 1, c.stream);
  dth.download(thist.data(), hs.it + 1, c.stream);
  RDD_CUDA(cudaStreamSynchronize(c.stream));
}

// the diagnostic true residual ‖b − A x‖/‖b‖ of every iteration (krylov.hpp:199, 256)
static void ss_true_residual(Ctx& c, const SsState* st, const double* b, const double* x, double* t, double* part,
                             double* thist) {
  if (c.pkind == RDD_PRECOND_NONE) return;  // k_ss_rel wrote it
  normal_operator(c, x, t);
  k_sub<<<kRB, kRT, 0, c.stream>>>(t, b, t, c.p, c.live);
  k_dot_part<<<kRB, kRT, 0, c.stream>>>(t, t, c.p, part, c.live);
  k_ss_thist<<<1, 32, 0, c.stream>>>(st, part, thist);
  RDD_LAUNCH_CHECK();
}

static void ss_dot(Ctx& c, const double* x, const double* y, double* part) {
  k_dot_part<<<kRB, kRT, 0, c.stream>>>(x, y, c.p, part, c.live);
  RDD_LAUNCH_CHECK();
}
static void ss_axpy(Ctx& c, double* out, const double* a, const double* b, const double* coef, double sgn) {
  k_axpy_dev<<<kRB, kRT, 0, c.stream>>>(out, a, b, coef, sgn, c.p, c.live);
  RDD_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- CGS (krylov.hpp:159-213)
static void cgs_solve(Ctx& c, const double* b, double* x, double tol, int max_iter, int comp) {
  const int n = c.p;
  double* part = c.scal.ensure(8 * kRB + 64);
  double* v = c.wk(static_cast<size_t>(n) * 9);
  double *r = v, *rstar = v + n, *p = v + 2 * n, *u = v + 3 * n, *q = v + 4 * n, *uq = v + 5 * n, *Cp = v + 6 * n,
         *t = v + 7 * n, *t2 = v + 8 * n;
  c.hist[comp].clear();
  c.true_hist[comp].clear();
  c.iters[comp] = 0;
  c.conv[comp] = 0;
  c.brk[comp] = 0;
  Vecs V{n, &c};
  const double bnorm = std::sqrt(dot_host(c, b, b, n, part));
  V.fill(x, 0.0);
  precond(c, b, r);  // g = M b
  const double gnorm = std::sqrt(dot_host(c, r, r, n, part));
  if (gnorm == 0.0) {
    c.hist[comp] = {0.0};
    c.true_hist[comp] = {0.0};
    c.conv[comp] = 1;
    return;
  }
  V.copy(rstar, r);
  V.copy(p, r);
  V.copy(u, r);
  const double rho = dot_host(c, rstar, r, n, part);
  DBuf<SsState> st;
  st.ensure(1);
  double* al = &st.p->alpha;
  double* be = &st.p->beta;
  auto Cop = [&](const double* in, double* out) {  // C = M A
    normal_operator(c, in, t2);
    precond(c, t2, out);
  };
  auto iteration = [&](double* dh, double* dth) {
    Cop(p, Cp);
    ss_dot(c, rstar, Cp, part);
    k_ss_alpha<<<1, 32, 0, c.stream>>>(st.p, part);
    RDD_LAUNCH_CHECK();
    ss_axpy(c, q, u, Cp, al, -1.0);    // q = u − α Cp
    ss_axpy(c, uq, u, q, &st.p->one, 1.0);  // uq = u + q
    ss_axpy(c, x, x, uq, al, 1.0);     // x += α uq
    Cop(uq, Cp);
    ss_axpy(c, r, r, Cp, al, -1.0);    // r −= α C uq
    ss_dot(c, r, r, part);
    k_ss_rel<<<1, 32, 0, c.stream>>>(st.p, part, dh, dth);
    RDD_LAUNCH_CHECK();
    ss_true_residual(c, st.p, b, x, t, part, dth);
    k_ss_finish<<<1, 32, 0, c.stream>>>(st.p);
    RDD_LAUNCH_CHECK();
    ss_dot(c, rstar, r, part);
    k_ss_beta<<<1, 32, 0, c.stream>>>(st.p, part);
    RDD_LAUNCH_CHECK();
    ss_axpy(c, u, r, q, be, 1.0);      // u = r + β q
    ss_axpy(c, t, q, p, be, 1.0);      // t = q + β p
    ss_axpy(c, p, u, t, be, 1.0);      // p = u + β t
  };
  ss_solve(c, b, x, r, tol, max_iter, comp, rho, gnorm, bnorm, iteration, st);
}

// ---------------------------------------------------------------- BiCG (krylov.hpp:216-270)
static void bicg_solve(Ctx& c, const double* b, double* x, double tol, int max_iter, int comp) {
  const int n = c.p;
  double* part = c.scal.ensure(8 * kRB + 64);
  double* v = c.wk(static_cast<size_t>(n) * 8);
  double *r = v, *rstar = v + n, *p = v + 2 * n, *ps = v + 3 * n, *Cp = v + 4 * n, *Cps = v + 5 * n, *t = v + 6 * n,
         *t2 = v + 7 * n;
  c.hist[comp].clear();
  c.true_hist[comp].clear();
  c.iters[comp] = 0;
  c.conv[comp] = 0;
  c.brk[comp] = 0;
  Vecs V{n, &c};
  const double bnorm = std::sqrt(dot_host(c, b, b, n, part));
  V.fill(x, 0.0);
  precond(c, b, r);
  const double gnorm = std::sqrt(dot_host(c, r, r, n, part));
  if (gnorm == 0.0) {
    c.hist[comp] = {0.0};
    c.true_hist[comp] = {0.0};
    c.conv[comp] = 1;
    return;
  }
  V.copy(rstar, r);
  V.copy(p, r);
  V.copy(ps, r);
  const double rho = dot_host(c, rstar, r, n, part);
  DBuf<SsState> st;
  st.ensure(1);
  double* al = &st.p->alpha;
  double* be = &st.p->beta;
  auto iteration = [&](double* dh, double* dth) {
    normal_operator(c, p, t2);  // C p = M (A p)
    precond(c, t2, Cp);
    ss_dot(c, ps, Cp, part);
    k_ss_alpha<<<1, 32, 0, c.stream>>>(st.p, part);
    RDD_LAUNCH_CHECK();
    ss_axpy(c, x, x, p, al, 1.0);
    ss_axpy(c, r, r, Cp, al, -1.0);
    precond_t(c, ps, t2);  // Cᵀ p* = Aᵀ (Mᵀ p*), A symmetric
    normal_operator(c, t2, Cps);
    ss_axpy(c, rstar, rstar, Cps, al, -1.0);
    ss_dot(c, r, r, part);
    k_ss_rel<<<1, 32, 0, c.stream>>>(st.p, part, dh, dth);
    RDD_LAUNCH_CHECK();
    ss_true_residual(c, st.p, b, x, t, part, dth);
    k_ss_finish<<<1, 32, 0, c.stream>>>(st.p);
    RDD_LAUNCH_CHECK();
    ss_dot(c, rstar, r, part);
    k_ss_beta<<<1, 32, 0, c.stream>>>(st.p, part);
    RDD_LAUNCH_CHECK();
    ss_axpy(c, p, r, p, be, 1.0);
    ss_axpy(c, ps, rstar, ps, be, 1.0);
  };
  ss_solve(c, b, x, r, tol, max_iter, comp, rho, gnorm, bnorm, iteration, st);
}

void solve_all(Ctx& c, int solver, double tol, int max_iter_cfg, int restart) {
  ScopedKernelTimer tk(c, "solve");
  if (max_iter_cfg < 0) throw std::invalid_argument("max_iter must be >= 1");
  const int max_iter = max_iter_cfg == 0 ? 10 * c.p : max_iter_cfg;
  const int C = c.C, n = c.p;
  c.hist.assign(C, {});
  c.true_hist.assign(C, {});
  c.iters.assign(C, 0);
  c.conv.assign(C, 0);
  c.brk.assign(C, 0);
  c.W.ensure(static_cast<size_t>(n) * C);
  DBuf<double> b, x;
  b.ensure(n);
  x.ensure(n);
  for (int comp = 0; comp < C; ++comp) {
    matvec_t_dev(c, c.F.p + static_cast<size_t>(comp) * c.N, b.p);
    if (solver == RDD_SOLVER_CG) cg_solve(c, b.p, x.p, tol, max_iter, comp);
    else if (solver == RDD_SOLVER_GMRES) gmres_solve(c, b.p, x.p, tol, max_iter, restart, comp);
    else if (solver == RDD_SOLVER_CGS) cgs_solve(c, b.p, x.p, tol, max_iter, comp);
    else if (solver == RDD_SOLVER_BICG) bicg_solve(c, b.p, x.p, tol, max_iter, comp);
    else throw std::invalid_argument("solver not available on the device path");
    k_scale_to<<<kRB, kRT, 0, c.stream>>>(c.W.p + static_cast<size_t>(comp) * n, x.p, c.scales.p, n, 1);
    RDD_LAUNCH_CHECK();
  }
  RDD_CUDA(cudaStreamSynchronize(c.stream));
}

}  // namespace rdd
