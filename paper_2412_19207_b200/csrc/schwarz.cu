// schwarz.cu — K8/K11: one-level overlapping Schwarz preconditioners (schwarz.hpp:39-215).
//
// Build (schwarz.hpp:93-148): S_i = concatenated column ranges of neighbour_sets[i]; A_i is
// gathered blockwise from the normal blocks (missing pairs are exact zeros); the local solve is
// the pseudo-inverse with eigenvalues <= 1e-12·λmax dropped. The device factors A_i = LLᵀ
// (cholesky.cu) and certifies that A_i is far from that cutoff (cond(A_i) < 1e11 from ‖A_i‖_F and
// a power iteration through the factor, refined by a power iteration on A_i when needed); then the
// pseudo-inverse is A_i⁻¹ and each apply is a forward + backward triangular solve. Blocks that
// fail either test take the reference's eigen path (Jacobi, same cutoff) and keep the dense
// pseudo-inverse. Apply (schwarz.hpp:153-185): z_i = A_i⁺ v[S_i]; the AS/SAS/RAS reduction is
// owner-computes: each column sums its (≤3^d) local contributions in ascending i, like the
// reference's serial scatter, without atomics. apply_transpose (schwarz.hpp:189-215) moves the
// SAS/RAS weights in front of the local solve.
#include <algorithm>
#include <cstdio>

#include "ctx.hpp"

namespace rdd {

namespace {

// gather A_i from normal blocks: one CTA per (i, part-pair). Blocks stored transposed (j1 > j2:
// NB holds H_j2ᵀH_j1) go through 32x33 shared-memory tiles so both the read and the write coalesce.
__global__ void k_gather_local(const double* __restrict__ NB, const int* __restrict__ task_i,
                               const int* __restrict__ task_j1, const int* __restrict__ task_j2,
                               const int* __restrict__ task_o1, const int* __restrict__ task_o2,
                               const long long* __restrict__ task_nb, const int* __restrict__ col_off,
                               const int* __restrict__ nvec, const long long* __restrict__ A_off,
                               double* __restrict__ A) {
  __shared__ double tile[32][33];
  const int t = blockIdx.x;
  const int i = task_i[t], j1 = task_j1[t], j2 = task_j2[t], o1 = task_o1[t], o2 = task_o2[t];
  const long long nb = task_nb[t];
  const int n = nvec[i];
  const int p1 = col_off[j1 + 1] - col_off[j1], p2 = col_off[j2 + 1] - col_off[j2];
  double* Ai = A + A_off[i];
  if (j1 <= j2 || nb < 0) {  // stored as (p1 x p2) column-major, or absent (zeros)
    for (int e = threadIdx.x; e < p1 * p2; e += blockDim.x) {
      const int r = e % p1, cc = e / p1;
      Ai[(o1 + r) + static_cast<long long>(o2 + cc) * n] = nb >= 0 ? NB[nb + r + static_cast<long long>(cc) * p1] : 0.0;
    }
    return;
  }
  // element (r, cc) of block (j1, j2) = NB[nb + cc + r·p2] (the (p2 x p1) block of (j2, j1))
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, ny = blockDim.x >> 5;
  for (int r0 = 0; r0 < p1; r0 += 32)
    for (int c0 = 0; c0 < p2; c0 += 32) {
      for (int y = ty; y < 32; y += ny) {  // read: rows r0+y of the target = columns of the source
        const int r = r0 + y, cc = c0 + tx;
        tile[y][tx] = (r < p1 && cc < p2) ? NB[nb + cc + static_cast<long long>(r) * p2] : 0.0;
      }
      __syncthreads();
      for (int y = ty; y < 32; y += ny) {  // write: column c0+y of the target, rows r0..r0+31
        const int cc = c0 + y, r = r0 + tx;
        if (r < p1 && cc < p2) Ai[(o1 + r) + static_cast<long long>(o2 + cc) * n] = tile[tx][y];
      }
      __syncthreads();
    }
}

// per i: keep λ > 1e-12·max(0, λmax) (schwarz.hpp:133-139); X = V diag(1/λ_kept); rank, cond
__global__ void k_local_scale(double* __restrict__ V, const double* __restrict__ lam, const int* __restrict__ nvec,
                              const long long* __restrict__ A_off, const long long* __restrict__ ev_off,
                              double* __restrict__ X, int* __restrict__ rank, double* __restrict__ cond) {
  const int i = blockIdx.x;
  const int n = nvec[i];
  const double* L = lam + ev_off[i];
  __shared__ double s_max, s_min;
  __shared__ int s_rank;
  if (threadIdx.x == 0) {
    double mx = -1e308;
    for (int k = 0; k < n; ++k) mx = fmax(mx, L[k]);
    const double cut = 1e-12 * fmax(0.0, mx);
    double mn = 1e308;
    int rk = 0;
    for (int k = 0; k < n; ++k)
      if (L[k] > cut) {
        ++rk;
        mn = fmin(mn, L[k]);
      }
    s_max = mx;
    s_min = mn;
    s_rank = rk;
    rank[i] = rk;
    cond[i] = rk > 0 ? mx / mn : 0.0;
  }
  __syncthreads();
  const double cut = 1e-12 * fmax(0.0, s_max);
  const double* Vi = V + A_off[i];
  double* Xi = X + A_off[i];
  for (long long e = threadIdx.x; e < static_cast<long long>(n) * n; e += blockDim.x) {
    const int k = static_cast<int>(e / n);
    Xi[e] = L[k] > cut ? Vi[e] / L[k] : 0.0;
  }
}


// out[col] = Σ_i weight · z_i[pos]  over the ≤3^d subdomains whose S_i contains col
// z2 (optional): a second partial of every local result (split local applies), added first
// (optional) v/pzz/pzv: per-CTA partials of out·out and out·v (the CG's ‖z‖², z·r), fixed order
__global__ void __launch_bounds__(256) k_reduce(const double* __restrict__ z, const double* __restrict__ z2,
                                                const int* __restrict__ gat_ptr, const int* __restrict__ gat_pos,
                                                const int* __restrict__ gat_owner_pos, const int* __restrict__ mult,
                                                int p, int kind, int transpose, double* __restrict__ out,
                                                const double* __restrict__ v, double* __restrict__ pzz,
                                                double* __restrict__ pzv, const int* __restrict__ live) {
  if (live && *live != 0) return;
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  double s = 0.0;
  if (col < p) {
    if (!transpose && kind == RDD_PRECOND_RAS) {
      const int q = gat_owner_pos[col];
      s = z2 ? z[q] + z2[q] : z[q];
    } else {
      for (int q = gat_ptr[col]; q < gat_ptr[col + 1]; ++q) {
        const double zz = z2 ? z[gat_pos[q]] + z2[gat_pos[q]] : z[gat_pos[q]];
        s += (!transpose && kind == RDD_PRECOND_SAS) ? zz / mult[col] : zz;
      }
    }
    out[col] = s;
  }
  if (pzz) {
    const double a = block_sum_256(s * s);
    const double b = block_sum_256(col < p ? s * v[col] : 0.0);
    if (threadIdx.x == 0) {
      pzz[blockIdx.x] = a;
      pzv[blockIdx.x] = b;
    }
  }
}




}  // namespace

// bytes the device can still hand out: free memory plus blocks cached (unused) in the pool
size_t device_available(Ctx& c) {
  size_t fr = 0, tot = 0;
  cudaMemGetInfo(&fr, &tot);
  cudaMemPool_t pool;
  uint64_t reserved = 0, used = 0;
  if (cudaDeviceGetDefaultMemPool(&pool, c.device) == cudaSuccess) {
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
  }
  return fr + static_cast<size_t>(reserved > used ? reserved - used : 0);
}

// drop the large PCA scratch (T, rotation logs, Jacobi work) and the unreduced samples S once H
// is assembled; the next build re-creates them
void release_scratch(Ctx& c) {
  for (const char* k : {"pca.T", "syevj.rot", "syevj.Vp", "syevj.Wk", "pca.G", "pca.V0", "pca.W", "pca.Vfull", "pca.L", "pca.Vr", "pca.H"}) {
    auto it = c.wsd.find(k);
    if (it != c.wsd.end()) it->second.release();
  }
  if (!c.identity_V) c.S.release();
}

// Gather A_i for the subdomains in `which` into a compact batch at offsets `off` (zero-filled).
void gather_locals(Ctx& c, const std::vector<int>& which, DBuf<double>& out, const std::vector<long long>& off,
                   bool lower_only) {
  long long tot = 0;
  std::vector<int> slot(c.J, -1), nn(which.size());
  for (size_t q = 0; q < which.size(); ++q) {
    slot[which[q]] = static_cast<int>(q);
    nn[q] = c.local_n[which[q]];
    tot = std::max(tot, off[q] + static_cast<long long>(nn[q]) * nn[q]);
  }
  const double h0 = now_s();
  out.zero(std::max<long long>(1, tot), c.stream);
  if (c.verbose) {
    RDD_CUDA(cudaStreamSynchronize(c.stream));
    std::fprintf(stderr, "[gather] zero %.1f GB %.3f s\n", tot * 8e-9, now_s() - h0);
  }
  std::vector<int> ti, tj1, tj2, to1, to2;
  std::vector<long long> tnb;
  for (const auto& t : c.gat_tasks) {
    if (slot[t.i] < 0) continue;
    if (lower_only && t.o1 < t.o2) continue;  // block entirely above the diagonal
    ti.push_back(slot[t.i]);
    tj1.push_back(t.j1);
    tj2.push_back(t.j2);
    to1.push_back(t.o1);
    to2.push_back(t.o2);
    tnb.push_back(t.nb);
  }
  if (ti.empty()) return;
  DBuf<int> dti, dtj1, dtj2, dto1, dto2, dn;
  DBuf<long long> dtnb, doff;
  dti.upload(ti, c.stream);
  dtj1.upload(tj1, c.stream);
  dtj2.upload(tj2, c.stream);
  dto1.upload(to1, c.stream);
  dto2.upload(to2, c.stream);
  dtnb.upload(tnb, c.stream);
  dn.upload(nn, c.stream);
  doff.upload(off, c.stream);
  k_gather_local<<<static_cast<int>(ti.size()), 256, 0, c.stream>>>(c.NB.p, dti.p, dtj1.p, dtj2.p, dto1.p, dto2.p,
                                                                   dtnb.p, c.dcol_off.p, dn.p, doff.p, out.p);
  RDD_LAUNCH_CHECK();
  if (c.verbose) {
    RDD_CUDA(cudaStreamSynchronize(c.stream));
    std::fprintf(stderr, "[gather] %zu tasks, total %.3f s\n", ti.size(), now_s() - h0);
  }
}

// local_cond as the reference reports it (λmax/λmin of the kept spectrum): power iterations on
// A_i and through its factor, computed on demand (the build only needs the certified bound)
void refresh_local_cond(Ctx& c) {
  if (c.local_cond_exact || c.pkind < 0) return;
  std::vector<int> which;
  for (int i = 0; i < c.J; ++i)
    if (std::find(c.fallback.begin(), c.fallback.end(), i) == c.fallback.end()) which.push_back(i);
  const size_t budget = std::max<size_t>(size_t(1) << 28, device_available(c) / 4);
  for (size_t q0 = 0; q0 < which.size();) {
    std::vector<int> sub, nn;
    std::vector<long long> off, poff;
    long long tot = 0;
    for (; q0 < which.size(); ++q0) {
      const int i = which[q0];
      const long long sz = static_cast<long long>(c.local_n[i]) * c.local_n[i];
      if (!sub.empty() && static_cast<size_t>(tot + sz) * sizeof(double) > budget) break;
      sub.push_back(i);
      off.push_back(tot);
      nn.push_back(c.local_n[i]);
      poff.push_back(c.P_off[i]);
      tot += sz;
    }
    DBuf<double> Af;
    gather_locals(c, sub, Af, off);
    const std::vector<double> la = batched_power(c, Af.p, nn, off, 200);
    const std::vector<double> lp = batched_inv_power(c, c.P.p, sub, nn, poff, 200, c.inv_mode);
    for (size_t q = 0; q < sub.size(); ++q) c.local_cond[sub[q]] = la[q] * lp[q];
  }
  c.local_cond_exact = true;
}

// index sets S_i (schwarz.hpp:39-61), multiplicities and the per-column gather map: host work that
// reads only the decomposition and the PCA ranks, so it can run on a host thread while the normal
// blocks are formed on the device
SchwarzIndex prepare_schwarz_index(const Ctx& c) {
  SchwarzIndex x;
  const int J = c.J;
  x.set_ptr.assign(J + 1, 0);
  x.n.resize(J);
  for (int i = 0; i < J; ++i) {
    int ni = 0;
    for (int q = c.nbr_ptr[i]; q < c.nbr_ptr[i + 1]; ++q) ni += c.h_p[c.nbr_idx[q]];
    if (ni == 0) throw std::runtime_error("empty index set for subdomain " + std::to_string(i));
    x.n[i] = ni;
    x.set_ptr[i + 1] = x.set_ptr[i] + ni;
  }
  x.set_idx.resize(x.set_ptr[J]);
  x.mult.assign(c.p, 0);
  for (int i = 0; i < J; ++i) {
    int* out = x.set_idx.data() + x.set_ptr[i];
    for (int q = c.nbr_ptr[i]; q < c.nbr_ptr[i + 1]; ++q) {
      const int j = c.nbr_idx[q];
      for (int col = c.h_col_off[j]; col < c.h_col_off[j + 1]; ++col) {
        *out++ = col;
        ++x.mult[col];
      }
    }
  }
  // gather map per column: positions (into the concatenated z) in ascending i — a counting sort
  // keyed by column (positions are visited in ascending order, so each column's list is sorted)
  x.gp.assign(c.p + 1, 0);
  x.gpos.resize(x.set_idx.size());
  x.owner_pos.assign(c.p, 0);
  for (int col = 0; col < c.p; ++col) x.gp[col + 1] = x.gp[col] + x.mult[col];
  std::vector<int> fill(x.gp.begin(), x.gp.end() - 1);
  for (int i = 0; i < J; ++i)
    for (int q = x.set_ptr[i]; q < x.set_ptr[i + 1]; ++q) {
      const int col = x.set_idx[q];
      x.gpos[fill[col]++] = q;
      if (c.h_owner[col] == i) x.owner_pos[col] = q;
    }
  return x;
}

void build_schwarz(Ctx& c, int kind, SchwarzIndex* pre) {
  ScopedKernelTimer tk(c, "schwarz_build");
  const int J = c.J;
  c.pkind = kind;
  const double th0 = now_s();
  SchwarzIndex own;
  if (!pre) own = prepare_schwarz_index(c);
  SchwarzIndex& x = pre ? *pre : own;
  c.set_ptr = std::move(x.set_ptr);
  c.set_idx = std::move(x.set_idx);
  c.h_mult = std::move(x.mult);
  std::vector<int> n = std::move(x.n), gp = std::move(x.gp), gpos = std::move(x.gpos),
                   owner_pos = std::move(x.owner_pos);
  c.gat_ptr.upload(gp, c.stream);
  c.gat_pos.upload(gpos, c.stream);
  c.gat_owner_pos.upload(owner_pos, c.stream);
  c.dset_ptr.upload(c.set_ptr, c.stream);
  c.dset_idx.upload(c.set_idx, c.stream);
  c.dmult.upload(c.h_mult, c.stream);
  c.zloc.ensure(std::max<size_t>(1, 2 * c.set_idx.size()));  // two partials in the inverse mode
  if (c.verbose) std::fprintf(stderr, "[schwarz] index sets + gather map (host) %.3f ms\n", 1e3 * (now_s() - th0));

  // local matrix sizes and gather plan (schwarz.hpp:112-130): A_i blocks come from NB. The pair
  // (j1, j2) is looked up in j1's sorted neighbour list (normal blocks exist for neighbour pairs).
  c.local_n = n;
  {
    std::vector<int> ord(J);
    for (int i = 0; i < J; ++i) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return n[a] > n[b]; });
    c.apply_order.upload(ord, c.stream);
  }
  c.gat_tasks.clear();
  c.inv_mode = *std::max_element(n.begin(), n.end()) <= c.inv_max;
  c.env_off.assign(J + 1, 0);
  for (int i = 0; i < J; ++i) c.env_off[i + 1] = c.env_off[i] + ceil_div(n[i], 64);
  c.env_first.assign(c.env_off[J], 0);
  c.env_base.assign(c.env_off[J], 0);
  c.env_entries = 0.0;
  c.P_off.assign(J + 1, 0);
  std::vector<int> po, bfirst;
  for (int i = 0; i < J; ++i) {
    po.clear();
    int o = 0;
    for (int q = c.nbr_ptr[i]; q < c.nbr_ptr[i + 1]; ++q) {
      po.push_back(o);
      o += c.h_p[c.nbr_idx[q]];
    }
    const int b0 = c.nbr_ptr[i], nn = c.nbr_ptr[i + 1] - b0;
    bfirst = po;  // per block row x: first column of its leftmost nonzero block (its own at least)
    for (int x = 0; x < nn; ++x)
      for (int y = 0; y < nn; ++y) {
        const int j1 = c.nbr_idx[b0 + x], j2 = c.nbr_idx[b0 + y];
        const int lo = std::min(j1, j2), hi = std::max(j1, j2);
        const int* beg = c.nbr_idx.data() + c.nbr_ptr[lo];
        const int* endp = c.nbr_idx.data() + c.nbr_ptr[lo + 1];
        const int* it = std::lower_bound(beg, endp, hi);
        if (it == endp || *it != hi) continue;
        const long long nbo = c.h_nb_look[it - c.nbr_idx.data()];
        if (nbo < 0) continue;  // neighbours without a row intersection: no normal block
        c.gat_tasks.push_back({i, j1, j2, po[x], po[y], nbo});
        if (y < x) bfirst[x] = std::min(bfirst[x], po[y]);
      }
    // tile-level envelope of the lower triangle and the packed row bases
    int* ef = c.env_first.data() + c.env_off[i];
    int* eb = c.env_base.data() + c.env_off[i];
    const int nbt = ceil_div(n[i], 64);
    long long tiles = 0;
    for (int k = 0; k < nbt; ++k) ef[k] = c.inv_mode ? 0 : k;
    for (int x = 0; x < nn; ++x) {
      const int r0 = po[x], r1 = (x + 1 < nn ? po[x + 1] : n[i]);  // rows of block x
      if (r1 == r0) continue;
      if (!c.inv_mode)
        for (int k = r0 / 64; k <= (r1 - 1) / 64; ++k) ef[k] = std::min(ef[k], bfirst[x] / 64);
      const double w0 = r0 - bfirst[x] + 1, cnt = r1 - r0;  // row r holds r - bfirst + 1 entries
      c.env_entries += c.inv_mode ? 0.0 : cnt * w0 + cnt * (cnt - 1) / 2.0;
    }
    if (c.inv_mode) c.env_entries += static_cast<double>(n[i]) * (n[i] + 1) / 2.0;
    for (int k = 0; k < nbt; ++k) {
      eb[k] = static_cast<int>(tiles) - ef[k];
      tiles += k - ef[k] + 1;
    }
    c.P_off[i + 1] = c.P_off[i] + (c.inv_mode ? packed_inverse_size(n[i]) : tiles * 64 * 64);
  }
  c.denv_off.upload(c.env_off, c.stream);
  c.denv_first.upload(c.env_first, c.stream);
  c.denv_base.upload(c.env_base, c.stream);
  if (c.verbose) std::fprintf(stderr, "[schwarz] + gather tasks (host) %.3f ms\n", 1e3 * (now_s() - th0));
  // storage: the tile-packed factor of every A_i (the eigen-fallback blocks keep a dense copy) or,
  // when every block is small, the packed explicit inverse: one symmetric tile pass per apply
  // instead of two triangular ones, for 2/3·n³ more build flops
  if (c.verbose) std::fprintf(stderr, "[schwarz] + gather tasks (host) %.3f ms\n", 1e3 * (now_s() - th0));
  c.dP_off.upload(c.P_off, c.stream);
  c.fb_store.clear();
  const size_t p_bytes = static_cast<size_t>(c.P_off[J]) * sizeof(double);
  // cudaMemGetInfo costs up to ~20 ms of host time: only ask when the factor storage must grow
  const bool grow = c.P.n < static_cast<size_t>(std::max<long long>(1, c.P_off[J]));
  {
    ScopedKernelTimer ta(c, "schwarz_alloc");
    if (grow && device_available(c) < p_bytes + (size_t(8) << 30)) release_scratch(c);
    c.P.ensure(std::max<long long>(1, c.P_off[J]));
  }
  // chunk budget for the gathered A_i: fixed at the first build of this context, so reruns reuse the
  // same chunking and the workspace never has to grow (growing a pooled buffer maps new pages: ~2 s
  // for 50 GB)
  if (c.schwarz_budget == 0)
    c.schwarz_budget =
        std::min<size_t>(size_t(40) << 30, std::max<size_t>(size_t(1) << 30, (device_available(c) * 3) / 5));
  if (grow)
    c.schwarz_budget = std::min(c.schwarz_budget, std::max<size_t>(size_t(1) << 30, (device_available(c) * 3) / 5));
  const size_t budget = c.schwarz_budget;
  c.local_rank.assign(J, 0);
  c.local_cond.assign(J, 0.0);
  c.local_cond_exact = false;
  c.fallback.clear();
  std::vector<double*> fbp(J, nullptr);
  for (int i0 = 0; i0 < J;) {
    std::vector<int> chunk, cn;
    std::vector<long long> coff, cpoff;
    long long used = 0;
    int i = i0;
    for (; i < J; ++i) {
      const long long sz = static_cast<long long>(n[i]) * n[i];
      if (!chunk.empty() && static_cast<size_t>(used + sz) * sizeof(double) > budget) break;
      chunk.push_back(i);
      coff.push_back(used);
      cpoff.push_back(c.P_off[i]);
      cn.push_back(n[i]);
      used += sz;
    }
    i0 = i;
    const int B = static_cast<int>(chunk.size());
    DBuf<double>& Aw = c.wsd["schwarz.A"];
    {
      ScopedKernelTimer tg(c, "schwarz_gather");
      gather_locals(c, chunk, Aw, coff, true);  // the factorisation reads the lower triangle
    }
    std::vector<int> fail;
    std::vector<double> fa;
    std::vector<double> fp;
    batched_cholesky_pack(c, Aw.p, chunk, cn, coff, c.P.p, cpoff, fail, fa, c.inv_mode, &fp);
    // rank decision: cond(A_i) <= ‖A_i‖_F·‖A_i⁻¹‖_F (explicit inverse) or ‖A_i‖_F·λmax(A_i⁻¹) (power
    // iteration through the factor); when that does not clear the threshold, λmax(A_i) by power
    // iteration and a longer λmax(A_i⁻¹)
    std::vector<int> ok_q, flagged;
    for (int q = 0; q < B; ++q)
      if (!fail[q]) ok_q.push_back(q);
    if (c.inv_mode) {
      for (int q : ok_q) {
        if (fa[q] * fp[q] < c.full_rank_cond) {
          c.local_rank[chunk[q]] = cn[q];
          c.local_cond[chunk[q]] = fa[q] * fp[q];
        } else {
          flagged.push_back(q);
        }
      }
    } else {
      std::vector<int> nn, okid;
      std::vector<long long> po;
      for (int q : ok_q) {
        nn.push_back(cn[q]);
        po.push_back(cpoff[q]);
        okid.push_back(chunk[q]);
      }
      // routing estimate only: blocks that do not clear the threshold are refined below (60
      // iterations on A_i⁻¹ and A_i), and the exported local_cond is recomputed exactly on demand
      // (refresh_local_cond); ‖A_i‖_F over-estimates λmax(A_i) by up to sqrt(n_i)
      const std::vector<double> lp = batched_inv_power(c, c.P.p, okid, nn, po, 4, false);
      for (size_t z = 0; z < ok_q.size(); ++z) {
        const int q = ok_q[z];
        if (fa[q] * lp[z] < c.full_rank_cond) {
          c.local_rank[chunk[q]] = cn[q];
          c.local_cond[chunk[q]] = fa[q] * lp[z];
        } else {
          flagged.push_back(q);
        }
      }
    }
    std::vector<int> fb;
    for (int q = 0; q < B; ++q)
      if (fail[q]) fb.push_back(q);
    if (!flagged.empty()) {
      std::vector<int> which, fnn;
      std::vector<long long> foff, po;
      long long t = 0;
      for (int q : flagged) {
        which.push_back(chunk[q]);
        fnn.push_back(cn[q]);
        foff.push_back(t);
        po.push_back(cpoff[q]);
        t += static_cast<long long>(cn[q]) * cn[q];
      }
      const std::vector<double> lp = batched_inv_power(c, c.P.p, which, fnn, po, 60, c.inv_mode);
      gather_locals(c, which, Aw, foff);
      const std::vector<double> la = batched_power(c, Aw.p, fnn, foff, 60);
      for (size_t z = 0; z < flagged.size(); ++z) {
        const int q = flagged[z];
        const double cond = la[z] * lp[z];
        if (cond < c.full_rank_cond) {
          c.local_rank[chunk[q]] = cn[q];
          c.local_cond[chunk[q]] = cond;
        } else {
          fb.push_back(q);
        }
      }
    }
    if (!fb.empty()) {  // eigen pseudo-inverse with the reference cutoff, kept dense
      std::sort(fb.begin(), fb.end());
      std::vector<int> which, fnn;
      std::vector<long long> foff, evo;
      long long t = 0, te = 0;
      for (int q : fb) {
        which.push_back(chunk[q]);
        fnn.push_back(cn[q]);
        foff.push_back(t);
        evo.push_back(te);
        t += static_cast<long long>(cn[q]) * cn[q];
        te += cn[q];
      }
      gather_locals(c, which, Aw, foff);
      double* V = c.ws("schwarz.V", t);
      double* X = c.ws("schwarz.X", t);
      double* lam = c.ws("schwarz.lam", te);
      EigOpts eo;  // backward stable like SelfAdjointEigenSolver; cutoff 1e-12·λmax (schwarz.hpp:82)
      eo.absolute = 1;
      eo.tol = 1e-15;
      eo.floor_rel = 1e-16;
      eo.conv_rel = 1e-14;
      eo.max_sweeps = 60;
      batched_syevj(c, Aw.p, V, lam, fnn, foff, eo);
      DBuf<long long> devo, dfoff;
      DBuf<int> drank, dfn;
      DBuf<double> dcond;
      devo.upload(evo, c.stream);
      dfoff.upload(foff, c.stream);
      dfn.upload(fnn, c.stream);
      drank.ensure(fb.size());
      dcond.ensure(fb.size());
      k_local_scale<<<static_cast<int>(fb.size()), 256, 0, c.stream>>>(V, lam, dfn.p, dfoff.p, devo.p, X, drank.p,
                                                                       dcond.p);
      RDD_LAUNCH_CHECK();
      std::vector<GemmTask> tk;
      for (size_t z = 0; z < fb.size(); ++z) {
        double* D = c.fb_store[which[z]].ensure(static_cast<size_t>(fnn[z]) * fnn[z]);
        fbp[which[z]] = D;
        for (int tm = 0; tm < ceil_div(fnn[z], 64); ++tm)
          for (int tn = 0; tn < ceil_div(fnn[z], 64); ++tn)
            tk.push_back({X + foff[z], V + foff[z], D, nullptr, nullptr, fnn[z], fnn[z], fnn[z], fnn[z], fnn[z],
                          fnn[z], tm, tn, 0.0});
      }
      gemm_nt(c, tk);
      std::vector<int> hr(fb.size());
      std::vector<double> hc(fb.size());
      drank.download(hr.data(), fb.size(), c.stream);
      dcond.download(hc.data(), fb.size(), c.stream);
      RDD_CUDA(cudaStreamSynchronize(c.stream));
      for (size_t z = 0; z < fb.size(); ++z) {
        c.local_rank[which[z]] = hr[z];
        c.local_cond[which[z]] = hc[z];
        c.fallback.push_back(which[z]);
      }
    }
  }
  std::sort(c.fallback.begin(), c.fallback.end());
  c.n_fallback = static_cast<int>(c.fallback.size());
  c.dfb_ptr.upload(fbp, c.stream);
  c.nmax_local = *std::max_element(n.begin(), n.end());
  build_ras_panels(c);
}

void precond_apply_dev(Ctx& c, const double* v, double* z, bool transpose, double* pzz, double* pzv) {
  ScopedKernelTimer tk(c, "precond_apply");
  const double* z2 = nullptr;
  if (c.ras_panel) {
    ras_panel_apply(c, v, transpose, c.zloc.p);
  } else {
    chol_apply(c, v, transpose, c.zloc.p);
    if (c.inv_mode) z2 = c.zloc.p + c.set_idx.size();  // second half-partials
  }
  k_reduce<<<ceil_div(c.p, 256), 256, 0, c.stream>>>(c.zloc.p, z2, c.gat_ptr.p, c.gat_pos.p, c.gat_owner_pos.p, c.dmult.p,
                                                     c.p, c.pkind, transpose ? 1 : 0, z, v, pzz, pzv, c.live);
  RDD_LAUNCH_CHECK();
}

}  // namespace rdd
