// hom_api.cu -- the C-ABI of libhom.so (include/hom.h): context setup (a0),
// and the four calls of the hot path (hom_condense, hom_macro_solve,
// hom_recover_fluctuations, hom_macro_kinematics).  Host code here only
// validates, builds index tables once, allocates, and enqueues kernels; every
// step of the method runs on the GPU.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges are no-ops unless a profiler injects itself

#include "hom_internal.cuh"

// NVTX range over one C-ABI call (visible in nsys / ncu --nvtx timelines)
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
};

using hom::CgState;
using hom::MacroDev;
using hom::RveDev;

struct hom_ctx {
  int device = 0;
  hom_options opt{};
  hom_error_info err{};
  int64_t launches = 0;
  int dim = 0, B = 0, m = 0, finite = 0, chunk = 0, macro_free = 0;
  int b_lo = 0, b_hi = 0;  // local RVE range (options.rve_begin / rve_count)
  RveDev R{};
  MacroDev M{};
  std::vector<void*> allocs;
  // chunk-local scratch
  double *Kt = nullptr, *Y = nullptr, *Cavg = nullptr, *Pavg = nullptr, *Aq = nullptr, *Pq = nullptr;
  int fs_slots = 0;                                // persistent CTAs of the fused finite-strain K1
  // whole-batch state
  double *X = nullptr, *rfn = nullptr, *w = nullptr, *kin = nullptr;
  int *info = nullptr, *jflag = nullptr, *first_fail = nullptr;
  // macro
  double *val = nullptr, *diag = nullptr, *rhs = nullptr, *cgwork = nullptr, *Rfree = nullptr, *scal = nullptr;
  double *cgl_sc = nullptr, *cgl_part = nullptr;  // grid-wide PCG scalars / block partials
  double* Cavg_e = nullptr;                       // <C> per element (constant macro basis)
  CgState* cgst = nullptr;
  size_t phase_bytes = 0, mat_bytes = 0;
  int max_slice_nnz = 0;  // largest CSR slice of a 8-CTA cluster partition (CG smem sizing)
  int cg2_slice[2][2] = {};
  hom::TileMask tmask{};     // tile-sparse structure as bitmasks (nt <= 64), k_condense MODE 1
  bool has_tmask = false;
  std::vector<int> nat_of;   // internal RVE node -> natural (API) node (empty: identity)  // k_macro_cg_cluster2 largest (rows, nnz) slice for G = 16, 8
  hom_work work{};
  // event profiling (hom_profile_enable / hom_profile_read)
  struct ProfRec {
    int cls;
    cudaEvent_t a, b;
  };
  bool prof_on = false;
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> pool, all_events;
};

namespace {

cudaEvent_t prof_event(hom_ctx* c) {
  if (!c->pool.empty()) {
    cudaEvent_t e = c->pool.back();
    c->pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  c->all_events.push_back(e);
  return e;
}

constexpr int JFLAG_NONE = 0x7f7f7f7f;  // jflag bytes memset to 0x7f: no failing qp

int set_err(hom_ctx* c, int code, const char* msg, int rve = -1, int row = -1, int cuda = 0) {
  if (c) {
    c->err.code = code;
    c->err.rve = rve;
    c->err.row = row;
    c->err.cuda_error = cuda;
    snprintf(c->err.message, sizeof(c->err.message), "%s", msg);
  }
  return code;
}

int check_cuda(hom_ctx* c, cudaError_t e, const char* where) {
  if (e == cudaSuccess) return HOM_OK;
  char buf[256];
  snprintf(buf, sizeof(buf), "%s: %s", where, cudaGetErrorString(e));
  return set_err(c, e == cudaErrorMemoryAllocation ? HOM_ERR_OOM : HOM_ERR_CUDA, buf, -1, -1, (int)e);
}

template <typename T>
T* dalloc(hom_ctx* c, size_t n, int* rc) {
  if (*rc) return nullptr;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T));
  if (e != cudaSuccess) {
    *rc = check_cuda(c, e, "cudaMalloc");
    return nullptr;
  }
  c->allocs.push_back(p);
  return static_cast<T*>(p);
}

template <typename T>
T* upload(hom_ctx* c, const std::vector<T>& v, cudaStream_t s, int* rc) {
  T* p = dalloc<T>(c, v.size(), rc);
  if (*rc) return nullptr;
  if (!v.empty()) {
    cudaError_t e = cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) *rc = check_cuda(c, e, "cudaMemcpyAsync");
  }
  return p;
}

// Reference element: multilinear Lagrange on [-1,1]^d, local order CCW (2-D) /
// bottom face then top face (3-D); 2-point Gauss per direction, x fastest.
double ref_sign(int dim, int a, int k) {
  int a2 = a & 3;
  if (k == 0) return (a2 == 1 || a2 == 2) ? 1.0 : -1.0;
  if (k == 1) return (a2 >= 2) ? 1.0 : -1.0;
  (void)dim;
  return a >= 4 ? 1.0 : -1.0;
}

// grads [nq][nen][dim], wdet [nq], shp [nq][nen] of one element; returns false if det J <= 0.
bool element_tables(int dim, const double* x /*[nen][dim]*/, double* grad, double* wdet, double* shp) {
  const int nen = 1 << dim, nq = 1 << dim;
  const double gp = 1.0 / std::sqrt(3.0);
  for (int q = 0; q < nq; ++q) {
    double xi[3];
    for (int k = 0; k < dim; ++k) xi[k] = ((q >> k) & 1) ? gp : -gp;
    double dN[8][3], N[8];
    for (int a = 0; a < nen; ++a) {
      double f[3];
      for (int k = 0; k < dim; ++k) f[k] = 0.5 * (1.0 + ref_sign(dim, a, k) * xi[k]);
      N[a] = 1.0;
      for (int k = 0; k < dim; ++k) N[a] *= f[k];
      for (int k = 0; k < dim; ++k) {
        double d = 0.5 * ref_sign(dim, a, k);
        for (int l = 0; l < dim; ++l)
          if (l != k) d *= f[l];
        dN[a][k] = d;
      }
    }
    double J[3][3] = {};
    for (int a = 0; a < nen; ++a)
      for (int i = 0; i < dim; ++i)
        for (int j = 0; j < dim; ++j) J[i][j] += x[a * dim + i] * dN[a][j];
    double det, Ji[3][3];
    if (dim == 1) {
      det = J[0][0];
      Ji[0][0] = 1.0 / det;
    } else if (dim == 2) {
      det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
      Ji[0][0] = J[1][1] / det; Ji[0][1] = -J[0][1] / det;
      Ji[1][0] = -J[1][0] / det; Ji[1][1] = J[0][0] / det;
    } else {
      double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
      double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
      double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
      det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
      Ji[0][0] = c00 / det;
      Ji[1][0] = c01 / det;
      Ji[2][0] = c02 / det;
      Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
      Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
      Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
      Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
      Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
      Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
    }
    if (!(det > 0.0)) return false;
    wdet[q] = det;  // Gauss weights are 1
    for (int a = 0; a < nen; ++a) {
      if (shp) shp[q * nen + a] = N[a];
      for (int i = 0; i < dim; ++i) {
        double s = 0.0;
        for (int j = 0; j < dim; ++j) s += dN[a][j] * Ji[j][i];
        grad[(q * nen + a) * dim + i] = s;
      }
    }
  }
  return true;
}

// Shared-element triples between node pairs of a mesh with element->node map `en`.
struct PairTables {
  std::vector<int> inc_ptr, inc;          // node -> (e<<4 | a)
  std::vector<int> nbr_ptr, nbr, owner;   // node -> sorted neighbours
  std::vector<int> sh_ptr, sh;            // neighbour entry -> (e<<8 | a<<4 | b)
};

PairTables build_pairs(int n_nodes, int ne, int nen, const std::vector<int>& en) {
  PairTables T;
  std::vector<std::vector<int>> inc(n_nodes);
  for (int e = 0; e < ne; ++e)
    for (int a = 0; a < nen; ++a) inc[en[e * nen + a]].push_back((e << 4) | a);
  T.inc_ptr.assign(n_nodes + 1, 0);
  for (int p = 0; p < n_nodes; ++p) {
    T.inc_ptr[p + 1] = T.inc_ptr[p] + (int)inc[p].size();
    T.inc.insert(T.inc.end(), inc[p].begin(), inc[p].end());
  }
  T.nbr_ptr.assign(n_nodes + 1, 0);
  T.sh_ptr.push_back(0);
  for (int p = 0; p < n_nodes; ++p) {
    std::map<int, std::vector<int>> nb;  // sorted by neighbour
    for (int code : inc[p]) {
      int e = code >> 4, a = code & 15;
      for (int b = 0; b < nen; ++b) nb[en[e * nen + b]].push_back((e << 8) | (a << 4) | b);
    }
    for (auto& kv : nb) {
      T.nbr.push_back(kv.first);
      T.owner.push_back(p);
      T.sh.insert(T.sh.end(), kv.second.begin(), kv.second.end());
      T.sh_ptr.push_back((int)T.sh.size());
    }
    T.nbr_ptr[p + 1] = (int)T.nbr.size();
  }
  return T;
}

}  // namespace

extern "C" {

int hom_setup(hom_ctx** out, const hom_macro_mesh* mac, const hom_rve_mesh* rve, const hom_phase_field* ph,
              const hom_materials* mat, const hom_options* options, void* stream) {
  NvtxScope nvtx_("hom_setup");
  if (!out) return HOM_ERR_INVALID_ARG;
  *out = nullptr;
  hom_ctx* c = new hom_ctx();
  cudaStream_t s = (cudaStream_t)stream;
  int rc = HOM_OK;
  auto fail = [&](int code, const char* msg) {
    set_err(c, code, msg);
    return code;
  };
  if (!mac || !rve || !ph || !mat || !options || !mac->coords || !mac->conn || !rve->coords || !rve->conn ||
      !ph->phase || !mat->params) {
    rc = fail(HOM_ERR_INVALID_ARG, "NULL argument");
    *out = c;
    return rc;
  }
  c->opt = *options;
  if (c->opt.cg_rtol <= 0) c->opt.cg_rtol = 1e-13;
  if (c->opt.cg_max_iter <= 0) c->opt.cg_max_iter = 20000;
  if (c->opt.mem_budget_gb <= 0) c->opt.mem_budget_gb = 96.0;
  cudaGetDevice(&c->device);
  const int dim = mac->dim;
  *out = c;
  if ((dim < 1 || dim > 3) || rve->dim != dim || mac->nodes_per_elem != (1 << dim) ||
      rve->nodes_per_elem != (1 << dim) || mac->n_elems <= 0 || rve->n_elems <= 0 || mat->n_phases <= 0 ||
      (mat->kind < 0 || mat->kind > 2) || (mat->kind >= 1 && dim != 2) ||
      (options->finite_strain != 0) != (mat->kind >= 1))
    return fail(HOM_ERR_INVALID_ARG, "unsupported dimension / element / material combination");
  const int nen = 1 << dim, nq = 1 << dim;
  c->dim = dim;
  c->finite = mat->kind >= 1;
  c->m = c->finite ? 4 : (dim == 1 ? 1 : (dim == 2 ? 3 : 6));
  if (options->macro_precond < 0 || options->macro_precond > 2)
    return fail(HOM_ERR_INVALID_ARG, "macro_precond must be 0 (auto), 1 (node-block Jacobi) or 2 (two-level)");
  if (options->macro_basis < 0 || options->macro_basis > 1 || (options->macro_basis == 1 && c->finite))
    return fail(HOM_ERR_INVALID_ARG, "macro_basis must be 0 (Dirac) or 1 (constant, small strain only)");
  c->B = mac->n_elems * (options->macro_basis == 1 ? 1 : nq);

  // ------------------------------------------------------------ macro mesh
  MacroDev& M = c->M;
  M.dim = dim; M.nen = nen; M.nq = nq; M.ne = mac->n_elems; M.n_nodes = mac->n_nodes;
  M.ndof = mac->n_nodes * dim; M.m = c->m; M.finite = c->finite;
  std::vector<int> mconn(mac->conn, mac->conn + (size_t)M.ne * nen);
  for (int v : mconn)
    if (v < 0 || v >= M.n_nodes) return fail(HOM_ERR_MESH, "macro connectivity out of range");
  std::vector<double> mgrad((size_t)M.ne * nq * nen * dim), mw((size_t)M.ne * nq), shp((size_t)nq * nen);
  for (int e = 0; e < M.ne; ++e) {
    double x[8 * 3];
    for (int a = 0; a < nen; ++a)
      for (int k = 0; k < dim; ++k) x[a * dim + k] = mac->coords[(size_t)mconn[e * nen + a] * dim + k];
    if (!element_tables(dim, x, &mgrad[(size_t)e * nq * nen * dim], &mw[(size_t)e * nq], e == 0 ? shp.data() : nullptr))
      return fail(HOM_ERR_MESH, "macro element with det J <= 0");
  }
  // shared-element records pack (e << 8 | a << 4 | b) into an int (build_pairs, k_macro_assemble)
  if (M.ne >= (1 << 23)) return fail(HOM_ERR_INVALID_ARG, "macro mesh too large (>= 2^23 elements)");
  PairTables MP = build_pairs(M.n_nodes, M.ne, nen, mconn);
  // scalar CSR over all DOFs, node-block structure
  std::vector<int> rowptr(M.ndof + 1, 0), col, nzblk;
  std::vector<uint8_t> nzcc;
  for (int n = 0; n < M.n_nodes; ++n)
    for (int ci = 0; ci < dim; ++ci) {
      int row = n * dim + ci;
      for (int k = MP.nbr_ptr[n]; k < MP.nbr_ptr[n + 1]; ++k)
        for (int cj = 0; cj < dim; ++cj) {
          int cl = MP.nbr[k] * dim + cj;
          col.push_back(cl);
          nzblk.push_back(k);
          nzcc.push_back((uint8_t)(ci * 4 + cj + (cl == row ? 16 : 0)));
        }
      rowptr[row + 1] = (int)col.size();
    }
  M.nnz = (int)col.size();
  for (int G : {8, 16})
    for (int g = 0; g < G; ++g) {
      int a = (int)((long)M.ndof * g / G), b = (int)((long)M.ndof * (g + 1) / G);
      c->max_slice_nnz = std::max(c->max_slice_nnz, rowptr[b] - rowptr[a]);
    }
  M.cg_ellw = 0;
  for (int i = 0; i < M.ndof; ++i) M.cg_ellw = std::max(M.cg_ellw, rowptr[i + 1] - rowptr[i]);
  hom::cg2_slice_sizes(M, rowptr.data(), 16, &c->cg2_slice[0][0], &c->cg2_slice[0][1]);
  hom::cg2_slice_sizes(M, rowptr.data(), 8, &c->cg2_slice[1][0], &c->cg2_slice[1][1]);
  {
    std::vector<int> win(2 * 16 * 2, 0);
    hom::cg2_windows(M, rowptr.data(), col.data(), 16, win.data(), &M.cg_wmax[0], &M.cg_wok[0]);
    hom::cg2_windows(M, rowptr.data(), col.data(), 8, win.data() + 32, &M.cg_wmax[1], &M.cg_wok[1]);
    M.cg_win = upload(c, win, s, &rc);
  }
  M.cg_gval = dalloc<double>(c, (size_t)M.ndof * M.cg_ellw, &rc);
  M.cg_gcol = dalloc<int>(c, (size_t)M.ndof * M.cg_ellw, &rc);
  std::vector<uint8_t> dmask(M.ndof, 0);
  std::vector<double> dval(M.ndof, 0.0), fbody(M.ndof, 0.0);
  if (mac->n_dirichlet > 0 && (!mac->dirichlet_dof || !mac->dirichlet_value))
    return fail(HOM_ERR_INVALID_ARG, "Dirichlet arrays missing");
  for (int i = 0; i < mac->n_dirichlet; ++i) {
    int d = mac->dirichlet_dof[i];
    if (d < 0 || d >= M.ndof) return fail(HOM_ERR_INVALID_ARG, "Dirichlet DOF out of range");
    dmask[d] = 1;
    dval[d] = mac->dirichlet_value[i];
  }
  c->macro_free = 0;
  for (int i = 0; i < M.ndof; ++i) c->macro_free += !dmask[i];
  if (mac->body_force) {  // consistent body load f_A = sum eta N^A b (a0 setup, eq:linSys)
    for (int e = 0; e < M.ne; ++e)
      for (int q = 0; q < nq; ++q)
        for (int a = 0; a < nen; ++a)
          for (int k = 0; k < dim; ++k)
            fbody[(size_t)mconn[e * nen + a] * dim + k] += mw[(size_t)e * nq + q] * shp[q * nen + a] * mac->body_force[k];
  }
  if (mac->nodal_force)  // surface tractions as consistent nodal forces (eq:weakMech, Gamma^sigma)
    for (int i = 0; i < M.ndof; ++i) fbody[i] += mac->nodal_force[i];
  M.load_factor = 1.0;

  // ------------------------------------------------------------ RVE mesh, periodic pairing
  RveDev& R = c->R;
  R.dim = dim; R.nen = nen; R.nq = nq; R.ne = rve->n_elems;
  R.m = c->m; R.finite = c->finite; R.ncol = c->m + (c->finite ? 1 : 0);
  const int rn = rve->n_nodes;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int n = 0; n < rn; ++n)
    for (int k = 0; k < dim; ++k) {
      lo[k] = std::min(lo[k], rve->coords[(size_t)n * dim + k]);
      hi[k] = std::max(hi[k], rve->coords[(size_t)n * dim + k]);
    }
  double Lmax = 0.0;
  for (int k = 0; k < dim; ++k) Lmax = std::max(Lmax, hi[k] - lo[k]);
  if (!(Lmax > 0.0)) return fail(HOM_ERR_MESH, "degenerate RVE box");
  const double tol = 1e-9 * Lmax;
  auto key_of = [&](int n, bool fold, int* lower_cnt) {
    std::vector<long long> key(dim);
    int lc = 0;
    for (int k = 0; k < dim; ++k) {
      double x = rve->coords[(size_t)n * dim + k] - lo[k];
      if (fold && std::fabs(x - (hi[k] - lo[k])) < tol) x = 0.0;
      if (std::fabs(x) < tol) { x = 0.0; lc++; }
      key[k] = std::llround(x / (1e-7 * Lmax));
    }
    if (lower_cnt) *lower_cnt = lc;
    return key;
  };
  auto on_upper = [&](int n) {
    for (int k = 0; k < dim; ++k)
      if (std::fabs(rve->coords[(size_t)n * dim + k] - hi[k]) < tol) return true;
    return false;
  };
  std::map<std::vector<long long>, int> indep_of;
  std::vector<int> indep(rn, -1), members, expect;
  for (int n = 0; n < rn; ++n) {
    if (on_upper(n)) continue;
    int lc = 0;
    auto key = key_of(n, false, &lc);
    if (indep_of.count(key)) return fail(HOM_ERR_MESH, "duplicate RVE node");
    int id = (int)indep_of.size();
    indep_of[key] = id;
    indep[n] = id;
    members.push_back(1);
    expect.push_back(1 << lc);
  }
  for (int n = 0; n < rn; ++n) {
    if (!on_upper(n)) continue;
    auto key = key_of(n, true, nullptr);
    auto it = indep_of.find(key);
    if (it == indep_of.end()) return fail(HOM_ERR_MESH, "unmatched periodic RVE node");
    indep[n] = it->second;
    members[it->second]++;
  }
  for (size_t p = 0; p < members.size(); ++p)
    if (members[p] != expect[p]) return fail(HOM_ERR_MESH, "periodic faces do not match");
  R.n_indep = (int)indep_of.size();
  {
    std::vector<long long> zero(dim, 0);
    auto it = indep_of.find(zero);
    if (it == indep_of.end()) return fail(HOM_ERR_MESH, "RVE has no node at its lower corner");
    R.corner = it->second;
  }
  if (options->rve_ordering != 0 && options->rve_ordering != 1)
    return fail(HOM_ERR_INVALID_ARG, "rve_ordering must be 0 (folded) or 1 (natural)");
  if (options->rve_ordering == 0) {  // folded order: interleave the periodic images on every axis
    std::vector<std::vector<long long>> fkey(R.n_indep);
    for (auto& kv : indep_of) {
      std::vector<long long> f;
      for (int k = dim - 1; k >= 0; --k) {  // slowest axis first, like the natural grid order
        const long long L = std::llround((hi[k] - lo[k]) / (1e-7 * Lmax)), x = kv.first[k];
        f.push_back(std::min(x, L - x));
        f.push_back(2 * x > L ? 0 : 1);  // the upper image of a pair first: 0, r-1, 1, r-2, ...
      }
      fkey[kv.second] = f;
    }
    std::vector<int> order(R.n_indep);
    for (int p = 0; p < R.n_indep; ++p) order[p] = p;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return fkey[a] < fkey[b]; });
    std::vector<int> int_of(R.n_indep);
    for (int p = 0; p < R.n_indep; ++p) int_of[order[p]] = p;
    for (int n = 0; n < rn; ++n) indep[n] = int_of[indep[n]];
    R.corner = int_of[R.corner];
    R.nat_of = upload(c, order, s, &rc);  // internal p -> natural order[p]
    R.int_of = upload(c, int_of, s, &rc);
    c->nat_of = order;
  }
  R.npad = dim * R.n_indep;
  R.nt = (R.npad + hom::TILE - 1) / hom::TILE;
  R.NT = R.nt * hom::TILE;
  std::vector<int> rconn(rve->conn, rve->conn + (size_t)R.ne * nen), eind((size_t)R.ne * nen);
  for (size_t i = 0; i < rconn.size(); ++i) {
    if (rconn[i] < 0 || rconn[i] >= rn) return fail(HOM_ERR_MESH, "RVE connectivity out of range");
    eind[i] = indep[rconn[i]];
  }
  if (R.ne >= (1 << 23)) return fail(HOM_ERR_INVALID_ARG, "RVE too large");
  std::vector<double> rgrad((size_t)R.ne * nq * nen * dim), rw((size_t)R.ne * nq);
  double vol = 0.0;
  for (int e = 0; e < R.ne; ++e) {
    double x[8 * 3];
    for (int a = 0; a < nen; ++a)
      for (int k = 0; k < dim; ++k) x[a * dim + k] = rve->coords[(size_t)rconn[e * nen + a] * dim + k];
    if (!element_tables(dim, x, &rgrad[(size_t)e * nq * nen * dim], &rw[(size_t)e * nq], nullptr))
      return fail(HOM_ERR_MESH, "RVE element with det J <= 0");
    for (int q = 0; q < nq; ++q) vol += rw[(size_t)e * nq + q];
  }
  R.vol = vol;
  PairTables RP = build_pairs(R.n_indep, R.ne, nen, eind);
  // geometry-only element matrices of the isotropic closed form (K1 small strain)
  const int ND = nen * dim, m = c->m;
  std::vector<double> Klam, Kmu, Flam, Fmu, evol(R.ne, 0.0);
  if (!c->finite) {
    Klam.assign((size_t)R.ne * ND * ND, 0.0);
    Kmu.assign((size_t)R.ne * ND * ND, 0.0);
    Flam.assign((size_t)R.ne * ND * m, 0.0);
    Fmu.assign((size_t)R.ne * ND * m, 0.0);
  }
  static const int shear2[1][2] = {{0, 1}};
  static const int shear3[3][2] = {{1, 2}, {0, 2}, {0, 1}};
  for (int e = 0; e < R.ne; ++e)
    for (int q = 0; q < nq; ++q) {
      const double w = rw[(size_t)e * nq + q];
      evol[e] += w;
      if (c->finite) continue;
      const double* G = &rgrad[((size_t)e * nq + q) * nen * dim];
      for (int a = 0; a < nen; ++a)
        for (int i = 0; i < dim; ++i) {
          const double* ga = G + a * dim;
          for (int bb = 0; bb < nen; ++bb) {
            const double* gb = G + bb * dim;
            double dot = 0.0;
            for (int t = 0; t < dim; ++t) dot += ga[t] * gb[t];
            for (int j = 0; j < dim; ++j) {
              size_t idx = (size_t)e * ND * ND + (size_t)(a * dim + i) * ND + bb * dim + j;
              Klam[idx] += w * ga[i] * gb[j];
              Kmu[idx] += w * (ga[j] * gb[i] + (i == j ? dot : 0.0));
            }
          }
          for (int k = 0; k < m; ++k) {
            size_t idx = ((size_t)e * ND + a * dim + i) * m + k;
            if (k < dim) {
              Flam[idx] += w * ga[i];
              Fmu[idx] += (i == k) ? w * 2.0 * ga[k] : 0.0;
            } else {
              const int* pr = dim == 2 ? shear2[k - 2] : shear3[k - 3];
              if (i == pr[0]) Fmu[idx] += w * ga[pr[1]];
              if (i == pr[1]) Fmu[idx] += w * ga[pr[0]];
            }
          }
        }
    }
  // structural nonzero pattern of the lower 64x64 tiles (same for every RVE)
  const int nt_ = (dim * R.n_indep + hom::TILE - 1) / hom::TILE;
  std::vector<uint8_t> tile_nz((size_t)nt_ * nt_, 0);
  for (int t = 0; t < nt_; ++t) tile_nz[(size_t)t * nt_ + t] = 1;
  for (int pp = 0; pp < R.n_indep; ++pp) {
    if (pp == R.corner) continue;
    for (int k = RP.nbr_ptr[pp]; k < RP.nbr_ptr[pp + 1]; ++k) {
      int qq = RP.nbr[k];
      if (qq == R.corner) continue;
      for (int ci = 0; ci < dim; ++ci)
        for (int cj = 0; cj < dim; ++cj) {
          int I = (pp * dim + ci) / hom::TILE, J = (qq * dim + cj) / hom::TILE;
          if (I >= J) tile_nz[(size_t)I * nt_ + J] = 1;
        }
    }
  }
  // tiles the factorisation processes: all lower tiles (dense) or the symbolic tile-level
  // fill of tile_nz, G(I,J) != 0 iff A(I,J) != 0 or G(I,K) G(J,K) != 0 for some K < J (tile-sparse)
  std::vector<uint8_t> g_nz((size_t)nt_ * nt_, 0);
  for (int I = 0; I < nt_; ++I)
    for (int J = 0; J <= I; ++J) {
      uint8_t v = c->opt.tile_sparse ? tile_nz[(size_t)I * nt_ + J] : 1;
      for (int K = 0; K < J && !v; ++K) v = g_nz[(size_t)I * nt_ + K] && g_nz[(size_t)J * nt_ + K];
      g_nz[(size_t)I * nt_ + J] = v;
    }
  std::vector<int> tslot((size_t)nt_ * nt_, -1);
  int nslot = 0;
  for (int I = 0; I < nt_; ++I)
    for (int J = 0; J <= I; ++J)
      if (g_nz[(size_t)I * nt_ + J]) tslot[(size_t)I * nt_ + J] = nslot++;
  R.nslot = nslot;
  R.dense_tiles = nslot == nt_ * (nt_ + 1) / 2;
  if (!R.dense_tiles && nt_ <= 64) {
    int slot = 0;
    for (int I = 0; I < nt_; ++I) {
      c->tmask.rowstart[I] = slot;
      for (int J = 0; J <= I; ++J)
        if (g_nz[(size_t)I * nt_ + J]) {
          c->tmask.row[I] |= 1ull << J;
          c->tmask.col[J] |= 1ull << I;
          if (tslot[(size_t)I * nt_ + J] != slot) return fail(HOM_ERR_INVALID_ARG, "tile slot order");
          ++slot;
        }
    }
    c->has_tmask = true;
  }
  {  // work per RVE in 64^3 tile products (hom_get_work)
    auto& W = c->work;
    W = hom_work{};
    for (int J = 0; J < nt_; ++J) {
      for (int K = 0; K < J; ++K) W.syrk_tiles += g_nz[(size_t)J * nt_ + K];
      for (int I = J + 1; I < nt_; ++I) {
        if (!g_nz[(size_t)I * nt_ + J]) continue;
        W.trsm_tiles += 1;
        for (int K = 0; K < J; ++K) W.gemm_tiles += g_nz[(size_t)I * nt_ + K] && g_nz[(size_t)J * nt_ + K];
      }
    }
    for (size_t t = 0; t < tile_nz.size(); ++t) W.a_tiles += tile_nz[t];
    W.g_tiles = nslot;
    W.diag_tiles = nt_;
    const double n = dim * R.n_indep - dim, mm = c->m + (c->finite ? 1 : 0);
    W.flop_dense = n * n * n / 3.0 + 2.0 * n * n * mm + n * mm * mm;
    // executed DMMA flops of k_condense (64^3 units: product 2*64^3; the diagonal SYRK skips
    // the strictly-upper 8x8 blocks, 36/64; TRSM with the triangular G_JJ^-1, 36/64; the
    // right-hand sides are 8 wide; diagonal factor + inverse ~420 m8n8k4 ops per tile)
    const double T3 = 2.0 * 64 * 64 * 64, rhs = 2.0 * 64 * 64 * 8;
    W.flop_executed = W.gemm_tiles * T3 + W.syrk_tiles * (T3 * 36.0 / 64.0 + rhs) +
                      W.trsm_tiles * (T3 * 36.0 / 64.0 + rhs) + nt_ * (420.0 * 512 + 2 * rhs);
  }
  R.phase_per_rve = ph->per_rve ? 1 : 0;
  R.mat_per_rve = mat->per_rve ? 1 : 0;
  R.n_phase = mat->n_phases;
  size_t nph_entries = (size_t)(R.phase_per_rve ? c->B : 1) * R.ne;
  std::vector<uint8_t> phase(ph->phase, ph->phase + nph_entries);
  for (uint8_t v : phase)
    if (v >= mat->n_phases) return fail(HOM_ERR_INVALID_ARG, "phase id >= n_phases");
  R.mat_stride = mat->kind == 2 ? 3 : 2;
  std::vector<double> params(mat->params, mat->params + (size_t)(R.mat_per_rve ? c->B : 1) * R.n_phase * R.mat_stride);

  // ------------------------------------------------------------ chunking + allocation
  const size_t tiles = (size_t)R.nslot;
  const size_t per_rve = tiles * hom::TILE_ELEMS * 8 + (size_t)R.NT * hom::RHSW * 8 + 64 * 8 * 2;
  if (c->opt.rve_count > 0 && (c->opt.rve_begin < 0 || c->opt.rve_begin + c->opt.rve_count > c->B))
    return fail(HOM_ERR_INVALID_ARG, "rve_begin / rve_count outside [0, B)");
  c->b_lo = c->opt.rve_count > 0 ? c->opt.rve_begin : 0;
  c->b_hi = c->opt.rve_count > 0 ? c->opt.rve_begin + c->opt.rve_count : c->B;
  const int nloc = c->b_hi - c->b_lo;
  int chunk = c->opt.rve_chunk > 0 ? c->opt.rve_chunk
                                   : (int)std::min<double>(nloc, std::floor(c->opt.mem_budget_gb * 1e9 / per_rve));
  chunk = std::max(1, std::min(chunk, nloc));
  if (c->opt.rve_chunk <= 0 && chunk < nloc) {
    // automatic chunks that do not hold the whole range: the fewest launches the budget allows, each a
    // whole number of k_condense waves (4 resident CTAs per SM) -- every launch ends with a drain, and
    // only the last chunk may end on a partial wave
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    const int wave = 4 * std::max(1, sms), maxc = chunk;
    if (maxc >= 2 * wave) {
      for (int L = (nloc + maxc - 1) / maxc;; ++L) {
        const int cl = ((nloc + L - 1) / L + wave - 1) / wave * wave;
        if (cl <= maxc) {
          chunk = cl;
          break;
        }
      }
    }
  }
  c->chunk = chunk;

  R.elem_indep = upload(c, eind, s, &rc);
  R.grad = upload(c, rgrad, s, &rc);
  R.wdet = upload(c, rw, s, &rc);
  R.fs_ntype = 0;
  if (c->finite) {  // qp geometry types of the material pass (a uniform grid has one)
    const int gq = nen * dim + 1;
    std::vector<double> tgeo;
    std::vector<int> fet(R.ne, 0);
    int nt_ = 0;
    for (int e = 0; e < R.ne && nt_ <= 16; ++e) {
      double scale = 0.0;
      for (size_t i = 0; i < (size_t)nq * nen * dim; ++i) scale = std::max(scale, std::fabs(rgrad[(size_t)e * nq * nen * dim + i]));
      int found = -1;
      for (int t = 0; t < nt_ && found < 0; ++t) {
        bool same = true;
        for (int q = 0; q < nq && same; ++q) {
          for (int i = 0; i < nen * dim && same; ++i)
            same = std::fabs(rgrad[((size_t)e * nq + q) * nen * dim + i] - tgeo[((size_t)t * nq + q) * gq + i]) <= 1e-13 * scale;
          same = same && std::fabs(rw[(size_t)e * nq + q] - tgeo[((size_t)t * nq + q) * gq + nen * dim]) <=
                             1e-13 * std::fabs(rw[(size_t)e * nq + q]);
        }
        if (same) found = t;
      }
      if (found < 0) {
        found = nt_++;
        for (int q = 0; q < nq; ++q) {
          for (int i = 0; i < nen * dim; ++i) tgeo.push_back(rgrad[((size_t)e * nq + q) * nen * dim + i]);
          tgeo.push_back(rw[(size_t)e * nq + q]);
        }
      }
      fet[e] = found;
    }
    if (nt_ <= 16) {
      R.fs_ntype = nt_;
      R.fs_tgeo = upload(c, tgeo, s, &rc);
      R.fs_etype = upload(c, fet, s, &rc);
    }
  }
  R.inc_ptr = upload(c, RP.inc_ptr, s, &rc);
  R.inc = upload(c, RP.inc, s, &rc);
  R.nbr_ptr = upload(c, RP.nbr_ptr, s, &rc);
  R.nbr = upload(c, RP.nbr, s, &rc);
  R.nbr_owner = upload(c, RP.owner, s, &rc);
  R.sh_ptr = upload(c, RP.sh_ptr, s, &rc);
  R.sh = upload(c, RP.sh, s, &rc);
  {  // element types: (Klam, Kmu) geometry blocks equal to 1e-13 relative share one table (a uniform
     // grid has one; the representative differs from the others only by coordinate rounding)
    std::vector<int> etype(R.ne, 0);
    std::vector<double> KlamT, KmuT, FlamT, FmuT;
    if (!c->finite) {
      const size_t blk = (size_t)ND * ND;
      for (int e = 0; e < R.ne; ++e) {
        double scale = 0.0;
        for (size_t i = 0; i < blk; ++i) scale = std::max(scale, std::fabs(Kmu[e * blk + i]));
        const double tol = 1e-13 * scale;
        int found = -1;
        for (int t = 0; t < (int)(KlamT.size() / blk) && found < 0; ++t) {
          bool same = true;
          for (size_t i = 0; i < blk && same; ++i)
            same = std::fabs(Klam[e * blk + i] - KlamT[t * blk + i]) <= tol &&
                   std::fabs(Kmu[e * blk + i] - KmuT[t * blk + i]) <= tol;
          const size_t fb = (size_t)ND * m;  // K_fe tables must match too (same geometry)
          for (size_t i = 0; i < fb && same; ++i)
            same = std::fabs(Flam[e * fb + i] - FlamT[t * fb + i]) <= tol &&
                   std::fabs(Fmu[e * fb + i] - FmuT[t * fb + i]) <= tol;
          if (same) found = t;
        }
        if (found < 0) {
          found = (int)(KlamT.size() / blk);
          KlamT.insert(KlamT.end(), Klam.begin() + e * blk, Klam.begin() + (e + 1) * blk);
          KmuT.insert(KmuT.end(), Kmu.begin() + e * blk, Kmu.begin() + (e + 1) * blk);
          const size_t fb = (size_t)ND * m;  // the element's K_fe tables (same geometry type)
          FlamT.insert(FlamT.end(), Flam.begin() + e * fb, Flam.begin() + (e + 1) * fb);
          FmuT.insert(FmuT.end(), Fmu.begin() + e * fb, Fmu.begin() + (e + 1) * fb);
        }
        etype[e] = found;
      }
    }
    R.ntype = c->finite ? 0 : (int)(KlamT.size() / ((size_t)ND * ND));
    // per-(type, phase) tables in K1's shared memory when they fit; else the global-table path
    R.gtab = (size_t)R.ntype * mat->n_phases * (nen * nen * ((dim * dim + 1) / 2 * 2) + ND * m) * sizeof(double) > 96 * 1024 ? 1 : 0;
    if (R.gtab && mat->n_phases > 256) return fail(HOM_ERR_INVALID_ARG, "more than 256 phases");
    int max_deg = 1;
    for (int pp = 0; pp < R.n_indep; ++pp) max_deg = std::max(max_deg, RP.nbr_ptr[pp + 1] - RP.nbr_ptr[pp]);

    {  // flattened gather records: one dependent load per (node, neighbour) in K1
      int max_sh = 0;
      for (size_t k = 0; k + 1 < RP.sh_ptr.size(); ++k) max_sh = std::max(max_sh, RP.sh_ptr[k + 1] - RP.sh_ptr[k]);
      R.maxdeg = max_deg;
      R.rs4 = (2 + max_sh + 3) / 4;
      // stencil classes (small strain, shared-memory tables): the sorted list of element-local node
      // pairs (a, b) of a record; when every shared element of a record has the same (type, phase)
      // table t, K_pq = sum_(a,b) K_t[a][b] is one precomputed block of the class (per RVE, K1)
      std::map<std::vector<int>, int> cls_of;
      std::vector<int> cls_ptr{0}, cls_ab;
      bool use_cls = !c->finite && !R.gtab;
      {  // HOM_K1_CLS=0: plain records (A/B)
        const char* e = getenv("HOM_K1_CLS");
        if (e && e[0] == '0') use_cls = false;
      }
      std::vector<int> rec((size_t)R.n_indep * max_deg * R.rs4 * 4, -1);
      for (int pp = 0; pp < R.n_indep; ++pp)
        for (int k = RP.nbr_ptr[pp]; k < RP.nbr_ptr[pp + 1]; ++k) {
          int* r = rec.data() + ((size_t)pp * max_deg + (k - RP.nbr_ptr[pp])) * R.rs4 * 4;
          r[0] = RP.nbr[k] == R.corner ? -1 : RP.nbr[k];
          const int nsh = RP.sh_ptr[k + 1] - RP.sh_ptr[k];
          r[1] = nsh;
          for (int sidx = RP.sh_ptr[k]; sidx < RP.sh_ptr[k + 1]; ++sidx) r[2 + sidx - RP.sh_ptr[k]] = RP.sh[sidx];
          if (use_cls && nsh >= 1) {
            std::vector<int> key;
            for (int sidx = RP.sh_ptr[k]; sidx < RP.sh_ptr[k + 1]; ++sidx) key.push_back(RP.sh[sidx] & 0xff);
            std::sort(key.begin(), key.end());
            auto it = cls_of.find(key);
            if (it == cls_of.end()) {
              if ((int)cls_of.size() == hom::MAX_K1_CLASSES) { use_cls = false; continue; }
              it = cls_of.emplace(key, (int)cls_of.size()).first;
              cls_ab.insert(cls_ab.end(), key.begin(), key.end());
              cls_ptr.push_back((int)cls_ab.size());
            }
            r[1] = nsh | ((it->second + 1) << 16);
          }
        }
      if ((size_t)R.ntype * mat->n_phases * cls_of.size() * ((dim * dim + 1) / 2 * 2) * sizeof(double) > 8192)
        use_cls = false;  // class blocks limited to 8 KB of K1's shared memory
      if (!use_cls) {  // too many classes: plain records
        for (size_t i = 0; i < rec.size(); i += (size_t)R.rs4 * 4)
          if (rec[i + 1] >= 0) rec[i + 1] &= 0xffff;
        cls_ptr.assign(1, 0);
        cls_ab.clear();
      }
      R.ncls = (int)cls_ptr.size() - 1;
      R.cls_ptr = upload(c, cls_ptr, s, &rc);
      R.cls_ab = upload(c, cls_ab.empty() ? std::vector<int>{0} : cls_ab, s, &rc);
      R.nrec = reinterpret_cast<const int4*>(upload(c, rec, s, &rc));
    }
    R.etype = upload(c, etype, s, &rc);
    R.Klam = upload(c, KlamT, s, &rc);
    R.Kmu = upload(c, KmuT, s, &rc);
    R.FlamT = upload(c, FlamT, s, &rc);
    R.FmuT = upload(c, FmuT, s, &rc);
  }
  R.Flam = upload(c, Flam, s, &rc);
  R.Fmu = upload(c, Fmu, s, &rc);
  R.evol = upload(c, evol, s, &rc);
  R.tile_nz = upload(c, tile_nz, s, &rc);
  R.g_nz = upload(c, g_nz, s, &rc);
  {
    std::vector<int> alist;
    for (int I = 0; I < nt_; ++I)
      for (int J = 0; J <= I; ++J)
        if (tile_nz[(size_t)I * nt_ + J]) alist.push_back((I << 16) | J);
    R.n_a = (int)alist.size();
    R.a_list = upload(c, alist, s, &rc);
    // finite strain: keep the RVE's packed K_e (36 doubles per element) in K1's shared memory when it fits
    // beside the row buffers at 2 CTAs/SM (HOM_FS_KS=0 forces the all-L2 variant, for A/B)
    {
      const char* e = getenv("HOM_FS_KS");
      R.fs_ks = c->finite && (size_t)R.ne * 36 * sizeof(double) <= 76 * 1024 && !(e && e[0] == '0');
    }
    R.npw = hom::rve_assemble_npw(R);
    if (R.fs_ks) R.fs_ke_off = (int)((hom::rve_assemble_smem(R, R.npw) - (size_t)R.ne * 36 * sizeof(double)) / 8);
    // K1 warp work items: the row nodes of each nonzero tile packed greedily into items of
    // <= npw consecutive nodes and <= 32 in-tile neighbour records (one per lane), dealt
    // round-robin over the warps
    const int dK = c->finite ? 2 : R.dim;
    // Per item and lane a coverage word (wcov): bit 2n + b = column 2 lane + b of node n's rows is covered by
    // a neighbour block -- the writer stores zeros elsewhere instead of clearing its row buffer first
    if (R.npw > 8) return fail(HOM_ERR_INVALID_ARG, "K1: row-buffer nodes exceed the coverage word");
    std::vector<int> witem, wlist, wcov;
    for (int t = 0; t < R.n_a; ++t) {
      const int r0 = (alist[t] >> 16) * 64, c0 = (alist[t] & 0xffff) * 64;
      const int p_lo = r0 / dK, p_hi = (r0 + 63) / dK;
      int p0 = p_lo, nn = 0;
      std::vector<int> lanes;
      std::vector<unsigned long long> nmask;  // covered columns of each node of the item
      auto flush = [&]() {
        if (nn == 0) return;
        bool pad = false;  // identity rows (corner class, tail) in the item
        for (int n = 0; n < nn; ++n) pad = pad || p0 + n >= R.n_indep || p0 + n == R.corner;
        witem.insert(witem.end(), {alist[t], p0, nn | (pad ? 1 << 8 : 0), tslot[(size_t)(alist[t] >> 16) * nt_ + (alist[t] & 0xffff)]});
        lanes.resize(32, -1);
        wlist.insert(wlist.end(), lanes.begin(), lanes.end());
        for (int L = 0; L < 32; ++L) {
          int w = 0;
          for (int n = 0; n < nn; ++n)
            for (int b = 0; b < 2; ++b)
              if ((nmask[n] >> (2 * L + b)) & 1ull) w |= 1 << (2 * n + b);
          wcov.push_back(w);
        }
        lanes.clear();
        nmask.clear();
        p0 += nn;
        nn = 0;
      };
      for (int pp = p_lo; pp <= p_hi; ++pp) {
        std::vector<int> mine;
        unsigned long long msk = 0;
        if (pp < R.n_indep && pp != R.corner)
          for (int k = RP.nbr_ptr[pp]; k < RP.nbr_ptr[pp + 1]; ++k) {
            const int q = RP.nbr[k], cq = q * dK - c0;
            if (q != R.corner && cq + dK > 0 && cq < 64) {
              mine.push_back(pp * R.maxdeg + (k - RP.nbr_ptr[pp]));
              for (int jj = 0; jj < dK; ++jj)
                if (cq + jj >= 0 && cq + jj < 64) msk |= 1ull << (cq + jj);
            }
          }
        if ((int)mine.size() > 32) return fail(HOM_ERR_INVALID_ARG, "K1: more than 32 neighbour blocks of one node in one tile");
        if (nn == R.npw || lanes.size() + mine.size() > 32) flush();
        for (int ridx : mine) lanes.push_back((nn << 24) | ridx);
        nmask.push_back(msk);
        ++nn;
      }
      flush();
    }
    if ((long)R.n_indep * R.maxdeg >= (1L << 24)) return fail(HOM_ERR_INVALID_ARG, "K1: RVE too large for 24-bit record indices");
    R.n_witem = (int)(witem.size() / 4);
    R.witem = reinterpret_cast<const int4*>(upload(c, witem, s, &rc));
    R.wlist = upload(c, wlist, s, &rc);
    R.wcov = upload(c, wcov, s, &rc);
  }
  R.tslot = upload(c, tslot, s, &rc);
  R.phase = upload(c, phase, s, &rc);
  R.mat = upload(c, params, s, &rc);
  c->phase_bytes = phase.size();
  c->mat_bytes = params.size() * sizeof(double);
  M.conn = upload(c, mconn, s, &rc);
  M.grad = upload(c, mgrad, s, &rc);
  M.shp = upload(c, shp, s, &rc);
  M.wdet = upload(c, mw, s, &rc);
  {  // element volumes |B_e| = sum_q eta j (constant macro basis)
    std::vector<double> ev(M.ne, 0.0);
    for (int e = 0; e < M.ne; ++e)
      for (int q = 0; q < nq; ++q) ev[e] += mw[(size_t)e * nq + q];
    M.evol = upload(c, ev, s, &rc);
  }
  M.constant_basis = c->opt.macro_basis == 1;
  if (M.constant_basis) {
    c->Cavg_e = dalloc<double>(c, (size_t)c->B * c->m * c->m, &rc);
    if (c->Cavg_e) cudaMemsetAsync(c->Cavg_e, 0, sizeof(double) * c->B * c->m * c->m, s);
    M.Cavg_e = c->Cavg_e;
  }
  M.rowptr = upload(c, rowptr, s, &rc);
  M.col = upload(c, col, s, &rc);
  M.nz_blk = upload(c, nzblk, s, &rc);
  M.nz_cc = upload(c, nzcc, s, &rc);
  M.blk_ptr = upload(c, MP.sh_ptr, s, &rc);
  M.blk_sh = upload(c, MP.sh, s, &rc);
  M.ninc_ptr = upload(c, MP.inc_ptr, s, &rc);
  M.ninc = upload(c, MP.inc, s, &rc);
  M.dmask = upload(c, dmask, s, &rc);
  M.dval = upload(c, dval, s, &rc);
  M.fbody = upload(c, fbody, s, &rc);
  M.cg_prof = nullptr;
  if (getenv("HOM_CG_PROF")) {  // experiment knob: phase timing of the cluster PCG (stderr)
    M.cg_prof = dalloc<unsigned long long>(c, 256, &rc);
    if (M.cg_prof) cudaMemsetAsync(M.cg_prof, 0, 256 * 8, s);
  }
  {  // coarse space of the two-level macro preconditioner (coarse.cu)
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    sms = std::max(sms, 1);
    // auto (0): the coarse space only when fewer than a quarter of the macro DOFs are prescribed
    const int one_level = c->opt.macro_precond == 1 ||
                          (c->opt.macro_precond == 0 && 4L * mac->n_dirichlet >= (long)M.n_nodes * dim);
    hom::CoarseHost H = hom::coarse_build(dim, M.n_nodes, mac->coords, rowptr.data(), col.data(), one_level, sms);
    hom::CoarseDev& C = M.cc;
    C = hom::CoarseDev{};
    if (H.nc > 0) {
      C.nc = H.nc; C.nm = H.nm; C.nagg = H.nagg; C.nbmax = H.nbmax;
      C.agg = upload(c, H.agg, s, &rc);
      C.rel = upload(c, H.rel, s, &rc);
      C.aptr = upload(c, H.aptr, s, &rc);
      C.anode = upload(c, H.anode, s, &rc);
      C.nbr = upload(c, H.nbr, s, &rc);
      C.Ac = dalloc<double>(c, (size_t)H.nc * H.nc, &rc);
      C.Ainv = dalloc<double>(c, (size_t)H.nc * H.nc, &rc);
      C.ggrid = H.ggrid;
      for (int gi = 0; gi < 3; ++gi) {
        const auto& L = H.loc[gi];
        const int* d_lptr = upload(c, L.lptr, s, &rc);
        const int* d_lagg = upload(c, L.lagg, s, &rc);
        const int* d_tch = upload(c, L.tch, s, &rc);
        const int* d_lnptr = upload(c, L.lnptr, s, &rc);
        const int* d_lnode = upload(c, L.lnode, s, &rc);
        const int* d_ntch = upload(c, L.ntch, s, &rc);
        if (gi < 2) {
          C.nla_max[gi] = L.nla_max; C.kmax[gi] = L.kmax;
          C.lptr[gi] = d_lptr; C.lagg[gi] = d_lagg; C.tch[gi] = d_tch;
          C.lnptr[gi] = d_lnptr; C.lnode[gi] = d_lnode; C.ntch[gi] = d_ntch;
        } else {
          C.nla_max_g = L.nla_max; C.kmax_g = L.kmax;
          C.lptr_g = d_lptr; C.lagg_g = d_lagg; C.tch_g = d_tch;
          C.lnptr_g = d_lnptr; C.lnode_g = d_lnode; C.ntch_g = d_ntch;
        }
      }
      C.gpart = dalloc<double2>(c, (size_t)std::max(H.ggrid, 1) * std::max(H.loc[2].nla_max, 1) * H.nm, &rc);
    }
  }

  c->Kt = dalloc<double>(c, tiles * hom::TILE_ELEMS * chunk, &rc);
  c->Y = dalloc<double>(c, (size_t)R.NT * hom::RHSW * chunk, &rc);
  c->Cavg = dalloc<double>(c, (size_t)64 * chunk, &rc);
  c->Pavg = dalloc<double>(c, (size_t)8 * chunk, &rc);
  if (c->finite) {
    c->fs_slots = hom::rve_assemble_fs_slots(R);  // persistent CTAs of the fused finite-strain K1
    c->Aq = dalloc<double>(c, (size_t)c->fs_slots * R.ne * hom::FS_RECORD, &rc);  // their element-record scratch
    c->Pq = nullptr;
    c->w = dalloc<double>(c, (size_t)c->B * R.npad, &rc);
  }
  c->X = dalloc<double>(c, (size_t)(c->b_hi - c->b_lo) * R.NT * hom::RHSW, &rc);  // local range only
  c->R.xb0 = c->b_lo;
  c->rfn = dalloc<double>(c, c->B, &rc);
  c->kin = dalloc<double>(c, (size_t)c->B * c->m, &rc);
  c->info = dalloc<int>(c, c->B, &rc);
  c->jflag = dalloc<int>(c, c->B, &rc);
  c->first_fail = dalloc<int>(c, 2, &rc);
  c->val = dalloc<double>(c, M.nnz, &rc);
  c->diag = dalloc<double>(c, M.ndof, &rc);
  c->rhs = dalloc<double>(c, M.ndof, &rc);
  c->Rfree = dalloc<double>(c, M.ndof, &rc);
  c->cgwork = dalloc<double>(c, (size_t)4 * M.ndof, &rc);
  c->scal = dalloc<double>(c, 4, &rc);
  c->cgl_sc = dalloc<double>(c, 16, &rc);
  c->cgl_part = dalloc<double>(c, 2 * 592 * 4, &rc);
  c->cgst = dalloc<CgState>(c, 1, &rc);
  if (rc) return rc;
  if (c->finite) cudaMemsetAsync(c->w, 0, sizeof(double) * (size_t)c->B * R.npad, s);
  cudaMemsetAsync(c->rfn, 0, sizeof(double) * c->B, s);
  rc = check_cuda(c, cudaStreamSynchronize(s), "hom_setup");
  return rc;
}

int hom_get_work(const hom_ctx* c, hom_work* o) {
  if (!c || !o) return HOM_ERR_INVALID_ARG;
  *o = c->work;
  return HOM_OK;
}

int hom_get_sizes(const hom_ctx* c, hom_sizes* o) {
  if (!c || !o) return HOM_ERR_INVALID_ARG;
  o->n_rve = c->B;
  o->m = c->m;
  o->n_pad = c->R.npad;
  o->n_tiles = c->R.nt;
  o->n_macro_dof = c->M.ndof;
  o->n_macro_free = c->macro_free;
  o->macro_nnz = c->M.nnz;
  o->rve_chunk = c->chunk;
  o->rve_volume = c->R.vol;
  o->rve_begin = c->b_lo;
  o->rve_count = c->b_hi - c->b_lo;
  return HOM_OK;
}

// Every kernel launch goes through run(): it counts the launch and, while profiling
// is enabled, brackets it with CUDA events on the launching stream.
extern "C++" template <typename F>
void run(hom_ctx* c, int cls, cudaStream_t s, F&& f) {
  cudaEvent_t a = nullptr, b = nullptr;
  if (c->prof_on) {
    a = prof_event(c);
    cudaEventRecord(a, s);
  }
  f();
  c->launches++;
  if (c->prof_on) {
    b = prof_event(c);
    cudaEventRecord(b, s);
    c->prof.push_back({cls, a, b});
  }
}

int hom_macro_kinematics(hom_ctx* c, const double* d_u, double* d_kin, void* stream) {
  NvtxScope nvtx_("hom_macro_kinematics");
  if (!c || !d_u || !d_kin) return set_err(c, HOM_ERR_INVALID_ARG, "hom_macro_kinematics: NULL");
  run(c, HOM_PROF_RECOVER, (cudaStream_t)stream,
      [&] { hom::launch_macro_kin(c->M, d_u, d_kin, 1, (cudaStream_t)stream); });
  return check_cuda(c, cudaGetLastError(), "hom_macro_kinematics");
}

int hom_condense(hom_ctx* c, const double* d_kin, double* d_C_eff, double* d_P_eff, double* d_P_avg,
                 void* stream) {
  NvtxScope nvtx_("hom_condense");
  if (!c || !d_C_eff) return set_err(c, HOM_ERR_INVALID_ARG, "hom_condense: NULL");
  if (c->finite && !d_kin) return set_err(c, HOM_ERR_INVALID_ARG, "hom_condense: finite strain needs F");
  cudaStream_t s = (cudaStream_t)stream;
  const RveDev& R = c->R;
  cudaMemsetAsync(c->info, 0, sizeof(int) * c->B, s);
  if (c->finite) cudaMemsetAsync(c->jflag, 0x7f, sizeof(int) * c->B, s);  // = JFLAG_NONE
  for (int b0 = c->b_lo; b0 < c->b_hi; b0 += c->chunk) {
    int nb = std::min(c->chunk, c->b_hi - b0);
    if (c->finite)
      run(c, HOM_PROF_RVE_ASSEMBLE, s, [&] {
        hom::launch_rve_assemble_fs(R, b0, nb, d_kin, c->w, c->Kt, c->Y, c->Cavg, c->Pavg, c->rfn, c->Aq,
                                    c->fs_slots, c->jflag, s);
      });
    else
      run(c, HOM_PROF_RVE_ASSEMBLE, s,
          [&] { hom::launch_rve_assemble(R, b0, nb, c->Kt, c->Y, c->Cavg, c->Pavg, c->rfn, s); });
    run(c, HOM_PROF_CONDENSE, s, [&] {
      hom::launch_condense(R, b0, nb, c->Kt, c->Y, c->Cavg, c->Pavg, d_C_eff, d_P_eff, d_P_avg, c->X, c->info, s,
                           c->has_tmask ? &c->tmask : nullptr);
    });
    if (c->Cavg_e)  // keep <C> of every element for the constant-basis macro stiffness
      cudaMemcpy2DAsync(c->Cavg_e + (size_t)b0 * c->m * c->m, sizeof(double) * c->m * c->m, c->Cavg,
                        sizeof(double) * 64, sizeof(double) * c->m * c->m, nb, cudaMemcpyDeviceToDevice, s);
  }
  int rc = check_cuda(c, cudaGetLastError(), "hom_condense");
  if (rc || !c->opt.check_info) return rc;
  int h[2] = {INT_MAX, INT_MAX};
  cudaMemcpyAsync(c->first_fail, h, sizeof(h), cudaMemcpyHostToDevice, s);
  const int nloc = c->b_hi - c->b_lo;
  run(c, HOM_PROF_OTHER, s, [&] { hom::launch_first_fail(c->info + c->b_lo, nloc, 0, c->first_fail, s); });
  if (c->finite)
    run(c, HOM_PROF_OTHER, s,
        [&] { hom::launch_first_fail(c->jflag + c->b_lo, nloc, JFLAG_NONE, c->first_fail + 1, s); });
  cudaMemcpyAsync(h, c->first_fail, sizeof(h), cudaMemcpyDeviceToHost, s);
  rc = check_cuda(c, cudaStreamSynchronize(s), "hom_condense sync");
  if (rc) return rc;
  if (h[0] != INT_MAX) h[0] += c->b_lo;
  if (h[1] != INT_MAX) h[1] += c->b_lo;
  if (h[1] != INT_MAX) {
    int q = -1;
    cudaMemcpy(&q, c->jflag + h[1], sizeof(int), cudaMemcpyDeviceToHost);
    return set_err(c, HOM_ERR_JACOBIAN, "micro Jacobian J <= 0", h[1], q);
  }
  if (h[0] != INT_MAX) {
    int row = -1;
    cudaMemcpy(&row, c->info + h[0], sizeof(int), cudaMemcpyDeviceToHost);
    --row;  // internal K_ff row -> DOF of the natural (API) fluctuation layout
    const int dr = c->R.npad / c->R.n_indep;
    if (!c->nat_of.empty() && row >= 0 && row < c->R.npad) row = c->nat_of[row / dr] * dr + row % dr;
    return set_err(c, HOM_ERR_NOT_SPD, "K_ff not positive definite", h[0], row);
  }
  return HOM_OK;
}

int hom_set_load_factor(hom_ctx* c, double load_factor) {
  if (!c || !(load_factor == load_factor)) return set_err(c, HOM_ERR_INVALID_ARG, "hom_set_load_factor");
  c->M.load_factor = load_factor;
  return HOM_OK;
}

int hom_macro_assemble(hom_ctx* c, const double* d_D, void* stream) {
  if (!c || !d_D) return set_err(c, HOM_ERR_INVALID_ARG, "hom_macro_assemble: NULL");
  cudaStream_t s = (cudaStream_t)stream;
  run(c, HOM_PROF_MACRO_ASSEMBLE, s, [&] { hom::launch_macro_assemble(c->M, d_D, c->val, c->diag, s); });
  return check_cuda(c, cudaGetLastError(), "hom_macro_assemble");
}

int hom_macro_spmv(hom_ctx* c, const double* d_x, double* d_y, void* stream) {
  if (!c || !d_x || !d_y) return set_err(c, HOM_ERR_INVALID_ARG, "hom_macro_spmv: NULL");
  cudaStream_t s = (cudaStream_t)stream;
  run(c, HOM_PROF_CG, s, [&] { hom::launch_spmv(c->M, c->val, d_x, d_y, s); });
  return check_cuda(c, cudaGetLastError(), "hom_macro_spmv");
}

int hom_debug_rve_kff(hom_ctx* c, int rve, double* d_Kff, void* stream) {
  if (!c || !d_Kff) return set_err(c, HOM_ERR_INVALID_ARG, "hom_debug_rve_kff: NULL");
  if (c->finite) return set_err(c, HOM_ERR_INVALID_ARG, "hom_debug_rve_kff: small strain only");
  if (rve < c->b_lo || rve >= c->b_hi) return set_err(c, HOM_ERR_INVALID_ARG, "hom_debug_rve_kff: RVE out of range");
  cudaStream_t s = (cudaStream_t)stream;
  hom::launch_rve_assemble(c->R, rve, 1, c->Kt, c->Y, c->Cavg, c->Pavg, c->rfn, s);
  hom::launch_expand_kff(c->R, c->Kt, d_Kff, s);
  return check_cuda(c, cudaStreamSynchronize(s), "hom_debug_rve_kff");
}

int hom_macro_solve(hom_ctx* c, const double* d_D, const double* d_S, double scale, double* d_x,
                    hom_solve_info* info, void* stream) {
  NvtxScope nvtx_("hom_macro_solve");
  if (!c || !d_D || !d_x) return set_err(c, HOM_ERR_INVALID_ARG, "hom_macro_solve: NULL");
  cudaStream_t s = (cudaStream_t)stream;
  run(c, HOM_PROF_MACRO_ASSEMBLE, s, [&] { hom::launch_macro_assemble(c->M, d_D, c->val, c->diag, s); });
  run(c, HOM_PROF_MACRO_ASSEMBLE, s, [&] { hom::launch_macro_rhs(c->M, c->val, d_S, scale, c->rhs, nullptr, s); });
  // macro PCG: one cluster with the matrix in shared memory when it fits (config sizes),
  // else grid-wide kernels (scaled meshes); the cluster kernel with a global CSR as the last resort
  int extra = 0;  // the two-level preconditioner's setup kernels (coarse.cu)
  const char* fge = getenv("HOM_CG_FORCE_GRID");  // test / experiment knobs: 1 = the persistent grid-wide
  const int force_grid = fge ? atoi(fge) : 0;      // PCG, 2 = the multi-kernel one (k_spmv + k_cgl_*)
  run(c, HOM_PROF_CG, s, [&] {
    if (!force_grid && hom::launch_macro_cg_cluster2(c->M, c->cg2_slice, c->val, c->rhs, scale, c->opt.cg_rtol,
                                                     c->opt.cg_max_iter, d_x, c->cgst, s, &extra))
      return;
    if (c->M.ndof >= 32768 || force_grid) {
      if (force_grid != 2 && hom::launch_macro_cg_grid(c->M, c->val, c->rhs, scale, c->opt.cg_rtol, c->opt.cg_max_iter, d_x, c->cgwork,
                                    c->cgl_part, c->cgst, s, &extra))
        return;
      hom::launch_macro_cg_large(c->M, c->val, c->diag, c->rhs, scale, c->opt.cg_rtol, c->opt.cg_max_iter, d_x,
                                 c->cgwork, c->cgl_sc, c->cgl_part, c->cgst, s);
      return;
    }
    if (!hom::launch_macro_cg_cluster(c->M, c->max_slice_nnz, c->val, c->diag, c->rhs, scale, c->opt.cg_rtol,
                                      c->opt.cg_max_iter, d_x, c->cgwork, c->cgst, s))
      hom::launch_macro_cg(c->M, c->val, c->diag, c->rhs, scale, c->opt.cg_rtol, c->opt.cg_max_iter, d_x,
                           c->cgwork, c->cgst, s);
  });
  c->launches += extra;
  int rc = check_cuda(c, cudaGetLastError(), "hom_macro_solve");
  if (rc) return rc;
  CgState st{};
  cudaMemcpyAsync(&st, c->cgst, sizeof(st), cudaMemcpyDeviceToHost, s);
  rc = check_cuda(c, cudaStreamSynchronize(s), "hom_macro_solve sync");
  if (rc) return rc;
  if (info) {
    info->iterations = st.iterations;
    info->rel_residual = st.rel_residual;
    info->rhs_norm = st.rhs_norm;
  }
  if (c->M.cg_prof) {
    unsigned long long pr[256];
    cudaMemcpy(pr, c->M.cg_prof, sizeof(pr), cudaMemcpyDeviceToHost);
    cudaMemset(c->M.cg_prof, 0, sizeof(pr));
    for (int g = 0; g < 16; ++g) {
      fprintf(stderr, "cgprof cta %2d it %d:", g, st.iterations);
      for (int k = 0; k < 12; ++k) fprintf(stderr, " %7.0f", (double)pr[g * 16 + k] / std::max(st.iterations, 1));
      fprintf(stderr, "\n");
    }
  }
  if (st.status == 5) return set_err(c, HOM_ERR_CG_NOT_CONVERGED, "macro CG did not converge");
  if (st.status == 6) return set_err(c, HOM_ERR_CG_BREAKDOWN, "macro CG breakdown (p^T K p <= 0)");
  return HOM_OK;
}

int hom_macro_residual_norm(hom_ctx* c, const double* d_S, double* norm, void* stream) {
  NvtxScope nvtx_("hom_macro_residual_norm");
  if (!c || !norm) return set_err(c, HOM_ERR_INVALID_ARG, "hom_macro_residual_norm: NULL");
  cudaStream_t s = (cudaStream_t)stream;
  run(c, HOM_PROF_MACRO_ASSEMBLE, s, [&] { hom::launch_macro_rhs(c->M, nullptr, d_S, 0.0, nullptr, c->Rfree, s); });
  run(c, HOM_PROF_OTHER, s, [&] { hom::launch_norm(c->Rfree, c->M.ndof, c->scal, s); });
  cudaMemcpyAsync(norm, c->scal, sizeof(double), cudaMemcpyDeviceToHost, s);
  return check_cuda(c, cudaStreamSynchronize(s), "hom_macro_residual_norm");
}

int hom_recover_fluctuations(hom_ctx* c, const double* d_x, double* d_w, void* stream) {
  NvtxScope nvtx_("hom_recover_fluctuations");
  if (!c || !d_x) return set_err(c, HOM_ERR_INVALID_ARG, "hom_recover_fluctuations: NULL");
  if (!c->finite && !d_w) return set_err(c, HOM_ERR_INVALID_ARG, "hom_recover_fluctuations: d_w NULL");
  cudaStream_t s = (cudaStream_t)stream;
  run(c, HOM_PROF_RECOVER, s, [&] { hom::launch_macro_kin(c->M, d_x, c->kin, 0, s); });
  if (c->finite) {
    run(c, HOM_PROF_RECOVER, s,
        [&] { hom::launch_recover(c->R, c->b_lo, c->b_hi - c->b_lo, c->X, c->kin, c->w, 1, s); });
    if (d_w) run(c, HOM_PROF_RECOVER, s, [&] { hom::launch_permute_w(c->R, c->B, c->w, d_w, 1, s); });
  } else {
    run(c, HOM_PROF_RECOVER, s,
        [&] { hom::launch_recover(c->R, c->b_lo, c->b_hi - c->b_lo, c->X, c->kin, d_w, 0, s); });
  }
  return check_cuda(c, cudaGetLastError(), "hom_recover_fluctuations");
}

int hom_newton_update(hom_ctx* c, double* d_u, const double* d_du, void* stream) {
  NvtxScope nvtx_("hom_newton_update");
  if (!c || !d_u || !d_du || !c->finite) return set_err(c, HOM_ERR_INVALID_ARG, "hom_newton_update");
  cudaStream_t s = (cudaStream_t)stream;
  run(c, HOM_PROF_RECOVER, s, [&] { hom::launch_macro_kin(c->M, d_du, c->kin, 0, s); });
  run(c, HOM_PROF_RECOVER, s,
      [&] { hom::launch_recover(c->R, c->b_lo, c->b_hi - c->b_lo, c->X, c->kin, c->w, 1, s); });
  run(c, HOM_PROF_OTHER, s, [&] { hom::launch_axpy(d_u, d_du, 1.0, c->M.ndof, s); });
  return check_cuda(c, cudaGetLastError(), "hom_newton_update");
}

int hom_set_fluctuations(hom_ctx* c, const double* d_w, void* stream) {
  if (!c || !d_w || !c->finite) return set_err(c, HOM_ERR_INVALID_ARG, "hom_set_fluctuations");
  hom::launch_permute_w(c->R, c->B, d_w, c->w, 0, (cudaStream_t)stream);
  return check_cuda(c, cudaGetLastError(), "hom_set_fluctuations");
}

int hom_get_fluctuations(hom_ctx* c, double* d_w, void* stream) {
  if (!c || !d_w || !c->finite) return set_err(c, HOM_ERR_INVALID_ARG, "hom_get_fluctuations");
  hom::launch_permute_w(c->R, c->B, c->w, d_w, 1, (cudaStream_t)stream);
  return check_cuda(c, cudaGetLastError(), "hom_get_fluctuations");
}

int hom_micro_residual_max(hom_ctx* c, double* out, void* stream) {
  if (!c || !out) return set_err(c, HOM_ERR_INVALID_ARG, "hom_micro_residual_max: NULL");
  cudaStream_t s = (cudaStream_t)stream;
  run(c, HOM_PROF_OTHER, s, [&] { hom::launch_max_reduce(c->rfn + c->b_lo, c->b_hi - c->b_lo, c->scal + 1, s); });
  double v = 0.0;
  cudaMemcpyAsync(&v, c->scal + 1, sizeof(double), cudaMemcpyDeviceToHost, s);
  int rc = check_cuda(c, cudaStreamSynchronize(s), "hom_micro_residual_max");
  *out = v / c->R.vol;  // R_micro of eq:constSolution2 carries 1/|Omega| (R21)
  return rc;
}

int hom_macro_update(hom_ctx* c, double* d_u, const double* d_du, void* stream) {
  if (!c || !d_u || !d_du) return set_err(c, HOM_ERR_INVALID_ARG, "hom_macro_update: NULL");
  cudaStream_t s = (cudaStream_t)stream;
  run(c, HOM_PROF_OTHER, s, [&] { hom::launch_axpy(d_u, d_du, 1.0, c->M.ndof, s); });
  return check_cuda(c, cudaGetLastError(), "hom_macro_update");
}

int hom_set_phases(hom_ctx* c, const uint8_t* h_phase, const double* h_params, void* stream) {
  NvtxScope nvtx_("hom_set_phases");
  if (!c) return HOM_ERR_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (h_phase) {
    // K1 indexes the material tables with the id: validate on the host before the copy
    // (one pass over the bytes; ~2 ms for config 3's 16.8 MB against a ~1.5 s step)
    uint8_t mx = 0;
    for (size_t i = 0; i < c->phase_bytes; ++i) mx = h_phase[i] > mx ? h_phase[i] : mx;
    if (mx >= c->R.n_phase) return set_err(c, HOM_ERR_INVALID_ARG, "hom_set_phases: phase id >= n_phases");
    cudaMemcpyAsync(const_cast<uint8_t*>(c->R.phase), h_phase, c->phase_bytes, cudaMemcpyHostToDevice, s);
  }
  if (h_params)
    cudaMemcpyAsync(const_cast<double*>(c->R.mat), h_params, c->mat_bytes, cudaMemcpyHostToDevice, s);
  return check_cuda(c, cudaGetLastError(), "hom_set_phases");
}

int hom_get_element_cavg(hom_ctx* c, double* d_cavg, void* stream) {
  if (!c || !d_cavg || !c->Cavg_e) return set_err(c, HOM_ERR_INVALID_ARG, "hom_get_element_cavg (constant basis only)");
  const size_t row = sizeof(double) * c->m * c->m;
  cudaMemcpyAsync(d_cavg + (size_t)c->b_lo * c->m * c->m, c->Cavg_e + (size_t)c->b_lo * c->m * c->m,
                  row * (c->b_hi - c->b_lo), cudaMemcpyDeviceToDevice, (cudaStream_t)stream);
  return check_cuda(c, cudaGetLastError(), "hom_get_element_cavg");
}

int hom_set_element_cavg(hom_ctx* c, const double* d_cavg, void* stream) {
  if (!c || !d_cavg || !c->Cavg_e) return set_err(c, HOM_ERR_INVALID_ARG, "hom_set_element_cavg (constant basis only)");
  cudaMemcpyAsync(c->Cavg_e, d_cavg, sizeof(double) * c->B * c->m * c->m, cudaMemcpyDeviceToDevice,
                  (cudaStream_t)stream);
  return check_cuda(c, cudaGetLastError(), "hom_set_element_cavg");
}

int hom_profile_enable(hom_ctx* c, int enable) {
  if (!c) return HOM_ERR_INVALID_ARG;
  c->prof_on = enable != 0;
  return HOM_OK;
}

int hom_profile_read(hom_ctx* c, double* ms, int64_t* launches) {
  if (!c || !ms) return HOM_ERR_INVALID_ARG;
  for (int i = 0; i < HOM_PROF_N; ++i) {
    ms[i] = 0.0;
    if (launches) launches[i] = 0;
  }
  if (!c->prof.empty()) {
    int rc = check_cuda(c, cudaEventSynchronize(c->prof.back().b), "hom_profile_read");
    if (rc) return rc;
  }
  for (auto& r : c->prof) {
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    ms[r.cls] += t;
    if (launches) launches[r.cls]++;
    c->pool.push_back(r.a);
    c->pool.push_back(r.b);
  }
  c->prof.clear();
  return HOM_OK;
}

int64_t hom_launch_count(const hom_ctx* c) { return c ? c->launches : 0; }

int hom_last_error(const hom_ctx* c, hom_error_info* out) {
  if (!c || !out) return HOM_ERR_INVALID_ARG;
  *out = c->err;
  return HOM_OK;
}

void hom_destroy(hom_ctx* c) {
  if (!c) return;
  for (void* p : c->allocs) cudaFree(p);
  for (cudaEvent_t e : c->all_events) cudaEventDestroy(e);
  delete c;
}

}  // extern "C"
