// coarse.cu -- coarse space of the two-level macro preconditioner (K6).
//
// The macro system K_M u = -R of eq:linSys is solved by PCG (the macro
// problem is global, every RVE enters it only through its condensed tangent).  The
// one-level node-block Jacobi preconditioner needs O(nel) iterations (246 at config 2, 846
// at config 3); the additive two-level form
//     z = B^-1 r + P A_c^-1 P^T r,   A_c = P^T K_M P
// adds a coarse space of aggregates (the macro nodes binned into na^dim boxes), each with
// its rigid-body modes (dim translations + dim(dim-1)/2 infinitesimal rotations about the
// aggregate centroid).  This file builds the aggregates on the host (once per mesh),
// assembles A_c on the device in a fixed summation order (bitwise reproducible) and
// inverts it with the symmetric sweep operator (Gauss-Jordan on an SPD matrix, one pivot
// per step; modes whose pivot vanishes -- aggregates without free DOFs, or dependent
// modes -- are dropped).  k_macro_cg_cluster2 applies the correction (macro.cu).
// Nothing here changes the solution of K_M u = -R, only the iteration count.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "hom_internal.cuh"

namespace hom {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

CoarseHost coarse_build(int dim, int n_nodes, const double* coords, const int* rowptr, const int* col,
                        int one_level, int ggrid) {
  CoarseHost H;
  H.nc = 0;
  const int ndof = n_nodes * dim;
  const char* e = getenv("HOM_CG_COARSE");  // experiment knob: 0 = one-level block Jacobi only
  if (one_level || (e && atoi(e) == 0) || dim < 2 || ndof < CC_MIN_DOF) return H;
  const char* ena = getenv("HOM_CG_COARSE_NA");  // experiment knob: aggregates per axis
  const int nm = dim == 2 ? 3 : 6, na = ena ? atoi(ena) : (dim == 2 ? CC_NA2 : CC_NA3);
  if (na < 1) return H;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int n = 0; n < n_nodes; ++n)
    for (int k = 0; k < dim; ++k) {
      lo[k] = std::min(lo[k], coords[(size_t)n * dim + k]);
      hi[k] = std::max(hi[k], coords[(size_t)n * dim + k]);
    }
  // bin the nodes into na^dim boxes of the bounding box, drop empty boxes
  std::vector<int> box(n_nodes), id(1, 0);
  int nbox = 1;
  for (int k = 0; k < dim; ++k) nbox *= na;
  id.assign(nbox, -1);
  for (int n = 0; n < n_nodes; ++n) {
    int b = 0;
    for (int k = dim - 1; k >= 0; --k) {
      const double ext = hi[k] - lo[k];
      int ik = ext > 0 ? (int)std::floor((coords[(size_t)n * dim + k] - lo[k]) / ext * na) : 0;
      ik = std::min(std::max(ik, 0), na - 1);
      b = b * na + ik;
    }
    box[n] = b;
  }
  int nagg = 0;
  for (int n = 0; n < n_nodes; ++n)
    if (id[box[n]] < 0) id[box[n]] = 1;
  for (int b = 0; b < nbox; ++b)
    if (id[b] > 0) id[b] = nagg++;
  H.agg.resize(n_nodes);
  for (int n = 0; n < n_nodes; ++n) H.agg[n] = id[box[n]];
  if (nagg * nm > CC_NC_MAX) return H;
  // centroids and the scaled relative coordinates (scale: the largest box edge)
  std::vector<double> cen((size_t)nagg * dim, 0.0);
  std::vector<int> cnt(nagg, 0);
  for (int n = 0; n < n_nodes; ++n) {
    cnt[H.agg[n]]++;
    for (int k = 0; k < dim; ++k) cen[(size_t)H.agg[n] * dim + k] += coords[(size_t)n * dim + k];
  }
  for (int a = 0; a < nagg; ++a)
    for (int k = 0; k < dim; ++k) cen[(size_t)a * dim + k] /= cnt[a];
  double h = 0.0;
  for (int k = 0; k < dim; ++k) h = std::max(h, (hi[k] - lo[k]) / na);
  if (!(h > 0.0)) return H;
  H.rel.resize((size_t)n_nodes * dim);
  for (int n = 0; n < n_nodes; ++n)
    for (int k = 0; k < dim; ++k)
      H.rel[(size_t)n * dim + k] = (coords[(size_t)n * dim + k] - cen[(size_t)H.agg[n] * dim + k]) / h;
  // nodes of each aggregate (increasing node index)
  H.aptr.assign(nagg + 1, 0);
  for (int n = 0; n < n_nodes; ++n) H.aptr[H.agg[n] + 1]++;
  for (int a = 0; a < nagg; ++a) H.aptr[a + 1] += H.aptr[a];
  H.anode.resize(n_nodes);
  {
    std::vector<int> fill(H.aptr.begin(), H.aptr.end() - 1);
    for (int n = 0; n < n_nodes; ++n) H.anode[fill[H.agg[n]]++] = n;
  }
  // neighbour aggregates through the CSR pattern (sorted; -1 padded to nbmax)
  std::vector<std::vector<int>> nb(nagg);
  for (int n = 0; n < n_nodes; ++n)
    for (int k = rowptr[(size_t)n * dim]; k < rowptr[(size_t)n * dim + 1]; ++k) nb[H.agg[n]].push_back(H.agg[col[k] / dim]);
  H.nbmax = 0;
  for (auto& v : nb) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    H.nbmax = std::max(H.nbmax, (int)v.size());
  }
  if (H.nbmax > CC_NB_MAX) return H;
  for (int i = 0; i < ndof; ++i)
    if (rowptr[i + 1] - rowptr[i] > CC_ROWMAX) return H;
  H.nbr.assign((size_t)nagg * H.nbmax, -1);
  for (int a = 0; a < nagg; ++a)
    for (size_t q = 0; q < nb[a].size(); ++q) H.nbr[(size_t)a * H.nbmax + q] = nb[a][q];
  // per cluster size: the aggregates each CTA's node range touches, its position among the
  // CTAs touching each aggregate, and its node list per local aggregate
  H.ggrid = ggrid;
  for (int gi = 0; gi < 3; ++gi) {
    const int G = gi == 0 ? 16 : (gi == 1 ? 8 : ggrid);
    auto& L = H.loc[gi];
    L.ntch.assign(nagg, 0);
    L.lptr.assign(G + 1, 0);
    L.lagg.clear(); L.lnptr.assign(1, 0); L.lnode.clear();
    std::vector<std::vector<int>> who(nagg);
    L.nla_max = 0;
    std::vector<std::vector<int>> bucket(nagg);  // this CTA's nodes of each aggregate (one pass)
    for (int g = 0; g < G; ++g) {
      const int nd0 = (int)((long)n_nodes * g / G), nd1 = (int)((long)n_nodes * (g + 1) / G);
      std::vector<int> la;
      for (int n = nd0; n < nd1; ++n) {
        if (bucket[H.agg[n]].empty()) la.push_back(H.agg[n]);
        bucket[H.agg[n]].push_back(n - nd0);
      }
      std::sort(la.begin(), la.end());
      for (int a : la) {
        who[a].push_back(g << 16 | (int)(L.lagg.size() - L.lptr[g]));
        L.lagg.push_back(a);
        L.ntch[a]++;
        L.lnode.insert(L.lnode.end(), bucket[a].begin(), bucket[a].end());  // increasing node order
        L.lnptr.push_back((int)L.lnode.size());
        bucket[a].clear();
      }
      L.lptr[g + 1] = (int)L.lagg.size();
      L.nla_max = std::max(L.nla_max, (int)la.size());
    }
    L.kmax = *std::max_element(L.ntch.begin(), L.ntch.end());
    L.tch.assign((size_t)nagg * L.kmax, 0);
    for (int a = 0; a < nagg; ++a)
      for (size_t k = 0; k < who[a].size(); ++k) L.tch[(size_t)a * L.kmax + k] = who[a][k];
  }
  H.nm = nm;
  H.nagg = nagg;
  H.nc = nagg * nm;
  return H;
}

// ---------------------------------------------------------------- A_c = P^T K_M P
// One CTA per aggregate a (row block a*nm .. a*nm+nm-1 of A_c).  Warp w takes the nodes
// w, w+NW, ... of the aggregate, one DOF row at a time: the lanes first stage the row's
// entries (value, neighbour slot of the column's aggregate, the column's P coefficients) in
// the warp's shared-memory buffer, all loads in flight together; then lane l < nm*nm owns the
// mode pair (m1, m2) and adds P[i,m1] K_ij P[j,m2] of every entry, in CSR order, into its
// column of the warp-private [nbmax][nm*nm] table.  The NW warp tables are summed in warp
// order (fixed summation order: bitwise reproducible).  Dirichlet rows and columns do not
// enter (their rows of P are zero).
template <int DIM>
__host__ __device__ constexpr int cca_warps() { return DIM == 2 ? 16 : 8; }
template <int DIM>
__global__ void __launch_bounds__(cca_warps<DIM>() * 32) k_coarse_assemble(MacroDev M, const double* __restrict__ val) {
  constexpr int NM = DIM == 2 ? 3 : 6, NP = NM * NM, NW = cca_warps<DIM>(), THR = NW * 32;
  const CoarseDev& C = M.cc;
  const int a = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nbm = C.nbmax, nc = C.nc;
  extern __shared__ double cca_sm[];
  double* acc = cca_sm;                                  // [NW][nbm][NP]
  double* stg = acc + (size_t)NW * nbm * NP;             // [NW][CC_ROWMAX][NM + 1]: K_ij, P[j, 0..NM-1]
  int* stq = reinterpret_cast<int*>(stg + (size_t)NW * CC_ROWMAX * (NM + 1));  // [NW][CC_ROWMAX]
  __shared__ int snb[CC_NB_MAX];
  for (int q = threadIdx.x; q < nbm; q += THR) snb[q] = C.nbr[(size_t)a * nbm + q];
  for (int t = threadIdx.x; t < NW * nbm * NP; t += THR) acc[t] = 0.0;
  for (int t = threadIdx.x; t < NM * nc; t += THR)  // zero the row block (non-neighbour columns)
    C.Ac[(size_t)(a * NM + t / nc) * nc + t % nc] = 0.0;
  __syncthreads();
  double* wacc = acc + (size_t)warp * nbm * NP;
  double* wst = stg + (size_t)warp * CC_ROWMAX * (NM + 1);
  int* wq = stq + warp * CC_ROWMAX;
  for (int k = C.aptr[a] + warp; k < C.aptr[a + 1]; k += NW) {
    const int n = C.anode[k];
    double di[DIM];
#pragma unroll
    for (int d = 0; d < DIM; ++d) di[d] = C.rel[(size_t)n * DIM + d];
#pragma unroll 1
    for (int ci = 0; ci < DIM; ++ci) {
      const int row = n * DIM + ci;
      if (M.dmask[row]) continue;
      const int e0 = M.rowptr[row], len = M.rowptr[row + 1] - e0;
      for (int t = lane; t < len; t += 32) {  // stage the row (independent loads per lane)
        const int j = M.col[e0 + t];
        const double v = val[e0 + t];
        const int nj = j / DIM, cj = j - nj * DIM, b = C.agg[nj];
        double dj[DIM];
#pragma unroll
        for (int d = 0; d < DIM; ++d) dj[d] = C.rel[(size_t)nj * DIM + d];
        const bool fr = !M.dmask[j];
        int q = 0;
        while (snb[q] != b) ++q;
        wq[t] = q;
        wst[t * (NM + 1)] = fr ? v : 0.0;
#pragma unroll
        for (int m = 0; m < NM; ++m) wst[t * (NM + 1) + 1 + m] = cc_coef(DIM, cj, m, dj);
      }
      __syncwarp();
      for (int p = lane; p < NP; p += 32) {
        const int m1 = p / NM, m2 = p % NM;
        const double pi = cc_coef(DIM, ci, m1, di);
        if (pi != 0.0)
          for (int t = 0; t < len; ++t) {
            const double pj = wst[t * (NM + 1) + 1 + m2];
            if (pj != 0.0) wacc[wq[t] * NP + p] += pi * wst[t * (NM + 1)] * pj;
          }
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nbm * NP; t += THR) {
    const int q = t / NP, p = t - q * NP, b = snb[q];
    if (b < 0) continue;
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += acc[(size_t)w * nbm * NP + t];
    C.Ac[(size_t)(a * NM + p / NM) * nc + b * NM + p % NM] = s;
  }
}

// ---------------------------------------------------------------- A_c^-1 (block sweep, DMMA)
// One CTA; the lower triangle of A_c (padded to NB = ceil(nc/8) block rows) as 8x8 blocks in
// shared memory.  Step K sweeps the 8 pivots of diagonal block K (the sweep operator: after
// all pivots the table holds -A_c^-1):
//   P1 (one warp) scalar sweep of the 8x8 block D_K -> D'; a pivot <= 1e-10 of its original
//      diagonal is not swept (an aggregate without free DOFs, or a mode dependent on the
//      others: that mode is dropped, its row and column are zero in the result).
//      Dinv = -D' on the swept set S, zero elsewhere; M = Dinv on the columns S, e_u - [D'_Su]
//      on the unswept columns u.
//   P2 W_I = a_IK Dinv, X_I = a_IK (saved), a_IK <- a_IK M for every block row I != K
//   P3 a_IJ -= W_I X_J^T for every block I >= J, I, J != K
// Look-ahead: warp 0 updates block (K+1, K+1) first in P3 and runs P1 of step K+1 while the
// other warps finish P3, so each step costs P2 + P3 and two CTA barriers.  Every 8x8x8
// product is two m8n8k4 DMMAs; blocks are stored with column ^ 4 on rows 2, 3, 6, 7 (fragment
// loads conflict-free).
constexpr int CCI_THR = 1024;
__device__ __forceinline__ int cci_e(int r, int c) { return r * 8 + (c ^ ((r & 2) << 1)); }
__device__ __forceinline__ double cci_rcp(double d) {  // 1/d to ~1 ulp: approximation + 2 Newton steps
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  y = fma(y, fma(-d, y, 1.0), y);
  return fma(y, fma(-d, y, 1.0), y);
}
__global__ void __launch_bounds__(CCI_THR) k_coarse_invert(CoarseDev C) {
  const int nc = C.nc, NB = (nc + 7) / 8, NBL = NB * (NB + 1) / 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = CCI_THR / 32;
  const int gr = lane >> 2, gc = lane & 3;  // DMMA fragment coordinates
  extern __shared__ double cci_sm[];
  double* T = cci_sm;                  // [NBL][64]
  double* W = T + (size_t)NBL * 64;    // [NB][64]
  double* X = W + (size_t)NB * 64;     // [NB][64]
  double* Dv = X + (size_t)NB * 64;    // [64] (plain row-major)
  double* Mm = Dv + 64;                // [64]
  double* d0 = Mm + 64;                // [NB * 8]
  int* sw = reinterpret_cast<int*>(d0 + NB * 8);  // [NB * 8]
  short2* bij = reinterpret_cast<short2*>(sw + NB * 8);  // [NBL]
  auto blk = [&](int I, int J) { return T + (size_t)(I * (I + 1) / 2 + J) * 64; };
  for (int t = threadIdx.x; t < NBL * 64; t += CCI_THR) {  // all loads independent
    const int p = t >> 6, e = t & 63;
    int I = (int)((sqrtf(8.0f * p + 1.0f) - 1.0f) * 0.5f);
    while (I * (I + 1) / 2 > p) --I;
    while ((I + 1) * (I + 2) / 2 <= p) ++I;
    const int J = p - I * (I + 1) / 2, r = e >> 3, c = e & 7, gi = I * 8 + r, gj = J * 8 + c;
    const double v = (gi < nc && gj < nc) ? C.Ac[(size_t)gi * nc + gj] : 0.0;
    T[(size_t)p * 64 + cci_e(r, c)] = v;
    if (e == 0) bij[p] = make_short2((short)I, (short)J);
    if (I == J && r == c) d0[gi] = v;
  }
  __syncthreads();
  auto p1 = [&](int K) {  // one warp
    double* D = blk(K, K);
    const int r0 = lane >> 3, c = lane & 7;
    const int rr[2] = {r0, r0 + 4};
    double v[2] = {D[cci_e(rr[0], c)], D[cci_e(rr[1], c)]};
#pragma unroll 1
    for (int k = 0; k < 8; ++k) {
      const int ekk = 9 * k;
      const double dkk = __shfl_sync(0xffffffffu, ekk < 32 ? v[0] : v[1], ekk & 31);
      const double crk0 = __shfl_sync(0xffffffffu, v[0], (rr[0] * 8 + k) & 31);
      const double crk1 = __shfl_sync(0xffffffffu, v[1], (rr[1] * 8 + k) & 31);
      const double t0 = __shfl_sync(0xffffffffu, v[0], (c * 8 + k) & 31);
      const double t1 = __shfl_sync(0xffffffffu, v[1], (c * 8 + k) & 31);
      const double cck = c < 4 ? t0 : t1;
      const bool piv = dkk > 1e-10 * d0[K * 8 + k];
      if (piv) {
        const double id = cci_rcp(dkk);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (rr[h] == k || c == k) v[h] = (rr[h] == k && c == k) ? -id : v[h] * id;
          else v[h] -= (h == 0 ? crk0 : crk1) * cck * id;
        }
      }
      if (lane == 0) sw[K * 8 + k] = piv;
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      D[cci_e(rr[h], c)] = v[h];
      const int e = rr[h] * 8 + c;
      const bool sr = sw[K * 8 + rr[h]], sc = sw[K * 8 + c];
      const double di = (sr && sc) ? -v[h] : 0.0;
      Dv[e] = di;
      Mm[e] = sc ? di : ((rr[h] == c ? 1.0 : 0.0) - (sr ? v[h] : 0.0));
    }
  };
  // a_IJ -= W_I X_J^T on block p = (I, J)
  auto p3 = [&](int p, int I, int J) {
    double* B = T + (size_t)p * 64;
    double2* cp = reinterpret_cast<double2*>(B + cci_e(gr, 2 * gc));
    double2 cv = *cp;
#pragma unroll
    for (int k0 = 0; k0 < 8; k0 += 4)
      dmma(cv.x, cv.y, -W[I * 64 + cci_e(gr, k0 + gc)], X[J * 64 + cci_e(gr, k0 + gc)]);
    *cp = cv;
  };
  if (warp == 0) p1(0);
  __syncthreads();
  for (int K = 0; K < NB; ++K) {
    for (int I = warp; I < NB; I += nw) {  // P2
      if (I == K) continue;
      const bool below = I > K;
      double* B = below ? blk(I, K) : blk(K, I);  // a_IK, or its transpose
      for (int e = lane; e < 64; e += 32) {
        const int r = e >> 3, cc = e & 7;
        X[I * 64 + cci_e(r, cc)] = below ? B[cci_e(r, cc)] : B[cci_e(cc, r)];
      }
      double w0 = 0.0, w1 = 0.0, z0 = 0.0, z1 = 0.0;
#pragma unroll
      for (int k0 = 0; k0 < 8; k0 += 4) {
        const int k = k0 + gc;
        const double av = below ? B[cci_e(gr, k)] : B[cci_e(k, gr)];
        dmma(w0, w1, av, Dv[k * 8 + gr]);
        dmma(z0, z1, av, Mm[k * 8 + gr]);
      }
      *reinterpret_cast<double2*>(W + I * 64 + cci_e(gr, 2 * gc)) = make_double2(w0, w1);
      __syncwarp();  // X saved before the block is overwritten
      if (below) {
        *reinterpret_cast<double2*>(B + cci_e(gr, 2 * gc)) = make_double2(z0, z1);
      } else {
        B[cci_e(2 * gc, gr)] = z0;
        B[cci_e(2 * gc + 1, gr)] = z1;
      }
    }
    __syncthreads();
    const int K1 = K + 1, pla = K1 < NB ? K1 * (K1 + 1) / 2 + K1 : -1;
    if (warp == 0) {  // look-ahead: block (K+1, K+1), then P1 of the next step
      if (pla >= 0) {
        p3(pla, K1, K1);
        __syncwarp();
        p1(K1);
      }
    } else {
      // P3: warp w - 1 takes a contiguous range of blocks (mostly one block row: its W_I
      // fragments stay in registers), two blocks in flight
      const int per = (NBL + nw - 2) / (nw - 1), pb = (warp - 1) * per, pe = min(NBL, pb + per);
      int wI = -1;
      double wa[2] = {0.0, 0.0};
      for (int p = pb; p < pe; p += 2) {
        const int q = p + 1;
        const short2 ij = bij[p], ij2 = bij[q < pe ? q : p];
        const bool a1 = !(ij.x == K || ij.y == K || p == pla);
        const bool a2 = q < pe && !(ij2.x == K || ij2.y == K || q == pla);
        double2* cp1 = reinterpret_cast<double2*>(T + (size_t)p * 64 + cci_e(gr, 2 * gc));
        double2* cp2 = reinterpret_cast<double2*>(T + (size_t)(a2 ? q : p) * 64 + cci_e(gr, 2 * gc));
        double2 c1 = *cp1, c2 = *cp2;
        if (ij.x != wI) {
          wI = ij.x;
#pragma unroll
          for (int h = 0; h < 2; ++h) wa[h] = -W[wI * 64 + cci_e(gr, 4 * h + gc)];
        }
        double wb[2], xa[2], xb[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          xa[h] = X[ij.y * 64 + cci_e(gr, 4 * h + gc)];
          wb[h] = ij2.x == wI ? wa[h] : -W[ij2.x * 64 + cci_e(gr, 4 * h + gc)];
          xb[h] = X[ij2.y * 64 + cci_e(gr, 4 * h + gc)];
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          dmma(c1.x, c1.y, wa[h], xa[h]);
          dmma(c2.x, c2.y, wb[h], xb[h]);
        }
        if (a1) *cp1 = c1;
        if (a2) *cp2 = c2;
      }
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < nc * nc; t += CCI_THR) {  // full symmetric matrix, coalesced rows
    const int i = t / nc, j = t - i * nc, hi = max(i, j), lo = min(i, j);
    C.Ainv[t] = (sw[i] && sw[j]) ? -blk(hi >> 3, lo >> 3)[cci_e(hi & 7, lo & 7)] : 0.0;
  }
}

bool launch_coarse_setup(const MacroDev& M, const double* val, cudaStream_t s) {
  const CoarseDev& C = M.cc;
  if (C.nc <= 0) return false;
  const int nm = M.dim == 2 ? 3 : 6;
  auto sa = [&](int nw) {
    return (size_t)nw * C.nbmax * nm * nm * 8 + (size_t)nw * CC_ROWMAX * ((nm + 1) * 8 + 4);
  };
  if (M.dim == 2) {
    const size_t b = sa(cca_warps<2>());
    cudaFuncSetAttribute(k_coarse_assemble<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b);
    k_coarse_assemble<2><<<C.nagg, cca_warps<2>() * 32, b, s>>>(M, val);
  } else {
    const size_t b = sa(cca_warps<3>());
    cudaFuncSetAttribute(k_coarse_assemble<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b);
    k_coarse_assemble<3><<<C.nagg, cca_warps<3>() * 32, b, s>>>(M, val);
  }
  const int NB = (C.nc + 7) / 8, NBL = NB * (NB + 1) / 2;
  const size_t si = ((size_t)NBL * 64 + 2 * (size_t)NB * 64 + 128 + NB * 8) * 8 + (size_t)NB * 8 * 4 + (size_t)NBL * 4;
  cudaFuncSetAttribute(k_coarse_invert, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)si);
  k_coarse_invert<<<1, CCI_THR, si, s>>>(C);
  return cudaGetLastError() == cudaSuccess;
}

}  // namespace hom
