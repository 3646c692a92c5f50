// rve_assembly.cu -- K1: batched RVE assembly of K_ff, K_fe (, r_f), <C> (, <P>).
//
// PAPER.md eq:discreteSys_D and eq:discreteSys_L: for RVE b the
// micro-micro block is K_ff = sum_e sum_qp eta~ B_f^T C B_f and the coupling is
// K_fe = sum eta~ B_f^T C (un-normalised, R2); the periodic
// constraint (eq:Con (iii); nodal coupling P:604-612) is applied on the
// fly through the element -> independent-node map, and the corner class is an
// identity pad.  Output is K_ff in 64x64 tiles: the structurally nonzero lower
// tiles (I,J) (RveDev::tile_nz), each row-major at its pool slot RveDev::tslot;
// structurally zero tiles are never written (k_condense starts their
// accumulators at zero).  K_fe (and r_f) go to the right-hand-side block Y [NT][8].
//
// One CTA per RVE; each warp gathers one node row-block of a tile at a time
// and streams it out with coalesced 16-byte stores -- the kernel is HBM-write
// bound (K1).
#include <algorithm>

#include "hom_internal.cuh"

namespace hom {

// sigma(e_k)[c][J] for the unit Voigt strain k of an isotropic material.
template <int DIM>
__device__ __forceinline__ double unit_stress(int k, int c, int J, double lam, double mu) {
  constexpr int NN = DIM;  // normal components first
  double s = 0.0;
  if (k < NN) {
    if (c == J) s += lam;
    if (c == k && J == k) s += 2.0 * mu;
  } else {
    int i, j;
    if (DIM == 2) { i = 0; j = 1; }
    else if (k == 3) { i = 1; j = 2; }
    else if (k == 4) { i = 0; j = 2; }
    else { i = 0; j = 1; }
    if ((c == i && J == j) || (c == j && J == i)) s += mu;  // 2 mu * (1/2)
  }
  return s;
}

// ---------------------------------------------------------------------------
// K1a (finite strain): per (RVE, element, qp) deformation gradient, stress and
// tangent of the paper's Cook energy, plane strain of the polyconvex
// Mooney-Rivlin form eq:MR:
//   Psi = alpha (F:F - 2) + beta (F:F + J^2 - 3) + kappa/2 (J - 1)^2 - 2 (alpha + 2 beta) ln J,
//   P = 2 (alpha + beta) F + g(J) H,  g = 2 beta J + kappa (J - 1) - 2 (alpha + 2 beta) / J,
//   A = 2 (alpha + beta) I + g'(J) H (x) H + g dH/dF,  g' = 2 beta + kappa + 2 (alpha + 2 beta) / J^2,
// with H = cof F (the 2-D specialisation of 1/2 F xx F).  kind 1 = beta 0 (R11).
// F~ = F + grad w (eq:microGrad).
// ---------------------------------------------------------------------------
// Element record per (RVE, element), 76 doubles (EL_STRIDE): K_e = sum_q eta G_q^T A_q G_q packed
// lower-triangular ([8][8] symmetric, 36 entries, EL_K), F_e [8][4] = sum_q eta G_q^T A_q (EL_F) and
// r_e [8] = sum_q eta G_q^T P_q (EL_R) -- the element parts of K_ff, K_fF and r_f (eq:discreteSys_D/L).
// The volume sums of A and P for <A>, <P> are reduced on chip, not stored.
constexpr int EL_STRIDE = FS_RECORD, EL_K = 0, EL_F = 36, EL_R = 68;
__device__ __forceinline__ int pk8(int r, int c) { return r >= c ? ((r * (r + 1)) >> 1) + c : ((c * (c + 1)) >> 1) + r; }

__device__ __forceinline__ bool cook_material(const double* F, double alpha, double beta, double kappa, double* P,
                                              double* A) {
  // J - 1 from the displacement-gradient part (no cancellation near F = I)
  const double g11 = F[0] - 1.0, g22 = F[3] - 1.0;
  const double Jm1 = g11 + g22 + g11 * g22 - F[1] * F[2];
  const double J = 1.0 + Jm1;
  if (!(J > 0.0)) return false;
  const double H[4] = {F[3], -F[2], -F[1], F[0]};  // cof F (2-D specialisation of 1/2 F xx F)
  const double ab = alpha + 2.0 * beta, iJ = 1.0 / J, abJ = 2.0 * ab * iJ;  // one division per material point
  const double dPsidJ = 2.0 * beta * J + kappa * Jm1 - abJ;
  const double d2 = 2.0 * beta + kappa + abJ * iJ;
  // P = 2 (alpha + beta) F + g H written as 2 (alpha + beta)(F - H) + (g + 2 (alpha + beta)) H with
  // g + 2 (alpha + beta) = (J - 1)(2 beta + kappa + 2 (alpha + 2 beta) / J): both terms vanish at F = I
  // (the stress-free reference) instead of cancelling
  const double c0 = 2.0 * (alpha + beta), c1 = Jm1 * (2.0 * beta + kappa + abJ);
  const double FmH[4] = {F[0] - F[3], F[1] + F[2], F[2] + F[1], F[3] - F[0]};
  for (int i = 0; i < 4; ++i) P[i] = c0 * FmH[i] + c1 * H[i];
  // dH/dF is the constant anti-diagonal [0 0 0 1; 0 0 -1 0; 0 -1 0 0; 1 0 0 0]
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      double v = d2 * H[i] * H[j];
      if (i == j) v += 2.0 * (alpha + beta);
      if (i + j == 3) v += ((i == 0 || i == 3) ? 1.0 : -1.0) * dPsidJ;
      A[i * 4 + j] = v;
    }
  return true;
}

// Element records of elements [e0, e0 + cnt) (cnt <= FS_ELB) of RVE b by the CTA's NTHR threads:
// phase 1, one thread per (element, qp) evaluates F~, P, A once (shared memory); phase 2, one
// thread per element row (a, i) forms its rows of K_e, F_e, r_e and the qp sums of A and P;
// the records are staged in shared memory and written as one contiguous, coalesced range to
// `out` (the CTA's L2-resident scratch, read back by the tile writer of the same CTA).
constexpr int FS_ELB = 32, FS_QW = 29;
constexpr int FS_SMEM_DBL = FS_ELB * 4 * FS_QW;
// L2 residency hints: the element records are re-read by the same CTA moments later (evict_last),
// the K_ff tiles stream out once (evict_first) so they do not push the records out of L2
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_hint(double* a, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void nh_elements(const RveDev& R, int b, int e0, int cnt, const double* __restrict__ Fbar,
                                            const double* __restrict__ w, double* __restrict__ out,
                                            int* __restrict__ jflag, double* sm, int* sOk, double (&avg)[4],
                                            double* ske) {  // ske: K_e of elements e0.. in shared memory, or null
  double (*sQ)[FS_QW] = reinterpret_cast<double (*)[FS_QW]>(sm);  // [FS_ELB * 4][FS_QW]
  const int ne = R.ne, nq = R.nq, tid = threadIdx.x;
  if (tid < FS_ELB) sOk[tid] = 1;
  __syncthreads();
  // ---- phase 1: material point per (element, qp) ----
  if (tid < FS_ELB * 4) {
    const int le = tid >> 2, q = tid & 3;
    if (le < cnt && q < nq) {
      const int e = e0 + le;
      const double* Fb = Fbar + (long)b * 4;
      const double* wb = w + (long)b * R.npad;
      const int ph = R.phase[(R.phase_per_rve ? (long)b * ne : 0) + e];
      const int np = R.mat_stride;
      const double* mp = R.mat + (R.mat_per_rve ? (long)b * R.n_phase * np : 0) + np * ph;
      const double alpha = mp[0], beta = np == 3 ? mp[1] : 0.0, kappa = mp[np - 1];
      const double* G = R.grad + (long)(e * nq + q) * 4 * 2;  // [nen][2]
      double F[4] = {Fb[0], Fb[1], Fb[2], Fb[3]};
      for (int aa = 0; aa < 4; ++aa) {  // F~ = F + grad w (eq:microGrad)
        const int p = R.elem_indep[e * 4 + aa];
        const double w0 = wb[2 * p], w1 = wb[2 * p + 1];
        F[0] += w0 * G[2 * aa]; F[1] += w0 * G[2 * aa + 1];
        F[2] += w1 * G[2 * aa]; F[3] += w1 * G[2 * aa + 1];
      }
      double* Q = sQ[tid];
#pragma unroll
      for (int k = 0; k < 8; ++k) Q[20 + k] = G[k];
      Q[28] = R.wdet[e * nq + q];
      if (!cook_material(F, alpha, beta, kappa, Q + 16, Q)) {
        atomicMin(&jflag[b], e * nq + q);  // first failing qp of this RVE (init INT_MAX)
        sOk[le] = 0;
      }
    }
  }
  __syncthreads();
  // ---- phase 2: element rows (a, i), written straight to the L2-resident scratch ----
  {
    const int le = tid >> 3, row = tid & 7, a = row >> 1, i = row & 1;
    double* o = out + (long)le * EL_STRIDE;
    const uint64_t pol = l2_policy_evict_last();
    if (le < cnt) {
      const bool ok = sOk[le];
      double ke[8] = {}, fe[4] = {}, re = 0.0;
      for (int q = 0; q < nq; ++q) {
        const double* A = sQ[le * 4 + q];
        const double* P = A + 16;
        const double* G = A + 20;
        const double wq = A[28];
        const double ga0 = G[2 * a], ga1 = G[2 * a + 1];
        double t[4];  // row (a, i): t[k] = sum_J g_a[J] A[(i,J), k]
        for (int k = 0; k < 4; ++k) t[k] = ga0 * A[(2 * i) * 4 + k] + ga1 * A[(2 * i + 1) * 4 + k];
        for (int k = 0; k < 4; ++k) fe[k] += wq * t[k];
        re += wq * (ga0 * P[2 * i] + ga1 * P[2 * i + 1]);
        for (int bb = 0; bb < 4; ++bb)
          for (int j = 0; j < 2; ++j)  // column (b, j): sum_L t[(j,L)] g_b[L]
            ke[2 * bb + j] += wq * (t[2 * j] * G[2 * bb] + t[2 * j + 1] * G[2 * bb + 1]);
      }
      if (ske) {
        for (int k = 0; k <= row; ++k) ske[le * 36 + pk8(row, k)] = ok ? ke[k] : 0.0;  // lower part
      } else {
        for (int k = 0; k <= row; ++k) st_hint(o + EL_K + pk8(row, k), ok ? ke[k] : 0.0, pol);
      }
      for (int k = 0; k < 4; ++k) st_hint(o + EL_F + row * 4 + k, ok ? fe[k] : 0.0, pol);
      st_hint(o + EL_R + row, ok ? re : 0.0, pol);
      if (row < 5 && ok) {  // running qp sums of A (rows 0-3: 4 entries each) and P (row 4) for <A>, <P>
        for (int q = 0; q < nq; ++q) {
          const double wq = sQ[le * 4 + q][28];
          for (int k = 0; k < 4; ++k) avg[k] += wq * sQ[le * 4 + q][row * 4 + k];
        }
      }
    }
  }
  __syncthreads();  // sQ reused by the next block
}

// Staged variant (K_e in shared memory and few element geometry types, R.fs_ntype > 0): the RVE's w,
// phases, connectivity and the per-type qp geometry are copied into shared memory once per RVE
// (fs_stage), so the material points read no global memory except the material constants; the
// symmetric tangent A is staged as its 10 distinct entries.  Same arithmetic order as nh_elements.
constexpr int FS_QW2 = 14, FS_ELB2 = 64;  // per qp: A (10, upper triangle packed), P (4); elements per pass
__device__ __forceinline__ int sym4(int i, int j) {
  const int lo = i < j ? i : j, hi = i < j ? j : i;
  return lo * 4 - (lo * (lo - 1)) / 2 + (hi - lo);
}
struct FsStage {
  double* w;        // [npad]
  double* geo;      // [fs_ntype][nq][9]
  int* ei;          // [ne][4]
  int* et;          // [ne]
  uint8_t* ph;      // [ne]
};
__device__ __forceinline__ FsStage fs_stage_layout(const RveDev& R, double* sm) {
  FsStage S;
  S.w = sm + FS_ELB2 * 4 * FS_QW2;
  S.geo = S.w + R.npad;
  S.ei = reinterpret_cast<int*>(S.geo + R.fs_ntype * R.nq * 9);
  S.et = S.ei + R.ne * 4;
  S.ph = reinterpret_cast<uint8_t*>(S.et + R.ne);
  return S;
}
__device__ __forceinline__ void fs_stage(const RveDev& R, int b, const double* __restrict__ w, const FsStage& S) {
  const int tid = threadIdx.x;
  const double* wb = w + (long)b * R.npad;
  for (int i = tid; i < R.npad; i += NTHR) S.w[i] = wb[i];
  for (int i = tid; i < R.fs_ntype * R.nq * 9; i += NTHR) S.geo[i] = R.fs_tgeo[i];
  for (int i = tid; i < R.ne * 4; i += NTHR) S.ei[i] = R.elem_indep[i];
  for (int i = tid; i < R.ne; i += NTHR) {
    S.et[i] = R.fs_etype[i];
    S.ph[i] = R.phase[(R.phase_per_rve ? (long)b * R.ne : 0) + i];
  }
  __syncthreads();
}
__device__ __forceinline__ void nh_elements_st(const RveDev& R, int b, int e0, int cnt, const double* __restrict__ Fbar,
                                               int* __restrict__ jflag, double* sm, int* sOk, double (&avg)[4],
                                               double* ske, const FsStage& S, double* __restrict__ out) {
  double (*sQ)[FS_QW2] = reinterpret_cast<double (*)[FS_QW2]>(sm);  // [FS_ELB2 * 4][FS_QW2]
  const int nq = R.nq, tid = threadIdx.x;
  if (tid < FS_ELB2) sOk[tid] = 1;
  __syncthreads();
  if (tid < FS_ELB2 * 4) {  // ---- phase 1: material point per (element, qp) ----
    const int le = tid >> 2, q = tid & 3;
    if (le < cnt && q < nq) {
      const int e = e0 + le;
      const double* Fb = Fbar + (long)b * 4;
      const int np = R.mat_stride;
      const double* mp = R.mat + (R.mat_per_rve ? (long)b * R.n_phase * np : 0) + np * S.ph[e];
      const double alpha = mp[0], beta = np == 3 ? mp[1] : 0.0, kappa = mp[np - 1];
      const double* G = S.geo + (S.et[e] * nq + q) * 9;
      double F[4] = {Fb[0], Fb[1], Fb[2], Fb[3]};
      for (int aa = 0; aa < 4; ++aa) {  // F~ = F + grad w (eq:microGrad)
        const int p = S.ei[e * 4 + aa];
        const double w0 = S.w[2 * p], w1 = S.w[2 * p + 1];
        F[0] += w0 * G[2 * aa]; F[1] += w0 * G[2 * aa + 1];
        F[2] += w1 * G[2 * aa]; F[3] += w1 * G[2 * aa + 1];
      }
      double A[16];
      double* Q = sQ[tid];
      if (!cook_material(F, alpha, beta, kappa, Q + 10, A)) {
        atomicMin(&jflag[b], e * nq + q);  // first failing qp of this RVE (init INT_MAX)
        sOk[le] = 0;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = i; j < 4; ++j) Q[sym4(i, j)] = A[i * 4 + j];
    }
  }
  __syncthreads();
  const uint64_t pol = l2_policy_evict_last();
  for (int le = tid >> 3; le < cnt; le += NTHR / 8) {  // ---- phase 2: element rows (a, i) ----
    const int row = tid & 7, a = row >> 1, i = row & 1;
    double* o = out + (long)le * EL_STRIDE;
    {
      const int e = e0 + le;
      const bool ok = sOk[le];
      double ke[8] = {}, fe[4] = {}, re = 0.0;
      for (int q = 0; q < nq; ++q) {
        const double* A = sQ[le * 4 + q];
        const double* P = A + 10;
        const double* G = S.geo + (S.et[e] * nq + q) * 9;
        const double wq = G[8];
        const double ga0 = G[2 * a], ga1 = G[2 * a + 1];
        double t[4];  // row (a, i): t[k] = sum_J g_a[J] A[(i,J), k]
        for (int k = 0; k < 4; ++k) t[k] = ga0 * A[sym4(2 * i, k)] + ga1 * A[sym4(2 * i + 1, k)];
        for (int k = 0; k < 4; ++k) fe[k] += wq * t[k];
        re += wq * (ga0 * P[2 * i] + ga1 * P[2 * i + 1]);
        for (int bb = 0; bb < 4; ++bb)
          for (int j = 0; j < 2; ++j)  // column (b, j): sum_L t[(j,L)] g_b[L]
            ke[2 * bb + j] += wq * (t[2 * j] * G[2 * bb] + t[2 * j + 1] * G[2 * bb + 1]);
        if (row < 5 && ok)  // running qp sums of A (rows 0-3: 4 entries each) and P (row 4) for <A>, <P>
          for (int k = 0; k < 4; ++k) avg[k] += wq * (row < 4 ? A[sym4(row, k)] : P[k]);
      }
      for (int k = 0; k <= row; ++k) ske[le * 36 + pk8(row, k)] = ok ? ke[k] : 0.0;  // lower part
      for (int k = 0; k < 4; ++k) st_hint(o + EL_F + row * 4 + k, ok ? fe[k] : 0.0, pol);
      st_hint(o + EL_R + row, ok ? re : 0.0, pol);
    }
  }
  __syncthreads();  // sQ reused by the next block
}

template <int DIM, bool ISO, bool GT = false>  // GT: global geometry tables (RveDev::gtab)
__device__ __forceinline__ void assemble_rve(const RveDev& R, const int b, const int bl, double* __restrict__ Kt,
                                             double* __restrict__ Y, double* __restrict__ Cavg,
                                             double* __restrict__ Pavg, double* __restrict__ rfn,
                                             const double* __restrict__ EL, double* smem,
                                             const double* KE = nullptr, int kes = 0) {  // finite strain: K_e, stride
  constexpr int NSTR = DIM * TILE;  // [8 warps][npw][DIM][64] tile-row buffers
  double* s_row = smem;
  double* red = s_row + (NTHR / 32) * R.npw * NSTR;  // [NTHR] reduction scratch
  // ISO element tables: [ntype][n_phase][ND][ND] (K_e) and [ntype][n_phase][ND][m] (K_fe rows) per RVE in shared
  // memory, or -- when they do not fit (R.gtab: meshes with many distinct element geometries) -- only the
  // per-phase (lam, mu) here and the geometry tables Klam/Kmu/FlamT/FmuT read from global memory (L2)
  // K_e tables block-major: [tab][a][b][BS] with the DIM x DIM block (a, b) contiguous, padded to BS doubles
  // (16-byte multiple) so a gather is BS/2 128-bit shared-memory loads instead of DIM^2 64-bit ones
  constexpr int NEN = 1 << DIM, BS = ((DIM * DIM + 1) / 2) * 2;
  const int ntab = ISO ? (GT ? 0 : R.ntype * R.n_phase) : 0;
  double* s_K = red + NTHR;
  double* s_F = s_K + (ISO ? (GT ? 2 * R.n_phase : ntab * NEN * NEN * BS) : 0);
  double* s_C = s_F + (ISO ? ntab * ((1 << DIM) * DIM) * R.m : 0);  // stencil-class blocks [ncls][ntab][BS]
  const int ncls = (ISO && !GT) ? R.ncls : 0;
  int* s_ep = reinterpret_cast<int*>(s_C + ncls * ntab * BS);
  // per independent node: the one (type, phase) table of all its incident elements, 255 = several (class path)
  uint8_t* s_nt = reinterpret_cast<uint8_t*>(s_ep + R.ne);
  const int tid = threadIdx.x;
  const int ne = R.ne;
  constexpr int ND = ISO ? (1 << DIM) * DIM : 8;  // nen*dim

  if (ISO) {
    const uint8_t* ph = R.phase + (R.phase_per_rve ? (long)b * ne : 0);
    const double* mt = R.mat + (R.mat_per_rve ? (long)b * R.n_phase * R.mat_stride : 0);
    if (GT) {  // (type << 8 | phase) per element, (lam, mu) per phase
      for (int e = tid; e < ne; e += NTHR) s_ep[e] = (R.etype[e] << 8) | ph[e];
      for (int pp = tid; pp < R.n_phase; pp += NTHR) {
        const double E = mt[2 * pp], nu = mt[2 * pp + 1];
        s_K[2 * pp] = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
        s_K[2 * pp + 1] = E / (2.0 * (1.0 + nu));
      }
    } else {
      for (int e = tid; e < ne; e += NTHR) s_ep[e] = R.etype[e] * R.n_phase + ph[e];
    }
    // K_e = lam Klam_t + mu Kmu_t for every (element type t, phase) of this RVE
    for (int i = tid; i < ntab * ND * ND; i += NTHR) {
      const int t = i / (R.n_phase * ND * ND), pp = (i / (ND * ND)) % R.n_phase, j = i % (ND * ND);
      const double E = mt[2 * pp], nu = mt[2 * pp + 1];
      const double lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), mu = E / (2.0 * (1.0 + nu));
      const int r = j / ND, c = j % ND;
      s_K[(((long)(i / (ND * ND)) * NEN + r / DIM) * NEN + c / DIM) * BS + (r % DIM) * DIM + c % DIM] =
          lam * R.Klam[(long)t * ND * ND + j] + mu * R.Kmu[(long)t * ND * ND + j];
    }
    for (int i = tid; i < ntab * ND * R.m; i += NTHR) {  // K_fe element tables
      const int t = i / (R.n_phase * ND * R.m), pp = (i / (ND * R.m)) % R.n_phase, j = i % (ND * R.m);
      const double E = mt[2 * pp], nu = mt[2 * pp + 1];
      const double lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), mu = E / (2.0 * (1.0 + nu));
      s_F[i] = lam * R.FlamT[(long)t * ND * R.m + j] + mu * R.FmuT[(long)t * ND * R.m + j];
    }
  }
  __syncthreads();
  if (ncls)
    for (int p = tid; p < R.n_indep; p += NTHR) {
      const int s0 = R.inc_ptr[p], s1 = R.inc_ptr[p + 1];
      int t = s1 > s0 ? s_ep[R.inc[s0] >> 4] : 255;
      for (int u = s0 + 1; u < s1; ++u)
        if (s_ep[R.inc[u] >> 4] != t) t = 255;
      s_nt[p] = (uint8_t)(t < 255 ? t : 255);
    }
  // stencil-class blocks: C_c,t = sum over the class's element-local pairs (a, b) of the table t block
  // (read by records whose shared elements all use table t; ordered before the gathers by the
  // barriers of the <C> reduction below)
  if (ISO && !GT)
  for (int i = tid; i < ncls * ntab * BS; i += NTHR) {
    const int cl = i / max(ntab * BS, 1), t = (i / BS) % max(ntab, 1), j = i % BS;
    double v = 0.0;
    if (j < DIM * DIM)
      for (int u = __ldg(R.cls_ptr + cl); u < __ldg(R.cls_ptr + cl + 1); ++u) {
        const int ab = __ldg(R.cls_ab + u);
        v += s_K[(((long)t * NEN + (ab >> 4)) * NEN + (ab & 15)) * BS + j];
      }
    s_C[i] = v;
  }

  // ---- volume average <C> (small strain; finite strain: <A>, <P> come from the element pass) ----
  if (ISO) {
    constexpr int NV = 2;
    double acc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) acc[i] = 0.0;
    if (ISO) {
      const uint8_t* ph = R.phase + (R.phase_per_rve ? (long)b * ne : 0);
      const double* mt = R.mat + (R.mat_per_rve ? (long)b * R.n_phase * R.mat_stride : 0);
      for (int e = tid; e < ne; e += NTHR) {
        const int p = ph[e];
        const double E = mt[2 * p], nu = mt[2 * p + 1], v = R.evol[e];
        acc[0] += v * (E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)));
        acc[1] += v * (E / (2.0 * (1.0 + nu)));
      }
    }
    // one pass: warp shuffles, then NV partial rows in smem
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[v] += __shfl_down_sync(0xffffffffu, acc[v], o);
    }
    if (lane == 0)
#pragma unroll
      for (int v = 0; v < NV; ++v) red[v * 8 + warp] = acc[v];
    __syncthreads();
    if (tid == 0) {
      double tot[NV];
      for (int v = 0; v < NV; ++v) {
        tot[v] = 0.0;
        for (int w = 0; w < NTHR / 32; ++w) tot[v] += red[v * 8 + w];
        tot[v] /= R.vol;
      }
      double* C = Cavg + (long)bl * 64;
      if (ISO) {
        const int m = R.m;
        for (int i = 0; i < m * m; ++i) C[i] = 0.0;
        for (int i = 0; i < DIM; ++i)
          for (int j = 0; j < DIM; ++j) C[i * m + j] = tot[0] + (i == j ? 2.0 * tot[1] : 0.0);
        for (int i = DIM; i < m; ++i) C[i * m + i] = tot[1];
      } else {
      }
    }
    __syncthreads();
  }

  // ---- right-hand sides: K_fe (cols 0..m-1) and r_f (col m, finite strain) ----
  {
    double rr = 0.0;
    double* Yb = Y + (long)bl * R.NT * RHSW;
    for (int i = tid; i < R.NT; i += NTHR) {
      double out[RHSW];
#pragma unroll
      for (int k = 0; k < RHSW; ++k) out[k] = 0.0;
      int p = i / DIM, c = i % DIM;
      if (i < R.npad && p != R.corner) {
        for (int s = R.inc_ptr[p]; s < R.inc_ptr[p + 1]; ++s) {
          int e = R.inc[s] >> 4, a = R.inc[s] & 15;
          if (ISO && GT) {
            const int tp = s_ep[e], t = tp >> 8, pp = tp & 255;
            const double lam = s_K[2 * pp], mu = s_K[2 * pp + 1];
            const long o = ((long)t * ND + a * DIM + c) * R.m;
#pragma unroll
            for (int k = 0; k < RHSW; ++k)
              if (k < R.m) out[k] += lam * __ldg(R.FlamT + o + k) + mu * __ldg(R.FmuT + o + k);
          } else if (ISO) {
            const double* fe = s_F + ((long)s_ep[e] * ND + a * DIM + c) * R.m;
#pragma unroll
            for (int k = 0; k < RHSW; ++k)
              if (k < R.m) out[k] += fe[k];
          } else {
            const double* el = EL + (long)e * EL_STRIDE;
            const int rw = a * DIM + c;
            for (int k = 0; k < 4; ++k) out[k] += el[EL_F + rw * 4 + k];
            out[4] += el[EL_R + rw];
          }
        }
        if (!ISO) rr += out[4] * out[4];
      }
      double2* dst = reinterpret_cast<double2*>(Yb + (long)i * RHSW);
#pragma unroll
      for (int k = 0; k < RHSW / 2; ++k) dst[k] = make_double2(out[2 * k], out[2 * k + 1]);
    }
    if (!ISO) {  // ||r_f|| over the free DOFs (R_micro)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) rr += __shfl_xor_sync(0xffffffffu, rr, o);  // fixed-order tree
      if ((tid & 31) == 0) red[tid >> 5] = rr;
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < NTHR / 32; ++w) t += red[w];
        rfn[b] = sqrt(t);
      }
    }
  }

  // ---- K_ff tiles: node-row gather, coalesced direct stores ----
  // A work item is nn <= R.npw consecutive row nodes of one tile whose in-tile neighbour blocks
  // (<= 32, packed on the host) are one per lane: the lane forms the DIM x DIM block K_pq of
  // its record (sum over the shared elements of the per-(type, phase) element matrix; the
  // periodic map is applied through the independent-node numbering) in the warp's row buffer;
  // then every lane stores its two columns of the nn*DIM rows (512 B per row per warp).
  // Structurally zero tiles are never touched (k_condense starts their accumulators at zero).
  double* Kb = Kt + (long)bl * R.nslot * TILE_ELEMS;
  const int lane = tid & 31, warp = tid >> 5;
  double* rowbuf = s_row + warp * R.npw * NSTR;
  // work items {tile, first row node p0, nn nodes} with one in-tile neighbour record per lane,
  // software-pipelined: the next item's header and gather record and the lane word of the item
  // after it are in flight while the current item is formed and stored
  // record int4s held per lane: 2-D all (<= 4 shared elements), 3-D the first 6 codes (the self pair's 8 are
  // loaded on demand; 3 int4s measured 2.70 vs 2.59 ms at config 4, 1 int4 2.85 ms)
  constexpr int RS4M = DIM == 3 ? 2 : (DIM == 2 ? 2 : 1);
  constexpr int WSTRIDE = NTHR / 32;
  const int nw = R.n_witem;
  auto load_rec = [&](int (&rv)[4 * RS4M], int lwv) {
#pragma unroll
    for (int u = 0; u < RS4M; ++u) {
      const int4 v = (lwv >= 0 && u < R.rs4) ? __ldg(R.nrec + (long)(lwv & 0xffffff) * R.rs4 + u)
                                             : make_int4(-1, -1, -1, -1);
      rv[4 * u] = v.x; rv[4 * u + 1] = v.y; rv[4 * u + 2] = v.z; rv[4 * u + 3] = v.w;
    }
  };
  int4 wi = warp < nw ? __ldg(R.witem + warp) : make_int4(0, 0, 0, 0);
  int lw = warp < nw ? __ldg(R.wlist + (long)warp * 32 + lane) : -1;
  int rv[4 * RS4M];
  load_rec(rv, lw);
  int cw = warp < nw ? __ldg(R.wcov + (long)warp * 32 + lane) : 0;
  int lw1 = warp + WSTRIDE < nw ? __ldg(R.wlist + (long)(warp + WSTRIDE) * 32 + lane) : -1;
  for (int it = warp; it < nw; it += WSTRIDE) {
    const int itn = it + WSTRIDE;
    const int4 wi_n = itn < nw ? __ldg(R.witem + itn) : wi;
    const int cw_n = itn < nw ? __ldg(R.wcov + (long)itn * 32 + lane) : 0;
    int rv_n[4 * RS4M];
    load_rec(rv_n, lw1);
    const int lw2 = itn + WSTRIDE < nw ? __ldg(R.wlist + (long)(itn + WSTRIDE) * 32 + lane) : -1;
    const int I = wi.x >> 16, J = wi.x & 0xffff;
    const int r0 = I * TILE;
    const int p0 = wi.y, nn = wi.z & 0xff;
    const bool ipad = (wi.z >> 8) & 1;  // the item has identity rows
    HOM_DCHECK(wi.w >= 0 && wi.w < R.nslot && nn <= R.npw);
    double* gt = Kb + (long)wi.w * TILE_ELEMS;
    const int c0 = J * TILE;
    // the item's rows inside the tile are contiguous: local rows j (node j / DIM, row j % DIM of it)
    const int jb = p0 * DIM - r0, j0 = max(0, -jb), j1 = min(nn * DIM, TILE - jb);
    {
      {
        // (no clearing of the row buffer: columns no neighbour block covers are stored as zeros, cw)
        if (lw >= 0) {
          HOM_DCHECK((lw >> 24) < nn && p0 + (lw >> 24) < R.n_indep);
          double* rb = rowbuf + (lw >> 24) * NSTR;
          {
            const int4* rec = R.nrec + (long)(lw & 0xffffff) * R.rs4;
            // the record was loaded a round earlier (rv); records longer than RS4M int4s (tiny
            // periodic meshes) fall back to extra loads
            const int q = rv[0];
            const int cq = q * DIM - c0;  // first column of q in this tile
            double blk[DIM][DIM];
#pragma unroll
            for (int i = 0; i < DIM; ++i)
#pragma unroll
              for (int jj = 0; jj < DIM; ++jj) blk[i][jj] = 0.0;
            const int nsh = rv[1] & 0xffff, cls = (rv[1] >> 16) - 1;
            // element block (a, b) of the element in `code`: the per-(type, phase) table in shared memory
            // (small strain) or the CTA's L2-resident element record, K_e packed lower-triangular
            auto blk_at = [&](int code, int i, int jj) -> double {
              const int e = code >> 8, r = ((code >> 4) & 15) * DIM + i, c = (code & 15) * DIM + jj;
              if (ISO && GT) {
                const int tp = s_ep[e], t = tp >> 8, pp = tp & 255;
                const long o = (long)t * ND * ND + r * ND + c;
                return s_K[2 * pp] * __ldg(R.Klam + o) + s_K[2 * pp + 1] * __ldg(R.Kmu + o);
              }
              if (ISO) {
                const int a = (code >> 4) & 15, bb = code & 15;
                return s_K[(((long)s_ep[e] * NEN + a) * NEN + bb) * BS + i * DIM + jj];
              }
              HOM_DCHECK(e < ne && r < 8 && c < 8);
              return KE[(long)e * kes + pk8(r, c)];
            };
            // a record of a node whose incident elements all use one (type, phase) table: the class block
            // of that table, one gather
            bool uni = false;
            if (ISO && !GT && cls >= 0) {
              const int t0 = s_nt[p0 + (lw >> 24)];
              uni = t0 != 255;
              HOM_DCHECK(cls < ncls && (!uni || t0 < ntab));
              if (uni) {
                const double2* kb = reinterpret_cast<const double2*>(s_C + ((long)cls * ntab + t0) * BS);
#pragma unroll
                for (int q = 0; q < BS / 2; ++q) {
                  const double2 t2 = kb[q];
                  if (2 * q < DIM * DIM) blk[(2 * q) / DIM][(2 * q) % DIM] = t2.x;
                  if (2 * q + 1 < DIM * DIM) blk[(2 * q + 1) / DIM][(2 * q + 1) % DIM] = t2.y;
                }
              }
            }
#pragma unroll
            for (int sidx = 0; sidx < 4 * RS4M - 2 + 1; ++sidx) {
              if (uni || sidx >= nsh) break;
              if (sidx < 4 * RS4M - 2) {
                const int code = rv[sidx + 2];
                if (ISO && !GT) {  // the whole block with BS/2 128-bit loads
                  const int e = code >> 8, a = (code >> 4) & 15, bb = code & 15;
                  HOM_DCHECK(e < ne && a < NEN && bb < NEN && s_ep[e] < ntab);
                  const double2* kb = reinterpret_cast<const double2*>(s_K + (((long)s_ep[e] * NEN + a) * NEN + bb) * BS);
                  double v[BS];
#pragma unroll
                  for (int q = 0; q < BS / 2; ++q) {
                    const double2 t2 = kb[q];
                    v[2 * q] = t2.x;
                    v[2 * q + 1] = t2.y;
                  }
#pragma unroll
                  for (int i = 0; i < DIM; ++i)
#pragma unroll
                    for (int jj = 0; jj < DIM; ++jj) blk[i][jj] += v[i * DIM + jj];
                } else {
#pragma unroll
                  for (int i = 0; i < DIM; ++i)
#pragma unroll
                    for (int jj = 0; jj < DIM; ++jj) blk[i][jj] += blk_at(code, i, jj);
                }
              } else {  // rare: records longer than RS4M int4s (tiny periodic meshes)
                for (int s2 = sidx; s2 < nsh; ++s2) {
                  const int slot = s2 + 2;
                  const int4 vv = __ldg(rec + (slot >> 2));
                  const int c2 = (slot & 3) == 0 ? vv.x : (slot & 3) == 1 ? vv.y : (slot & 3) == 2 ? vv.z : vv.w;
                  for (int i = 0; i < DIM; ++i)
                    for (int jj = 0; jj < DIM; ++jj) blk[i][jj] += blk_at(c2, i, jj);
                }
                break;
              }
            }
#pragma unroll
            for (int i = 0; i < DIM; ++i)
#pragma unroll
              for (int jj = 0; jj < DIM; ++jj) {
                const int cc = cq + jj;
                if (cc >= 0 && cc < TILE) rb[i * TILE + cc] = blk[i][jj];
              }
          }
        }
        __syncwarp();
        auto row_store = [&](int j, double2 v) {
          if (ISO) __stcg(reinterpret_cast<double2*>(gt + (jb + j) * TILE + 2 * lane), v);
          else __stcs(reinterpret_cast<double2*>(gt + (jb + j) * TILE + 2 * lane), v);  // evict-first: keep records in L2
        };
        if (!ipad) {
#pragma unroll 3
          for (int j = j0; j < j1; ++j) {
            double2 v = *reinterpret_cast<const double2*>(rowbuf + j * TILE + 2 * lane);
            const int cb = cw >> (2 * (j / DIM));
            if (!(cb & 1)) v.x = 0.0;
            if (!(cb & 2)) v.y = 0.0;
            row_store(j, v);
          }
        } else {
          for (int j = j0; j < j1; ++j) {
            double2 v = *reinterpret_cast<const double2*>(rowbuf + j * TILE + 2 * lane);
            const int n = j / DIM, cb = cw >> (2 * n);
            if (!(cb & 1)) v.x = 0.0;
            if (!(cb & 2)) v.y = 0.0;
            const int pn = p0 + n, row = jb + r0 + j;
            if (pn >= R.n_indep || pn == R.corner) {  // identity rows (corner class, tail)
              v.x = (c0 + 2 * lane == row) ? 1.0 : 0.0;
              v.y = (c0 + 2 * lane + 1 == row) ? 1.0 : 0.0;
            }
            row_store(j, v);
          }
        }
        __syncwarp();
      }
    }
    wi = wi_n;
    cw = cw_n;
    lw = lw1;
#pragma unroll
    for (int u = 0; u < 4 * RS4M; ++u) rv[u] = rv_n[u];
    lw1 = lw2;
  }
}

template <int DIM, bool ISO, bool GT>
__global__ void __launch_bounds__(NTHR) k_rve_assemble(RveDev R, int b0, double* __restrict__ Kt,
                                                       double* __restrict__ Y, double* __restrict__ Cavg,
                                                       double* __restrict__ Pavg, double* __restrict__ rfn) {
  extern __shared__ __align__(128) double smem[];
  assemble_rve<DIM, ISO, GT>(R, b0 + blockIdx.x, blockIdx.x, Kt, Y, Cavg, Pavg, rfn, nullptr, smem);
}

// Finite strain, fused: a persistent CTA per slot walks its RVEs; for each it first
// evaluates every material point and forms the element records into its own scratch slice (one
// RVE, ne x EL_STRIDE doubles, written and read back by the same CTA while L2-resident), then runs
// the tile writer from them -- no batch-wide element table round trip through HBM.
// KS: the RVE's K_e (36 doubles per element) stays in shared memory for the tile writer (2 CTAs per SM);
// otherwise every record lives in the L2 scratch (4 CTAs per SM)
template <bool KS>
__global__ void __launch_bounds__(NTHR, KS ? 2 : 4) k_rve_assemble_fs(RveDev R, int b0, int nb, const double* __restrict__ Fbar,
                                                          const double* __restrict__ w, double* __restrict__ Kt,
                                                          double* __restrict__ Y, double* __restrict__ Cavg,
                                                          double* __restrict__ Pavg, double* __restrict__ rfn,
                                                          double* __restrict__ scratch, int* __restrict__ jflag) {
  extern __shared__ __align__(128) double smem[];
  __shared__ int sOk[FS_ELB2];
  double* scr = scratch + (long)blockIdx.x * R.ne * EL_STRIDE;
  double* sKe = KS ? smem + R.fs_ke_off : nullptr;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, row = tid & 7;
  for (int bl = blockIdx.x; bl < nb; bl += gridDim.x) {
    const int b = b0 + bl;
    double avg[4] = {0.0, 0.0, 0.0, 0.0};  // this thread's share of sum eta A (row < 4) / sum eta P (row 4)
    if (KS && R.fs_ntype > 0) {  // staged material pass
      const FsStage S = fs_stage_layout(R, smem);
      fs_stage(R, b, w, S);
      for (int e0 = 0; e0 < R.ne; e0 += FS_ELB2)
        nh_elements_st(R, b, e0, min(FS_ELB2, R.ne - e0), Fbar, jflag, smem, sOk, avg, sKe + (long)e0 * 36, S,
                       scr + (long)e0 * EL_STRIDE);
    } else {
      for (int e0 = 0; e0 < R.ne; e0 += FS_ELB)
        nh_elements(R, b, e0, min(FS_ELB, R.ne - e0), Fbar, w, scr + (long)e0 * EL_STRIDE, jflag, smem, sOk, avg,
                    KS ? sKe + (long)e0 * 36 : nullptr);
    }
    // <A>, <P>: sum over the elements (lanes with equal row: xor 8, 16; then the 8 warps), / |Omega|
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      avg[k] += __shfl_xor_sync(0xffffffffu, avg[k], 8);
      avg[k] += __shfl_xor_sync(0xffffffffu, avg[k], 16);
    }
    double* red = smem;  // [8 warps][5 rows][4]
    if (lane < 5)
#pragma unroll
      for (int k = 0; k < 4; ++k) red[(warp * 5 + row) * 4 + k] = avg[k];
    __syncthreads();
    if (tid < 20) {
      double t = 0.0;
      for (int wv = 0; wv < NTHR / 32; ++wv) t += red[wv * 20 + tid];
      t /= R.vol;
      if (tid < 16) Cavg[(long)bl * 64 + tid] = t;
      else Pavg[(long)bl * 8 + tid - 16] = t;
    }
    __syncthreads();
    if (KS) assemble_rve<2, false>(R, b, bl, Kt, Y, Cavg, Pavg, rfn, scr, smem, sKe, 36);
    else assemble_rve<2, false>(R, b, bl, Kt, Y, Cavg, Pavg, rfn, scr, smem, scr + EL_K, EL_STRIDE);
    __syncthreads();
  }
}

size_t rve_assemble_smem(const RveDev& R, int npw) {
  const int dim = R.finite ? 2 : R.dim, nd = (1 << dim) * dim;  // nen*dim
  size_t sm = (size_t)((NTHR / 32) * npw * dim * TILE + NTHR) * sizeof(double) +
              (R.finite ? 0
                   : (R.gtab ? (size_t)2 * R.n_phase
                             : (size_t)R.ntype * R.n_phase * ((size_t)(R.ncls + (1 << dim) * (1 << dim)) * ((dim * dim + 1) / 2 * 2) + nd * R.m)) *
                                 sizeof(double) +
                         (size_t)R.ne * sizeof(int) + (R.ncls ? (size_t)R.n_indep : 0));
  if (R.finite) sm = std::max(sm, (size_t)FS_SMEM_DBL * sizeof(double));  // element staging aliases the row buffers
  if (R.finite && R.fs_ks && R.fs_ntype > 0)  // staged material pass (w, phases, connectivity, qp geometry)
    sm = std::max(sm, (size_t)(FS_ELB2 * 4 * FS_QW2 + R.npad + R.fs_ntype * R.nq * 9) * 8 + (size_t)R.ne * 5 * 4 + R.ne);
  if (R.finite && R.fs_ks) sm = ((sm + 127) / 128) * 128 + (size_t)R.ne * 36 * sizeof(double);  // + K_e of the RVE
  return sm;
}

int rve_assemble_npw(const RveDev& R) {
  // largest row buffer (<= 16 rows per warp) that keeps 4 CTAs per SM (<= 56 KB each), or 2 CTAs per SM
  // (<= 112 KB) for the finite-strain kernel with K_e in shared memory
  const int dim = R.finite ? 2 : R.dim;
  const size_t budget = (R.finite && R.fs_ks) ? 112 * 1024 : 56 * 1024;
  int npw = std::min(8, 16 / dim);
  while (npw > 1 && rve_assemble_smem(R, npw) > budget) --npw;
  return npw;
}

int rve_assemble_fs_slots(const RveDev& R) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t sm = rve_assemble_smem(R, R.npw);
  auto k = R.fs_ks ? k_rve_assemble_fs<true> : k_rve_assemble_fs<false>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, NTHR, sm);
  return std::max(1, per) * std::max(1, sms);
}

void launch_rve_assemble_fs(const RveDev& R, int b0, int nb, const double* F, const double* w, double* Kt,
                            double* Y, double* Cavg, double* Pavg, double* rfn, double* scratch, int slots,
                            int* jflag, cudaStream_t s) {
  const size_t sm = rve_assemble_smem(R, R.npw);
  auto k = R.fs_ks ? k_rve_assemble_fs<true> : k_rve_assemble_fs<false>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  k<<<std::min(nb, slots), NTHR, sm, s>>>(R, b0, nb, F, w, Kt, Y, Cavg, Pavg, rfn, scratch, jflag);
}

template <int DIM, bool GT>
static void launch_k1(const RveDev& R, int b0, int nb, double* Kt, double* Y, double* Cavg, double* Pavg, double* rfn,
                      size_t sm, cudaStream_t s) {
  auto k = k_rve_assemble<DIM, true, GT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  k<<<nb, NTHR, sm, s>>>(R, b0, Kt, Y, Cavg, Pavg, rfn);
}

void launch_rve_assemble(const RveDev& R, int b0, int nb, double* Kt, double* Y, double* Cavg, double* Pavg,
                         double* rfn, cudaStream_t s) {
  const size_t sm = rve_assemble_smem(R, R.npw);
  if (R.dim == 1)  // the paper's 1-D benchmark on the device
    R.gtab ? launch_k1<1, true>(R, b0, nb, Kt, Y, Cavg, Pavg, rfn, sm, s)
           : launch_k1<1, false>(R, b0, nb, Kt, Y, Cavg, Pavg, rfn, sm, s);
  else if (R.dim == 2)
    R.gtab ? launch_k1<2, true>(R, b0, nb, Kt, Y, Cavg, Pavg, rfn, sm, s)
           : launch_k1<2, false>(R, b0, nb, Kt, Y, Cavg, Pavg, rfn, sm, s);
  else
    R.gtab ? launch_k1<3, true>(R, b0, nb, Kt, Y, Cavg, Pavg, rfn, sm, s)
           : launch_k1<3, false>(R, b0, nb, Kt, Y, Cavg, Pavg, rfn, sm, s);
}

}  // namespace hom
