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
__global__ void k_rve_material_nh(RveDev R, int b0, int nb, const double* __restrict__ Fbar,
                                  const double* __restrict__ w, double* __restrict__ Aq,
                                  double* __restrict__ Pq, int* __restrict__ jflag) {
  const int per = R.ne * R.nq;
  long gid = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long)nb * per) return;
  int bl = (int)(gid / per), eq = (int)(gid % per);
  int e = eq / R.nq, q = eq % R.nq;
  int b = b0 + bl;
  const double* Fb = Fbar + (long)b * 4;
  double F[4] = {Fb[0], Fb[1], Fb[2], Fb[3]};
  const double* wb = w + (long)b * R.npad;
  for (int a = 0; a < R.nen; ++a) {
    int p = R.elem_indep[e * R.nen + a];
    const double* g = R.grad + ((long)(e * R.nq + q) * R.nen + a) * 2;
    double w0 = wb[2 * p], w1 = wb[2 * p + 1];
    F[0] += w0 * g[0]; F[1] += w0 * g[1];
    F[2] += w1 * g[0]; F[3] += w1 * g[1];
  }
  int ph = R.phase[(R.phase_per_rve ? (long)b * R.ne : 0) + e];
  const int np = R.mat_stride;
  const double* mp = R.mat + (R.mat_per_rve ? (long)b * R.n_phase * np : 0) + np * ph;
  const double alpha = mp[0], beta = np == 3 ? mp[1] : 0.0, kappa = mp[np - 1];
  // J - 1 from the displacement-gradient part (no cancellation near F = I)
  const double g11 = F[0] - 1.0, g22 = F[3] - 1.0;
  const double Jm1 = g11 + g22 + g11 * g22 - F[1] * F[2];
  double J = 1.0 + Jm1;
  double* A = Aq + gid * 16;
  double* P = Pq + gid * 4;
  if (!(J > 0.0)) {
    atomicMin(&jflag[b], eq);  // first failing qp of this RVE (jflag init INT_MAX)
    for (int i = 0; i < 16; ++i) A[i] = 0.0;
    for (int i = 0; i < 4; ++i) P[i] = 0.0;
    return;
  }
  double H[4] = {F[3], -F[2], -F[1], F[0]};  // cof F (2-D specialisation of 1/2 F xx F)
  const double ab = alpha + 2.0 * beta;
  double dPsidJ = 2.0 * beta * J + kappa * Jm1 - 2.0 * ab / J;
  double d2 = 2.0 * beta + kappa + 2.0 * ab / (J * J);
  // P = 2 (alpha + beta) F + g H written as 2 (alpha + beta)(F - H) + (g + 2 (alpha + beta)) H with
  // g + 2 (alpha + beta) = (J - 1)(2 beta + kappa + 2 (alpha + 2 beta) / J): both terms vanish at F = I
  // (the stress-free reference) instead of cancelling, so R_micro reaches ~1e-15 (classical scheme)
  const double c0 = 2.0 * (alpha + beta), c1 = Jm1 * (2.0 * beta + kappa + 2.0 * ab / J);
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
}

void launch_rve_material_nh(const RveDev& R, int b0, int nb, const double* F, const double* w,
                            double* Aq, double* Pq, int* jflag, cudaStream_t s) {
  long n = (long)nb * R.ne * R.nq;
  int thr = 256;
  k_rve_material_nh<<<(unsigned)((n + thr - 1) / thr), thr, 0, s>>>(R, b0, nb, F, w, Aq, Pq, jflag);
}

// ---------------------------------------------------------------------------
// K1: assembly.  ISO (small strain): element blocks from geometry-only tables,
// K_e = lam_e Klam_e + mu_e Kmu_e (isotropic closed form K_ab^{ij} = lam g_a^i g_b^j
// + mu g_a^j g_b^i + mu d_ij g_a.g_b integrated at setup).  Finite strain: the
// tangent is read per qp from Aq (full-gradient form).
//
// Tiles: only the structurally nonzero tiles (per-mesh bitmap) are written,
// row by row with coalesced 16-byte stores (see the tile writer below).
// ---------------------------------------------------------------------------


template <int DIM, bool ISO>
__global__ void __launch_bounds__(NTHR) k_rve_assemble(RveDev R, int b0, double* __restrict__ Kt,
                                                       double* __restrict__ Y, double* __restrict__ Cavg,
                                                       double* __restrict__ Pavg, double* __restrict__ rfn,
                                                       const double* __restrict__ Aq,
                                                       const double* __restrict__ Pq) {
  extern __shared__ __align__(128) double smem[];
  double* s_row = smem;                      // [8 warps][npw][DIM][64] tile-row buffers
  double* red = s_row + (NTHR / 32) * R.npw * DIM * TILE;  // [NTHR] reduction scratch
  double* s_lam = red + NTHR;                // [ne] (ISO)
  double* s_mu = s_lam + R.ne;               // [ne] (ISO)
  double* s_K = s_mu + R.ne;                 // [ntype][n_phase][ND][ND] element matrices (ISO)
  int* s_ep = reinterpret_cast<int*>(s_K + (ISO ? R.ntype * R.n_phase * ((1 << DIM) * DIM) * ((1 << DIM) * DIM) : 0));
  const int tid = threadIdx.x;
  const int bl = blockIdx.x;
  const int b = b0 + bl;
  const int nen = R.nen, nq = R.nq, ne = R.ne;
  constexpr int ND = ISO ? (1 << DIM) * DIM : 8;  // nen*dim
  const long tq0 = (long)bl * ne * nq;  // offset of this RVE in Aq/Pq (chunk-local)

  if (ISO) {
    const uint8_t* ph = R.phase + (R.phase_per_rve ? (long)b * ne : 0);
    const double* mt = R.mat + (R.mat_per_rve ? (long)b * R.n_phase * R.mat_stride : 0);
    for (int e = tid; e < ne; e += NTHR) {
      int p = ph[e];
      double E = mt[2 * p], nu = mt[2 * p + 1];
      s_lam[e] = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
      s_mu[e] = E / (2.0 * (1.0 + nu));
      s_ep[e] = R.etype[e] * R.n_phase + p;
    }
    // K_e = lam Klam_t + mu Kmu_t for every (element type t, phase) of this RVE
    for (int i = tid; i < R.ntype * R.n_phase * ND * ND; i += NTHR) {
      const int t = i / (R.n_phase * ND * ND), pp = (i / (ND * ND)) % R.n_phase, j = i % (ND * ND);
      const double E = mt[2 * pp], nu = mt[2 * pp + 1];
      const double lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), mu = E / (2.0 * (1.0 + nu));
      s_K[i] = lam * R.Klam[(long)t * ND * ND + j] + mu * R.Kmu[(long)t * ND * ND + j];
    }
  }
  __syncthreads();

  // ---- volume averages <C> (and <P>) ----
  {
    constexpr int NV = ISO ? 2 : 20;
    double acc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) acc[i] = 0.0;
    if (ISO) {
      for (int e = tid; e < ne; e += NTHR) {
        double v = R.evol[e];
        acc[0] += v * s_lam[e];
        acc[1] += v * s_mu[e];
      }
    } else {
      for (int eq = tid; eq < ne * nq; eq += NTHR) {
        double wq = R.wdet[eq];
        const double* A = Aq + (tq0 + eq) * 16;
        const double* P = Pq + (tq0 + eq) * 4;
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] += wq * A[i];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[16 + i] += wq * P[i];
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
        for (int i = 0; i < 16; ++i) C[i] = tot[i];
        for (int i = 0; i < 4; ++i) Pavg[(long)bl * 8 + i] = tot[16 + i];
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
          if (ISO) {
            const double lam = s_lam[e], mu = s_mu[e];
            const double* fl = R.Flam + ((long)e * ND + a * DIM + c) * R.m;
            const double* fm = R.Fmu + ((long)e * ND + a * DIM + c) * R.m;
#pragma unroll
            for (int k = 0; k < RHSW; ++k)
              if (k < R.m) out[k] += lam * fl[k] + mu * fm[k];
          } else {
            for (int q = 0; q < nq; ++q) {
              const double* g = R.grad + ((long)(e * nq + q) * nen + a) * DIM;
              double wq = R.wdet[e * nq + q];
              const double* A = Aq + (tq0 + e * nq + q) * 16;
              const double* P = Pq + (tq0 + e * nq + q) * 4;
              for (int k = 0; k < 4; ++k) {
                double v = 0.0;
#pragma unroll
                for (int J = 0; J < DIM; ++J) v += g[J] * A[(c * DIM + J) * 4 + k];
                out[k] += wq * v;
              }
              double v = 0.0;
#pragma unroll
              for (int J = 0; J < DIM; ++J) v += g[J] * P[c * DIM + J];
              out[4] += wq * v;
            }
          }
        }
        if (!ISO) rr += out[4] * out[4];
      }
      double2* dst = reinterpret_cast<double2*>(Yb + (long)i * RHSW);
#pragma unroll
      for (int k = 0; k < RHSW / 2; ++k) dst[k] = make_double2(out[2 * k], out[2 * k + 1]);
    }
    if (!ISO) {  // ||r_f|| over the free DOFs (R_micro)
      red[tid] = rr;
      __syncthreads();
      for (int s = NTHR / 2; s > 0; s >>= 1) {
        if (tid < s) red[tid] += red[tid + s];
        __syncthreads();
      }
      if (tid == 0) rfn[b] = sqrt(red[0]);
      __syncthreads();
    }
  }

  // ---- K_ff tiles: node-row gather, coalesced direct stores ----
  // A warp owns R.npw consecutive RVE nodes p at a time; lane group g = lane / S (S = 32/npw)
  // serves node p0 + g and its lane j forms the DIM x DIM block K_pq of neighbour q = nbr(p, j)
  // (sum over the shared elements of the per-(type, phase) element matrix; the periodic map
  // is applied through the independent-node numbering) into the warp's row buffer; then every
  // lane stores its two columns of the npw*DIM rows (512 B per row per warp, 16 B per lane).
  // Structurally zero tiles are never touched (k_condense starts their accumulators at zero).
  const int nt = R.nt, npw = R.npw, S = 32 / npw;
  double* Kb = Kt + (long)bl * R.nslot * TILE_ELEMS;
  const int lane = tid & 31, warp = tid >> 5;
  double* rowbuf = s_row + warp * npw * DIM * TILE;
  const int g = lane / S, jl = lane % S;
  for (int I = 0; I < nt; ++I) {
    const int r0 = I * TILE;
    const int p_lo = r0 / DIM, p_hi = (r0 + TILE - 1) / DIM;  // nodes touching rows r0..r0+63
    for (int J = 0; J <= I; ++J) {
      if (!R.tile_nz[I * nt + J]) continue;
      double* gt = Kb + (long)R.tslot[I * nt + J] * TILE_ELEMS;
      const int c0 = J * TILE;
      for (int p0 = p_lo + warp * npw; p0 <= p_hi; p0 += (NTHR / 32) * npw) {
        for (int i = lane; i < npw * DIM * TILE / 2; i += 32)
          reinterpret_cast<double2*>(rowbuf)[i] = make_double2(0.0, 0.0);
        __syncwarp();
        const int p = p0 + g;
        if (g < npw && p <= p_hi && p < R.n_indep && p != R.corner) {
          double* rb = rowbuf + g * DIM * TILE;
          const int k0 = R.nbr_ptr[p], deg = R.nbr_ptr[p + 1] - k0;
          for (int j = jl; j < deg; j += S) {
            const int k = k0 + j, q = R.nbr[k];
            const int cq = q * DIM - c0;  // first column of q in this tile
            if (q == R.corner || cq + DIM <= 0 || cq >= TILE) continue;
            double blk[DIM][DIM];
#pragma unroll
            for (int i = 0; i < DIM; ++i)
#pragma unroll
              for (int jj = 0; jj < DIM; ++jj) blk[i][jj] = 0.0;
            for (int sh = R.sh_ptr[k]; sh < R.sh_ptr[k + 1]; ++sh) {
              const int code = R.sh[sh];
              const int e = code >> 8, a = (code >> 4) & 15, bb = code & 15;
              if (ISO) {
                const double* ke = s_K + (long)s_ep[e] * ND * ND + (a * DIM) * ND + bb * DIM;
#pragma unroll
                for (int i = 0; i < DIM; ++i)
#pragma unroll
                  for (int jj = 0; jj < DIM; ++jj) blk[i][jj] += ke[i * ND + jj];
              } else {
                for (int qq = 0; qq < nq; ++qq) {
                  const double* ga = R.grad + ((long)(e * nq + qq) * nen + a) * DIM;
                  const double* gb = R.grad + ((long)(e * nq + qq) * nen + bb) * DIM;
                  const double wq = R.wdet[e * nq + qq];
                  const double* A = Aq + (tq0 + e * nq + qq) * 16;
#pragma unroll
                  for (int i = 0; i < DIM; ++i)
#pragma unroll
                    for (int jj = 0; jj < DIM; ++jj) {
                      double v = 0.0;
#pragma unroll
                      for (int Jd = 0; Jd < DIM; ++Jd)
#pragma unroll
                        for (int Ld = 0; Ld < DIM; ++Ld) v += ga[Jd] * A[(i * DIM + Jd) * 4 + jj * DIM + Ld] * gb[Ld];
                      blk[i][jj] += wq * v;
                    }
                }
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
        for (int n = 0; n < npw; ++n) {
          const int pn = p0 + n;
          if (pn > p_hi) break;
          const bool pad = pn >= R.n_indep || pn == R.corner;  // identity rows (corner class, tail)
#pragma unroll
          for (int ci = 0; ci < DIM; ++ci) {
            const int row = pn * DIM + ci, rr = row - r0;
            if (rr < 0 || rr >= TILE) continue;
            double2 v = *reinterpret_cast<const double2*>(rowbuf + (n * DIM + ci) * TILE + 2 * lane);
            if (pad || row >= R.npad) {
              v.x = (c0 + 2 * lane == row) ? 1.0 : 0.0;
              v.y = (c0 + 2 * lane + 1 == row) ? 1.0 : 0.0;
            }
            __stcg(reinterpret_cast<double2*>(gt + rr * TILE + 2 * lane), v);
          }
        }
        __syncwarp();
      }
    }
  }
}

void launch_rve_assemble(const RveDev& R, int b0, int nb, double* Kt, double* Y, double* Cavg,
                         double* Pavg, double* rfn, const double* Aq, const double* Pq,
                         cudaStream_t s) {
  const int dim = R.finite ? 2 : R.dim, nd = (1 << dim) * dim;  // nen*dim
  size_t sm = (size_t)((NTHR / 32) * R.npw * dim * TILE + NTHR + 2 * R.ne) * sizeof(double) +
              (R.finite ? 0 : (size_t)R.ntype * R.n_phase * nd * nd * sizeof(double) + (size_t)R.ne * sizeof(int));
  if (R.finite) {
    auto k = k_rve_assemble<2, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<nb, NTHR, sm, s>>>(R, b0, Kt, Y, Cavg, Pavg, rfn, Aq, Pq);
  } else if (R.dim == 1) {  // the paper's 1-D benchmark on the device
    auto k = k_rve_assemble<1, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<nb, NTHR, sm, s>>>(R, b0, Kt, Y, Cavg, Pavg, rfn, Aq, Pq);
  } else if (R.dim == 2) {
    auto k = k_rve_assemble<2, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<nb, NTHR, sm, s>>>(R, b0, Kt, Y, Cavg, Pavg, rfn, Aq, Pq);
  } else {
    auto k = k_rve_assemble<3, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<<<nb, NTHR, sm, s>>>(R, b0, Kt, Y, Cavg, Pavg, rfn, Aq, Pq);
  }
}

}  // namespace hom
