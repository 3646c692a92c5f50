// macro.cu -- K5-K8: macro kinematics, condensed macro stiffness into CSR,
// right-hand side with Dirichlet lifting, Jacobi-PCG, fluctuation recovery.
//
// PAPER.md eq:linSys / eq:linSys2 with the condensed tangent of
// eq:solution1/2: K_M = sum_qp eta B_q^T D_b B_q and
// R = sum_qp eta B_q^T S_b - f_body.  Recovery follows eq:reduction
// and the dw update.  All reductions run in a fixed order so the
// results are bitwise reproducible.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "hom_internal.cuh"

namespace cgx = cooperative_groups;

namespace hom {

// Voigt strain-displacement entry B_a[k][c] from the gradient g of N_a.
template <int DIM>
__device__ __forceinline__ double voigtB(const double* g, int k, int c) {
  if (DIM == 1) return g[0];  // eps11 = du/dX
  if (DIM == 2) {
    if (k == 0) return c == 0 ? g[0] : 0.0;
    if (k == 1) return c == 1 ? g[1] : 0.0;
    return c == 0 ? g[1] : g[0];  // g12
  } else {
    switch (k) {
      case 0: return c == 0 ? g[0] : 0.0;
      case 1: return c == 1 ? g[1] : 0.0;
      case 2: return c == 2 ? g[2] : 0.0;
      case 3: return c == 1 ? g[2] : (c == 2 ? g[1] : 0.0);  // g23
      case 4: return c == 0 ? g[2] : (c == 2 ? g[0] : 0.0);  // g13
      default: return c == 0 ? g[1] : (c == 1 ? g[0] : 0.0); // g12
    }
  }
}

// ---------------------------------------------------------------- kinematics
template <int DIM>
__global__ void k_macro_kin(MacroDev M, const double* __restrict__ u, double* __restrict__ kin,
                            int add_identity) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (M.constant_basis) {  // element-average strain eps_bar_e = |B_e|^-1 sum_q eta B_q u_e
    if (t >= M.ne) return;
    double out[9];
    for (int k = 0; k < M.m; ++k) out[k] = 0.0;
    for (int q = 0; q < M.nq; ++q) {
      const int tq = t * M.nq + q;
      const double w = M.wdet[tq];
      for (int a = 0; a < M.nen; ++a) {
        const double* g = M.grad + ((long)tq * M.nen + a) * DIM;
        for (int c = 0; c < DIM; ++c) {
          const double uc = u[M.conn[t * M.nen + a] * DIM + c];
          for (int k = 0; k < M.m; ++k) out[k] += w * voigtB<DIM>(g, k, c) * uc;
        }
      }
    }
    for (int k = 0; k < M.m; ++k) kin[(long)t * M.m + k] = out[k] / M.evol[t];
    return;
  }
  if (t >= M.ne * M.nq) return;
  const int e = t / M.nq;  // qp t % nq: grad is indexed by t directly
  double out[9];
  for (int k = 0; k < M.m; ++k) out[k] = 0.0;
  for (int a = 0; a < M.nen; ++a) {
    int n = M.conn[e * M.nen + a];
    const double* g = M.grad + ((long)t * M.nen + a) * DIM;
    for (int c = 0; c < DIM; ++c) {
      double uc = u[n * DIM + c];
      if (M.finite) {
        for (int J = 0; J < DIM; ++J) out[c * DIM + J] += uc * g[J];
      } else {
        for (int k = 0; k < M.m; ++k) out[k] += voigtB<DIM>(g, k, c) * uc;
      }
    }
  }
  if (M.finite && add_identity)
    for (int i = 0; i < DIM; ++i) out[i * DIM + i] += 1.0;
  for (int k = 0; k < M.m; ++k) kin[(long)t * M.m + k] = out[k];
}

void launch_macro_kin(const MacroDev& M, const double* u, double* kin, int add_identity, cudaStream_t s) {
  int n = M.constant_basis ? M.ne : M.ne * M.nq;
  if (M.dim == 1) k_macro_kin<1><<<(n + 127) / 128, 128, 0, s>>>(M, u, kin, add_identity);
  else if (M.dim == 2) k_macro_kin<2><<<(n + 127) / 128, 128, 0, s>>>(M, u, kin, add_identity);
  else k_macro_kin<3><<<(n + 127) / 128, 128, 0, s>>>(M, u, kin, add_identity);
}

// ---------------------------------------------------------------- K5 assembly
template <int DIM>
__global__ void k_macro_assemble(MacroDev M, const double* __restrict__ D, double* __restrict__ val,
                                 double* __restrict__ diag) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= M.nnz) return;
  int blk = M.nz_blk[k];
  int ci = (M.nz_cc[k] >> 2) & 3, cj = M.nz_cc[k] & 3;
  const int m = M.m;
  double v = 0.0;
  for (int s = M.blk_ptr[blk]; s < M.blk_ptr[blk + 1]; ++s) {
    int code = M.blk_sh[s];
    int E = code >> 8, a = (code >> 4) & 15, b = code & 15;
    if (M.constant_basis) {
      // K_e = sum_q eta B_q^T <C>_e B_q - |B_e|^-1 (sum_q eta B_q)^T (<C>_e - C_eff,e) (sum_q eta B_q)
      const double* Ca = M.Cavg_e + (long)E * m * m;
      const double* Ce = D + (long)E * m * m;
      double ba[6] = {0, 0, 0, 0, 0, 0}, bb[6] = {0, 0, 0, 0, 0, 0};
      for (int q = 0; q < M.nq; ++q) {
        const int t = E * M.nq + q;
        const double* ga = M.grad + ((long)t * M.nen + a) * DIM;
        const double* gb = M.grad + ((long)t * M.nen + b) * DIM;
        const double w = M.wdet[t];
        double s2 = 0.0;
        for (int kk = 0; kk < m; ++kk) {
          const double bak = voigtB<DIM>(ga, kk, ci);
          ba[kk] += w * bak;
          bb[kk] += w * voigtB<DIM>(gb, kk, cj);
          if (bak == 0.0) continue;
          double t2 = 0.0;
          for (int l = 0; l < m; ++l) t2 += Ca[kk * m + l] * voigtB<DIM>(gb, l, cj);
          s2 += bak * t2;
        }
        v += w * s2;
      }
      double corr = 0.0;
      for (int kk = 0; kk < m; ++kk)
        for (int l = 0; l < m; ++l) corr += ba[kk] * (Ca[kk * m + l] - Ce[kk * m + l]) * bb[l];
      v -= corr / M.evol[E];
      continue;
    }
    for (int q = 0; q < M.nq; ++q) {
      int t = E * M.nq + q;
      const double* ga = M.grad + ((long)t * M.nen + a) * DIM;
      const double* gb = M.grad + ((long)t * M.nen + b) * DIM;
      const double* Dq = D + (long)t * m * m;
      double w = M.wdet[t], s2 = 0.0;
      if (M.finite) {
        for (int J = 0; J < DIM; ++J)
          for (int L = 0; L < DIM; ++L) s2 += ga[J] * Dq[(ci * DIM + J) * m + cj * DIM + L] * gb[L];
      } else {
        for (int kk = 0; kk < m; ++kk) {
          double bak = voigtB<DIM>(ga, kk, ci);
          if (bak == 0.0) continue;
          double t2 = 0.0;
          for (int l = 0; l < m; ++l) t2 += Dq[kk * m + l] * voigtB<DIM>(gb, l, cj);
          s2 += bak * t2;
        }
      }
      v += w * s2;
    }
  }
  val[k] = v;
  if (M.nz_cc[k] & 16) diag[M.col[k]] = v;  // bit 4: col == row (set by hom_setup)
}

void launch_macro_assemble(const MacroDev& M, const double* D, double* val, double* diag, cudaStream_t s) {
  if (M.dim == 1) k_macro_assemble<1><<<(M.nnz + 255) / 256, 256, 0, s>>>(M, D, val, diag);
  else if (M.dim == 2) k_macro_assemble<2><<<(M.nnz + 255) / 256, 256, 0, s>>>(M, D, val, diag);
  else k_macro_assemble<3><<<(M.nnz + 255) / 256, 256, 0, s>>>(M, D, val, diag);
}

// ---------------------------------------------------------------- RHS
// rhs_i = -R_i - sum_j K_ij x_D,j (free rows), 0 on Dirichlet rows;  Rfree_i = R_i (free) or 0.
template <int DIM>
__global__ void k_macro_rhs(MacroDev M, const double* __restrict__ val, const double* __restrict__ S,
                            double scale, double* __restrict__ rhs, double* __restrict__ Rfree) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M.ndof) return;
  if (M.dmask[i]) {
    if (rhs) rhs[i] = 0.0;
    if (Rfree) Rfree[i] = 0.0;
    return;
  }
  int n = i / DIM, c = i % DIM;
  double R = -M.load_factor * M.fbody[i];
  if (S) {
    for (int s = M.ninc_ptr[n]; s < M.ninc_ptr[n + 1]; ++s) {
      int E = M.ninc[s] >> 4, a = M.ninc[s] & 15;
      for (int q = 0; q < M.nq; ++q) {
        int t = E * M.nq + q;
        const double* g = M.grad + ((long)t * M.nen + a) * DIM;
        const double* Sq = S + (long)t * M.m;
        double v = 0.0;
        if (M.finite) {
          for (int J = 0; J < DIM; ++J) v += g[J] * Sq[c * DIM + J];
        } else {
          for (int k = 0; k < M.m; ++k) v += voigtB<DIM>(g, k, c) * Sq[k];
        }
        R += M.wdet[t] * v;
      }
    }
  }
  if (Rfree) Rfree[i] = R;
  if (rhs) {
    double lift = 0.0;
    if (val) {
      for (int k = M.rowptr[i]; k < M.rowptr[i + 1]; ++k) {
        int j = M.col[k];
        if (M.dmask[j]) lift += val[k] * (scale * M.dval[j]);
      }
    }
    rhs[i] = -R - lift;
  }
}

void launch_macro_rhs(const MacroDev& M, const double* val, const double* S, double scale, double* rhs,
                      double* Rfree, cudaStream_t s) {
  if (M.dim == 1) k_macro_rhs<1><<<(M.ndof + 255) / 256, 256, 0, s>>>(M, val, S, scale, rhs, Rfree);
  else if (M.dim == 2) k_macro_rhs<2><<<(M.ndof + 255) / 256, 256, 0, s>>>(M, val, S, scale, rhs, Rfree);
  else k_macro_rhs<3><<<(M.ndof + 255) / 256, 256, 0, s>>>(M, val, S, scale, rhs, Rfree);
}

// ---------------------------------------------------------------- reductions
constexpr int CG_THR = 1024;

__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double x = (lane < (int)(blockDim.x >> 5)) ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) red[32] = x;
  }
  __syncthreads();
  double r = red[32];
  __syncthreads();
  return r;
}

__device__ __forceinline__ void block_sum2(double& a, double& b, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
  }
  if (lane == 0) { red[warp] = a; red[40 + warp] = b; }
  __syncthreads();
  if (warp == 0) {
    int nw = blockDim.x >> 5;
    double x = lane < nw ? red[lane] : 0.0, y = lane < nw ? red[40 + lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      x += __shfl_down_sync(0xffffffffu, x, o);
      y += __shfl_down_sync(0xffffffffu, y, o);
    }
    if (lane == 0) { red[32] = x; red[33] = y; }
  }
  __syncthreads();
  a = red[32];
  b = red[33];
  __syncthreads();
}

__global__ void k_norm(const double* __restrict__ v, int n, double* out) {
  __shared__ double red[80];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += v[i] * v[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = sqrt(s);
}
void launch_norm(const double* v, int n, double* out, cudaStream_t s) { k_norm<<<1, CG_THR, 0, s>>>(v, n, out); }

// ---------------------------------------------------------------- K6/K7: PCG
// One persistent CTA: SpMV, dots and axpys of every iteration in one launch,
// no host round trip per iteration (K6/K7).
__global__ void __launch_bounds__(CG_THR) k_macro_cg(MacroDev M, const double* __restrict__ val,
                                                     const double* __restrict__ diag,
                                                     const double* __restrict__ b, double scale,
                                                     double rtol, int max_iter, double* __restrict__ xout,
                                                     double* __restrict__ work, CgState* st) {
  __shared__ double red[80];
  const int n = M.ndof, tid = threadIdx.x;
  double* x = work;
  double* r = work + n;
  double* p = work + 2 * (long)n;
  double* q = work + 3 * (long)n;
  double rz = 0.0, bb = 0.0;
  for (int i = tid; i < n; i += CG_THR) {
    double bi = M.dmask[i] ? 0.0 : b[i];
    double zi = M.dmask[i] ? 0.0 : bi / diag[i];
    x[i] = 0.0;
    r[i] = bi;
    p[i] = zi;
    rz += bi * zi;
    bb += bi * bi;
  }
  block_sum2(rz, bb, red);
  const double bnorm = sqrt(bb);
  int it = 0, status = 0;
  double rr = bb;
  if (bnorm > 0.0) {
    for (it = 1; it <= max_iter; ++it) {
      double pq = 0.0;
      for (int i = tid; i < n; i += CG_THR) {
        double s = 0.0;
        if (!M.dmask[i]) {
          for (int k = M.rowptr[i]; k < M.rowptr[i + 1]; ++k) s += val[k] * p[M.col[k]];
        }
        q[i] = s;
        pq += p[i] * s;
      }
      pq = block_sum(pq, red);
      if (!(pq > 0.0)) { status = 6; break; }
      const double alpha = rz / pq;
      double rzn = 0.0;
      rr = 0.0;
      for (int i = tid; i < n; i += CG_THR) {
        x[i] += alpha * p[i];
        double ri = r[i] - alpha * q[i];
        r[i] = ri;
        double zi = M.dmask[i] ? 0.0 : ri / diag[i];
        rr += ri * ri;
        rzn += ri * zi;
      }
      block_sum2(rr, rzn, red);
      if (sqrt(rr) <= rtol * bnorm) break;
      const double beta = rzn / rz;
      rz = rzn;
      for (int i = tid; i < n; i += CG_THR) {
        double zi = M.dmask[i] ? 0.0 : r[i] / diag[i];
        p[i] = zi + beta * p[i];
      }
      __syncthreads();
    }
    if (status == 0 && it > max_iter) { status = 5; it = max_iter; }
  }
  for (int i = tid; i < n; i += CG_THR) xout[i] = M.dmask[i] ? scale * M.dval[i] : x[i];
  if (tid == 0) {
    st->iterations = it;
    st->status = status;
    st->rel_residual = bnorm > 0.0 ? sqrt(rr) / bnorm : 0.0;
    st->rhs_norm = bnorm;
  }
}

void launch_macro_cg(const MacroDev& M, const double* val, const double* diag, const double* rhs,
                     double scale, double rtol, int max_iter, double* x, double* work, CgState* st,
                     cudaStream_t s) {
  k_macro_cg<<<1, CG_THR, 0, s>>>(M, val, diag, rhs, scale, rtol, max_iter, x, work, st);
}

__global__ void k_axpy(double* __restrict__ y, const double* __restrict__ x, double a, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] += a * x[i];
}
void launch_axpy(double* y, const double* x, double a, int n, cudaStream_t s) {
  k_axpy<<<(n + 255) / 256, 256, 0, s>>>(y, x, a, n);
}

// ---------------------------------------------------------------- K6/K7: cluster PCG
// One thread-block cluster (16 CTAs where the device allows it, else 8) runs the
// whole Jacobi-PCG in a single launch: CTA g owns a contiguous slice of rows and
// keeps that slice of the CSR matrix and of x, r, 1/diag, q, p in shared memory;
// p is published in global memory (L2) for the SpMV gathers of the other CTAs;
// dot products are reduced through DSMEM in a fixed order (bitwise deterministic,
// identical in every CTA), and cluster barriers (barrier.cluster, which also
// invalidates L1) separate the phases -- three per iteration, no host round trip.
constexpr int CGC_THR = 512;
constexpr int CGC_MAXG = 16;

__device__ __forceinline__ void cl_reduce2(cgx::cluster_group& cl, double* slots, double& a, double& b,
                                           double* wred) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
  }
  if (lane == 0) { wred[warp] = a; wred[32 + warp] = b; }
  __syncthreads();
  const int G = cl.num_blocks();
  if (threadIdx.x < G) {  // thread t publishes this CTA's partials into CTA t's slots
    double sa = 0.0, sb = 0.0;
    for (int w = 0; w < CGC_THR / 32; ++w) { sa += wred[w]; sb += wred[32 + w]; }
    double* remote = cl.map_shared_rank(slots, (int)threadIdx.x);
    remote[cl.block_rank()] = sa;
    remote[CGC_MAXG + cl.block_rank()] = sb;
  }
  cl.sync();
  a = 0.0;
  b = 0.0;
  for (int k = 0; k < G; ++k) { a += slots[k]; b += slots[CGC_MAXG + k]; }
}

__global__ void __launch_bounds__(CGC_THR) k_macro_cg_cluster(MacroDev M, const double* __restrict__ val,
                                                              const double* __restrict__ diag,
                                                              const double* __restrict__ b, double scale,
                                                              double rtol, int max_iter, double* __restrict__ xout,
                                                              double* __restrict__ pg, CgState* st,
                                                              int csr_in_smem) {
  cgx::cluster_group cl = cgx::this_cluster();
  const int G = cl.num_blocks(), g = cl.block_rank();
  const int n = M.ndof, tid = threadIdx.x;
  const int r0 = (int)((long)n * g / G), r1 = (int)((long)n * (g + 1) / G), nr = r1 - r0;
  extern __shared__ __align__(16) double sm[];
  double* slots = sm;                      // [2 buffers][2*CGC_MAXG]
  double* wred = sm + 4 * CGC_MAXG;        // [64]
  double* sx = wred + 64;
  double* sr = sx + nr;
  double* sdi = sr + nr;
  double* sq = sdi + nr;
  double* sp = sq + nr;
  double* sval = sp + nr;
  const int nz0 = M.rowptr[r0], nnz = M.rowptr[r1] - nz0;
  int* scol = reinterpret_cast<int*>(sval + (csr_in_smem ? nnz : 0));
  int* srow = scol + (csr_in_smem ? nnz : 0);
  if (csr_in_smem) {
    for (int k = tid; k < nnz; k += CGC_THR) { sval[k] = val[nz0 + k]; scol[k] = M.col[nz0 + k]; }
    for (int i = tid; i <= nr; i += CGC_THR) srow[i] = M.rowptr[r0 + i] - nz0;
  }
  double rz = 0.0, bb = 0.0;
  for (int i = tid; i < nr; i += CGC_THR) {
    int gi = r0 + i;
    bool d = M.dmask[gi];
    double bi = d ? 0.0 : b[gi];
    double di = d ? 0.0 : 1.0 / diag[gi];
    double zi = bi * di;
    sx[i] = 0.0; sr[i] = bi; sdi[i] = di; sp[i] = zi;
    pg[gi] = zi;
    rz += bi * zi;
    bb += bi * bi;
  }
  cl_reduce2(cl, slots + 2 * CGC_MAXG, rz, bb, wred);  // also publishes p
  const double bnorm = sqrt(bb);
  int it = 0, status = 0;
  double rr = bb;
  if (bnorm > 0.0) {
    for (it = 1; it <= max_iter; ++it) {
      double pq = 0.0, dummy = 0.0;
      for (int i = tid; i < nr; i += CGC_THR) {
        double s = 0.0;
        if (sdi[i] != 0.0) {
          if (csr_in_smem) {
            for (int k = srow[i]; k < srow[i + 1]; ++k) s += sval[k] * pg[scol[k]];
          } else {
            for (int k = M.rowptr[r0 + i]; k < M.rowptr[r0 + i + 1]; ++k) s += val[k] * pg[M.col[k]];
          }
        }
        sq[i] = s;
        pq += sp[i] * s;
      }
      cl_reduce2(cl, slots, pq, dummy, wred);
      if (!(pq > 0.0)) { status = 6; break; }
      const double alpha = rz / pq;
      double rzn = 0.0;
      rr = 0.0;
      for (int i = tid; i < nr; i += CGC_THR) {
        sx[i] += alpha * sp[i];
        double ri = sr[i] - alpha * sq[i];
        sr[i] = ri;
        rr += ri * ri;
        rzn += ri * ri * sdi[i];
      }
      cl_reduce2(cl, slots + 2 * CGC_MAXG, rr, rzn, wred);
      if (sqrt(rr) <= rtol * bnorm) break;
      const double beta = rzn / rz;
      rz = rzn;
      for (int i = tid; i < nr; i += CGC_THR) {
        double pi = sr[i] * sdi[i] + beta * sp[i];
        sp[i] = pi;
        pg[r0 + i] = pi;
      }
      cl.sync();  // p visible cluster-wide (release/acquire; L1 invalidated)
    }
    if (status == 0 && it > max_iter) { status = 5; it = max_iter; }
  }
  for (int i = tid; i < nr; i += CGC_THR) {
    int gi = r0 + i;
    xout[gi] = M.dmask[gi] ? scale * M.dval[gi] : sx[i];
  }
  if (g == 0 && tid == 0) {
    st->iterations = it;
    st->status = status;
    st->rel_residual = bnorm > 0.0 ? sqrt(rr) / bnorm : 0.0;
    st->rhs_norm = bnorm;
  }
  cl.sync();  // no CTA exits while others may still read its shared memory
}

// Returns false if no cluster configuration fits (caller falls back to one CTA).
bool launch_macro_cg_cluster(const MacroDev& M, int max_slice_nnz, const double* val, const double* diag,
                             const double* rhs, double scale, double rtol, int max_iter, double* x, double* p,
                             CgState* st, cudaStream_t s) {
  for (int G : {16, 8}) {
    int max_rows = (M.ndof + G - 1) / G + 1;
    size_t base = (size_t)(4 * CGC_MAXG + 64 + 5 * max_rows) * 8;
    size_t with_csr = base + (size_t)max_slice_nnz * 12 + (size_t)(max_rows + 1) * 4 + 64;
    int csr = with_csr <= 200 * 1024;
    size_t sm = csr ? with_csr : base;
    if (sm > 200 * 1024) continue;
    cudaFuncSetAttribute(k_macro_cg_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (G > 8) cudaFuncSetAttribute(k_macro_cg_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G, 1, 1);
    cfg.blockDim = dim3(CGC_THR, 1, 1);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, k_macro_cg_cluster, &cfg) != cudaSuccess || ncl < 1) {
      cudaGetLastError();
      continue;
    }
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_macro_cg_cluster, M, val, diag, rhs, scale, rtol, max_iter, x, p,
                                       st, csr);
    if (e == cudaSuccess) return true;
    cudaGetLastError();
  }
  return false;
}

// ---------------------------------------------------------------- K6/K7: cluster PCG, v2
// Chronopoulos-Gear PCG (one fused reduction + one vector broadcast per iteration instead
// of two reductions + a publish) with a node-block Jacobi preconditioner (the dim x dim
// diagonal block of every macro node, Dirichlet components removed).  One cluster of G CTAs;
// CTA g owns the rows of a contiguous node range, keeps that CSR slice and the slices of
// x, r, p, s, w and of the block inverse in shared memory, and ALSO a full copy of the
// preconditioned residual z: every CTA scatters its new slice of z into all G copies with
// DSMEM stores, so the SpMV gathers are shared-memory loads.  Two cluster barriers per
// iteration; every dot product is summed in a fixed order (bitwise deterministic).
//   loop: x += a p; r -= a s; z = M^-1 r; [z slices + (r.z, r.r) partials -> all CTAs; sync]
//         w = A z; [(z.w) partials -> all CTAs; sync]
//         b = g'/g; a = g'/(d - b g'/a); p = z + b p; s = w + b s

template <int CG2_THR>
__device__ __forceinline__ void cg2_publish(cgx::cluster_group& cl, double* slots, int nv, double* v, double* wred) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = 0; j < nv; ++j) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[j] += __shfl_down_sync(0xffffffffu, v[j], o);
    if (lane == 0) wred[j * 32 + warp] = v[j];
  }
  __syncthreads();
  const int G = cl.num_blocks();
  if ((int)threadIdx.x < G) {  // thread t writes this CTA's partials into CTA t's slots
    double* remote = cl.map_shared_rank(slots, (int)threadIdx.x);
    for (int j = 0; j < nv; ++j) {
      double a = 0.0;
      for (int w = 0; w < CG2_THR / 32; ++w) a += wred[j * 32 + w];
      remote[j * CGC_MAXG + cl.block_rank()] = a;
    }
  }
}
__device__ __forceinline__ double cg2_sum(const double* slots, int j, int G) {
  // fixed-order pairwise tree over the G partials (G = 8 or 16; unused slots of G = 8 skipped):
  // the same order in every CTA, 4 dependent adds instead of G
  const double* s = slots + j * CGC_MAXG;
  double t[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) t[k] = G > 8 ? s[2 * k] + s[2 * k + 1] : s[k];
#pragma unroll
  for (int k = 0; k < 4; ++k) t[k] = t[2 * k] + t[2 * k + 1];
  return (t[0] + t[1]) + (t[2] + t[3]);
}

// CC: two-level additive preconditioner z = B^-1 r + P A_c^-1 P^T r (coarse.cu).
// The restriction P^T r of the new residual r_{k+1} = r_k - alpha s_{k+1} is assembled from the
// partials of P^T r_k and P^T s_{k+1}, which every CTA publishes (one double2 per coarse DOF per
// destination) together with its (z.w) partial -- alpha is known only after that exchange, so
// no extra cluster barrier is needed.  Each CTA then forms A_c^-1 r_c on the coarse DOFs of
// the aggregates its rows touch (fp32 rows of the symmetric A_c^-1: a fixed SPD operator) and
// adds P z_c in the preconditioner pass.
template <bool WIN, int CG2_THR, bool CC>  // CG2_THR: 256, or 512 for long slices (more rows in flight)
__global__ void __launch_bounds__(CG2_THR) k_macro_cg_cluster2(MacroDev M, const double* __restrict__ val,
                                                               const double* __restrict__ b, double scale,
                                                               double rtol, int max_iter, double* __restrict__ xout,
                                                               CgState* st, int js) {
  cgx::cluster_group cl = cgx::this_cluster();
  const int G = cl.num_blocks(), g = cl.block_rank();
  const int n = M.ndof, dim = M.dim, tid = threadIdx.x;
  const int nd0 = (int)((long)M.n_nodes * g / G), nd1 = (int)((long)M.n_nodes * (g + 1) / G);
  const int r0 = nd0 * dim, r1 = nd1 * dim, nr = r1 - r0;
  extern __shared__ __align__(16) double sm[];
  double* slotsA = sm;                       // [3][CGC_MAXG]: (r.z, r.r)
  double* slotsB = slotsA + 3 * CGC_MAXG;    // [3][CGC_MAXG]: (z.w)
  double* wred = slotsB + 3 * CGC_MAXG;      // [3][32]
  // CC: this CTA's (P^T r, P^T s) partials on its local aggregates, [nla_max][NM] (same offset
  // in every CTA: the other CTAs read them through DSMEM)
  const int gi = G == 16 ? 0 : 1;
  const int NM = CC ? M.cc.nm : 1, nc = CC ? M.cc.nc : 1, KC = CC ? M.cc.kmax[gi] : 0;
  const int la0 = CC ? M.cc.lptr[gi][g] : 0, nla = CC ? M.cc.lptr[gi][g + 1] - la0 : 0;
  double2* lpart = reinterpret_cast<double2*>(wred + 96);
  // z: a full copy (WIN = false) or this CTA's column window [wlo, whi) (WIN = true; indices into zf
  // are then offset by wlo, the CSR columns in shared memory pre-offset)
  const int* wtab = M.cg_win + (G == 16 ? 0 : 2 * CGC_MAXG);
  const int wlo = WIN ? __ldg(wtab + 2 * g) : 0;
  const int zlen = WIN ? M.cg_wmax[G == 16 ? 0 : 1] : n;
  double* zf = reinterpret_cast<double*>(lpart + (CC ? M.cc.nla_max[gi] * NM : 0));  // [zlen]
  double* x = zf + zlen;
  double* r = x + nr;
  double* p = r + nr;
  double* sv = p + nr;
  double* w = sv + nr;
  double* mi = w + nr;                       // [nr][dim] block-Jacobi inverse rows
  // the CSR slice as column-major ELL (slot j of local row i at j * nr + i: consecutive threads read
  // consecutive words), padded to the longest row with zero values pointing at the row's own z.
  // Slots j < js live in shared memory, the rest (large meshes) in global memory at [j][n], read
  // back from L2 every SpMV
  const int nz0 = M.rowptr[r0], ew = M.cg_ellw, nell = js * nr;
  double* sval = mi + nr * dim;
  int* scol = reinterpret_cast<int*>(sval + nell);
  int* srow = scol + nell;
  // CC, this CTA only: zc [nla * NM], rc [nc], srel [nr] (coordinate i % dim of local node
  // i / dim, scaled, relative to its aggregate), sainv [nc][nlp] fp32 columns of A_c^-1 on this
  // CTA's coarse DOFs (nlp = 8 mod 16: conflict-free), sq [nr] local aggregate of each row (-1:
  // Dirichlet row, zero row of P), the local aggregates' node lists and ids, ntch [nagg]
  const int nl = nla * NM, nlp = CC ? (nl + 7) / 16 * 16 + 8 : 0;
  double* zc = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(srow + nr + 1) + 15) & ~uintptr_t(15));
  float* rcf = reinterpret_cast<float*>(zc + nl);  // [nc] (fp32 coarse solve)
  double* cpart = zc + nl + (CC ? (nc + 1) / 2 : 0);  // [2 nl][CC_NCH] restriction chunk sums
  double* srel = cpart + (CC ? 2 * nl * CC_NCH : 0);
  float* sainv = reinterpret_cast<float*>(srel + (CC ? nr : 0));
  int* sq = reinterpret_cast<int*>(sainv + (size_t)nlp * nc);
  int* slnp = sq + (CC ? nr : 0);   // [nla + 1]
  int* sln = slnp + nla + 1;        // [nr / dim]
  int* sntch = sln + (CC ? nr / dim : 0);  // [nagg]
  int* stch = sntch + (CC ? M.cc.nagg : 0);  // [nagg][KC]
  constexpr int NWARP = CG2_THR / 32;
  const int lane = tid & 31, warp = tid >> 5;
  double* gval = M.cg_gval + r0;
  int* gcol = M.cg_gcol + r0;
  for (int i = tid; i <= nr; i += CG2_THR) srow[i] = M.rowptr[r0 + i] - nz0;
  __syncthreads();
  for (int e = tid; e < ew * nr; e += CG2_THR) {
    const int j = e / nr, i = e - j * nr, k = srow[i] + j;
    const bool in = k < srow[i + 1];
    const double vv = in ? val[nz0 + k] : 0.0;
    const int cc = in ? M.col[nz0 + k] - wlo : r0 + i - wlo;
    if (j < js) {
      sval[e] = vv;
      scol[e] = cc;
    } else {
      gval[(size_t)j * n + i] = vv;
      gcol[(size_t)j * n + i] = cc;
    }
  }
  __syncthreads();  // also orders this CTA's global ELL writes before its own reads
  // remote copies of z: this CTA's slice in every CTA of the cluster (addresses mapped once);
  // WIN: only the CTAs whose window meets these rows, local rows [dlo, dhi) of each
  double* zrem[WIN ? CG_WDEST + 1 : CGC_MAXG];
  int dlo[WIN ? CG_WDEST + 1 : 1], dhi[WIN ? CG_WDEST + 1 : 1];
  int ndst = 0;
  if (WIN) {
#pragma unroll
    for (int q = 0; q < CG_WDEST + 1; ++q) { zrem[q] = nullptr; dlo[q] = 0; dhi[q] = 0; }
    for (int t = 0; t < G; ++t) {
      const int lo = max(r0, __ldg(wtab + 2 * t)), hi = min(r1, __ldg(wtab + 2 * t + 1));
      if (lo >= hi || ndst > CG_WDEST) continue;
#pragma unroll
      for (int q = 0; q < CG_WDEST + 1; ++q)
        if (q == ndst) {
          zrem[q] = cl.map_shared_rank(zf, t) + (r0 - __ldg(wtab + 2 * t));
          dlo[q] = lo - r0;
          dhi[q] = hi - r0;
        }
      ++ndst;
    }
  } else {
#pragma unroll
    for (int t = 0; t < CGC_MAXG; ++t) zrem[t] = t < G ? cl.map_shared_rank(zf, t) + r0 : nullptr;
  }
  auto put_z = [&](int i, double z) {  // local row i of this CTA -> every copy that reads it
    if (WIN) {
#pragma unroll
      for (int q = 0; q < CG_WDEST + 1; ++q)
        if (q < ndst && i >= dlo[q] && i < dhi[q]) zrem[q][i] = z;
    } else {
#pragma unroll
      for (int t = 0; t < CGC_MAXG; ++t)
        if (t < G) zrem[t][i] = z;
    }
  };
  const int zown = r0 - wlo;  // zf index of local row 0
  // node-block Jacobi: invert the free part of each dim x dim diagonal block
  for (int nd = nd0 + tid; nd < nd1; nd += CG2_THR) {
    double a[3][3] = {}, inv[3][3] = {};
    bool fr[3] = {false, false, false};
    for (int ci = 0; ci < dim; ++ci) {
      const int row = nd * dim + ci;
      fr[ci] = !M.dmask[row];
      const int li = row - r0, len = srow[li + 1] - srow[li];
      for (int j = 0; j < len; ++j) {
        const int cc = (j < js ? scol[j * nr + li] : gcol[(size_t)j * n + li]) + wlo - nd * dim;
        if (cc >= 0 && cc < dim) a[ci][cc] = j < js ? sval[j * nr + li] : gval[(size_t)j * n + li];
      }
    }
    for (int ci = 0; ci < 3; ++ci)
      for (int cj = 0; cj < 3; ++cj)
        if (ci >= dim || cj >= dim || !fr[ci] || !fr[cj]) a[ci][cj] = (ci == cj) ? 1.0 : 0.0;
    const double det = a[0][0] * (a[1][1] * a[2][2] - a[1][2] * a[2][1]) -
                       a[0][1] * (a[1][0] * a[2][2] - a[1][2] * a[2][0]) +
                       a[0][2] * (a[1][0] * a[2][1] - a[1][1] * a[2][0]);
    inv[0][0] = (a[1][1] * a[2][2] - a[1][2] * a[2][1]) / det;
    inv[0][1] = (a[0][2] * a[2][1] - a[0][1] * a[2][2]) / det;
    inv[0][2] = (a[0][1] * a[1][2] - a[0][2] * a[1][1]) / det;
    inv[1][0] = (a[1][2] * a[2][0] - a[1][0] * a[2][2]) / det;
    inv[1][1] = (a[0][0] * a[2][2] - a[0][2] * a[2][0]) / det;
    inv[1][2] = (a[0][2] * a[1][0] - a[0][0] * a[1][2]) / det;
    inv[2][0] = (a[1][0] * a[2][1] - a[1][1] * a[2][0]) / det;
    inv[2][1] = (a[0][1] * a[2][0] - a[0][0] * a[2][1]) / det;
    inv[2][2] = (a[0][0] * a[1][1] - a[0][1] * a[1][0]) / det;
    for (int ci = 0; ci < dim; ++ci)
      for (int cj = 0; cj < dim; ++cj)
        mi[((nd - nd0) * dim + ci) * dim + cj] = (fr[ci] && fr[cj]) ? inv[ci][cj] : 0.0;
  }
  __syncthreads();  // the block-Jacobi setup has read the diagonal blocks
  for (int i = tid; i < nr; i += CG2_THR) {
    const int gi = r0 + i;
    x[i] = 0.0;
    r[i] = M.dmask[gi] ? 0.0 : b[gi];
    if (M.dmask[gi])  // Dirichlet row: w_i = 0 without a mask test in the SpMV
      for (int j = 0; j < ew; ++j) {
        if (j < js) sval[j * nr + i] = 0.0;
        else gval[(size_t)j * n + i] = 0.0;
      }
  }
  if (CC) {
    const int e00 = M.cc.lnptr[gi][la0];
    for (int i = tid; i < nr; i += CG2_THR) {
      srel[i] = M.cc.rel[(size_t)r0 + i];
      sv[i] = 0.0;
    }
    for (int q = tid; q <= nla; q += CG2_THR) slnp[q] = M.cc.lnptr[gi][la0 + q] - e00;
    for (int a = tid; a < M.cc.nagg; a += CG2_THR) sntch[a] = M.cc.ntch[gi][a];
    for (int t = tid; t < M.cc.nagg * KC; t += CG2_THR) stch[t] = M.cc.tch[gi][t];
    for (int q = warp; q < nla; q += NWARP)
      for (int e = M.cc.lnptr[gi][la0 + q] + lane; e < M.cc.lnptr[gi][la0 + q + 1]; e += 32) {
        const int l = M.cc.lnode[gi][e];
        sln[e - e00] = l;
        for (int c = 0; c < dim; ++c) sq[l * dim + c] = M.dmask[r0 + l * dim + c] ? -1 : q;
      }
    for (int t = tid; t < nl * nc; t += CG2_THR) {
      const int cc = t / nl, rw = t - cc * nl, q = rw / NM, m = rw - q * NM;
      sainv[cc * nlp + rw] = (float)M.cc.Ainv[(size_t)(M.cc.lagg[gi][la0 + q] * NM + m) * nc + cc];
    }
  }
  cl.sync();  // every CTA of the cluster is running before the first DSMEM store
  // CC: (P^T r, P^T s) over this CTA's rows of each local aggregate -> lpart
  auto cc_restrict = [&](bool with_s) {
    // thread per (local coarse DOF t = q * NM + m, vector, chunk of the aggregate's local node
    // list): serial sums in list order, then the CC_NCH chunk sums in chunk order (fixed order)
    for (int u = tid; u < 2 * nl * CC_NCH; u += CG2_THR) {
      const int ch = u % CC_NCH, tv = u / CC_NCH, t = tv >> 1, q = t / NM, m = t - q * NM;
      const double* vec = (tv & 1) ? sv : r;
      const int e0 = slnp[q], L = slnp[q + 1] - e0;
      double acc = 0.0;
      if (!(tv & 1) || with_s)
        for (int e = e0 + L * ch / CC_NCH; e < e0 + L * (ch + 1) / CC_NCH; ++e) {
          const int l = sln[e];
          if (m < dim) {
            acc += vec[l * dim + m];
          } else {
            const double* d = srel + l * dim;
#pragma unroll
            for (int c = 0; c < 3; ++c)
              if (c < dim) acc += cc_coef(dim, c, m, d) * vec[l * dim + c];
          }
        }
      cpart[u] = acc;
    }
    __syncthreads();
    for (int tv = tid; tv < 2 * nl; tv += CG2_THR) {
      double acc = 0.0;
#pragma unroll
      for (int ch = 0; ch < CC_NCH; ++ch) acc += cpart[tv * CC_NCH + ch];
      reinterpret_cast<double*>(lpart)[tv] = acc;
    }
  };
  // CC: r_c = sum_k (P^T r)_k - alpha sum_k (P^T s)_k (thread per coarse DOF), then
  // zc = A_c^-1 r_c on this CTA's coarse DOFs: lane = (row t0 + lane % 8, column group lane / 8),
  // columns c = group + 4 u, two butterfly steps (fixed order)
  auto cc_rc = [&](double alpha) {
    for (int c = tid; c < nc; c += CG2_THR) {
      const int a = c / NM, m = c - a * NM, nt = sntch[a];
      double sr = 0.0, ss = 0.0;
      double2 t4[4];
#pragma unroll
      for (int k = 0; k < 4; ++k)  // DSMEM loads from the CTAs touching aggregate a, in flight together
        if (k < nt) {
          const int tk = stch[a * KC + k];
          t4[k] = cl.map_shared_rank(lpart, tk >> 16)[(tk & 0xffff) * NM + m];
        }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < nt) {
          sr += t4[k].x;
          ss += t4[k].y;
        }
      for (int k = 4; k < nt; ++k) {
        const int tk = stch[a * KC + k];
        const double2 t = cl.map_shared_rank(lpart, tk >> 16)[(tk & 0xffff) * NM + m];
        sr += t.x;
        ss += t.y;
      }
      rcf[c] = (float)(sr - alpha * ss);
    }
    __syncthreads();
  };
  auto cc_mv = [&]() {
    for (int t0 = warp * 8; t0 < nl; t0 += NWARP * 8) {
      const int t = t0 + (lane & 7), cg = lane >> 3;
      float a0 = 0.0f, a1 = 0.0f;
      if (t < nl) {
        int c = cg;
#pragma unroll 4
        for (; c + 4 < nc; c += 8) {
          a0 = fmaf(sainv[c * nlp + t], rcf[c], a0);
          a1 = fmaf(sainv[(c + 4) * nlp + t], rcf[c + 4], a1);
        }
        if (c < nc) a0 = fmaf(sainv[c * nlp + t], rcf[c], a0);
      }
      float a = a0 + a1;
      a += __shfl_xor_sync(0xffffffffu, a, 8);
      a += __shfl_xor_sync(0xffffffffu, a, 16);
      if (cg == 0 && t < nl) zc[t] = (double)a;
    }
    __syncthreads();
  };
  // CC: (P z_c)_i for local row i
  auto cc_prolong = [&](int i) {
    const int q = sq[i];
    if (q < 0) return 0.0;
    const int l = i / dim, c = i - l * dim;
    double z = 0.0;
#pragma unroll
    for (int m = 0; m < 6; ++m)
      if (m < NM) z += cc_coef(dim, c, m, srel + l * dim) * zc[q * NM + m];
    return z;
  };
  if (CC) {  // r_c of r_0 = b: one extra exchange before the first preconditioner application
    cc_restrict(false);
    cl.sync();
    cc_rc(0.0);
    cc_mv();
  }

  // z = M^-1 r on the local rows, scattered into every CTA's copy; returns (r.z, r.r) partials
  auto precond_publish = [&](double* part) {
    double rz = 0.0, rr = 0.0;
    for (int i = tid; i < nr; i += CG2_THR) {
      const int nl = i / dim, ci = i % dim;
      double z = 0.0;
      for (int cj = 0; cj < dim; ++cj) z += mi[i * dim + cj] * r[nl * dim + cj];
      if (CC) z += cc_prolong(i);
      rz += r[i] * z;
      rr += r[i] * r[i];
      put_z(i, z);
      (void)ci;
    }
    part[0] = rz;
    part[1] = rr;
  };
  // w = A z (local rows, free DOFs only); returns the (z.w) partial
  auto spmv = [&](double beta_s) {  // CC: also s = w + beta_s s (needed before the exchange)
    double zw = 0.0;
    for (int i = tid; i < nr; i += CG2_THR) {
      double s0 = 0.0, s1 = 0.0;
      {  // Dirichlet rows have zero values (set up above)
        const double* vv = sval + i;
        const int* cc = scol + i;
        int j = 0;
        for (; j + 1 < js; j += 2) {  // js is even unless js == ew
          s0 += vv[j * nr] * zf[cc[j * nr]];
          s1 += vv[(j + 1) * nr] * zf[cc[(j + 1) * nr]];
        }
        if (j < js) {
          s0 += vv[j * nr] * zf[cc[j * nr]];
        } else if (j < ew) {  // spilled slots, from L2
          const double* gv = gval + i;
          const int* gc = gcol + i;
          for (; j + 1 < ew; j += 2) {
            const double v0 = __ldcg(gv + (size_t)j * n), v1 = __ldcg(gv + (size_t)(j + 1) * n);
            const int c0 = __ldcg(gc + (size_t)j * n), c1 = __ldcg(gc + (size_t)(j + 1) * n);
            s0 += v0 * zf[c0];
            s1 += v1 * zf[c1];
          }
          if (j < ew) s0 += __ldcg(gv + (size_t)j * n) * zf[__ldcg(gc + (size_t)j * n)];
        }
      }
      const double wi = s0 + s1;
      w[i] = wi;
      if (CC) sv[i] = wi + beta_s * sv[i];
      zw += zf[zown + i] * wi;
    }
    return zw;
  };

  double v[3];
  precond_publish(v);
  cg2_publish<CG2_THR>(cl, slotsA, 2, v, wred);
  cl.sync();
  double gam = cg2_sum(slotsA, 0, G), rr = cg2_sum(slotsA, 1, G);
  const double bnorm = sqrt(rr);
  int it = 0, status = 0;
  if (bnorm > 0.0) {
    v[0] = spmv(0.0);
    cg2_publish<CG2_THR>(cl, slotsB, 1, v, wred);  // its CTA barrier also completes r and s
    if (CC) cc_restrict(true);
    cl.sync();
    double del = cg2_sum(slotsB, 0, G);
    if (!(del > 0.0)) status = 6;
    double alpha = gam / del;
    for (int i = tid; i < nr; i += CG2_THR) { p[i] = zf[zown + i]; sv[i] = w[i]; }
    // 2-D: the direction update of the previous iteration, the x / r update and z = M^-1 r in one
    // pass -- threads i and i^1 hold the two rows of a node (node-aligned slices), the 2x2 block
    // preconditioner takes the sibling residual by a shuffle: no CTA barrier (same arithmetic)
    double beta = 0.0;
    // OVL (256-thread CTAs): the direction update p = z + beta p, s = w + beta s runs between the
    // arrive and the wait of the (z.w) cluster barrier; the 512-thread variant (long, L2-spilled
    // slices) measured faster with it fused into the x / r pass.  Same arithmetic either way.
    constexpr bool OVL = CG2_THR == 256;
    auto fused2 = [&](bool first, double* part) {
      double rz = 0.0, rr2 = 0.0;
      for (int base = 0; base < nr; base += CG2_THR) {
        const int i = base + tid;
        const bool act = i < nr;
        double ri = 0.0;
        if (act) {
          double pi = p[i], si = sv[i];
          if (!OVL && !first) {
            pi = zf[zown + i] + beta * pi;
            p[i] = pi;
            if (!CC) {
              si = w[i] + beta * si;
              sv[i] = si;
            }
          }
          x[i] += alpha * pi;
          ri = r[i] - alpha * si;
          r[i] = ri;
        }
        const double rsib = __shfl_xor_sync(0xffffffffu, ri, 1);
        if (act) {
          const double re = (i & 1) ? rsib : ri, ro = (i & 1) ? ri : rsib;
          double z = 0.0;
          z += mi[i * 2] * re;
          z += mi[i * 2 + 1] * ro;
          if (CC) {
            const int q = sq[i];
            if (q >= 0) {
              const int c = i & 1;
              z += zc[q * 3 + c] + (c == 0 ? -srel[i + 1] : srel[i - 1]) * zc[q * 3 + 2];
            }
          }
          rz += ri * z;
          rr2 += ri * ri;
          put_z(i, z);
        }
      }
      part[0] = rz;
      part[1] = rr2;
    };
    long long tprev = clock64();
    auto mark = [&](int k) {  // HOM_CG_PROF phase timing (thread 0 of every CTA)
      if (M.cg_prof && tid == 0) {
        const long long t = clock64();
        M.cg_prof[g * 16 + k] += (unsigned long long)(t - tprev);
        tprev = t;
      }
    };
    for (it = 1; it <= max_iter && status == 0; ++it) {
      mark(0);
      if (CC) {
        cc_rc(alpha);
        mark(11);
        cc_mv();
      }
      mark(1);
      if (dim == 2) {
        fused2(it == 1, v);
      } else {
        for (int i = tid; i < nr; i += CG2_THR) {
          x[i] += alpha * p[i];
          r[i] -= alpha * sv[i];
        }
        __syncthreads();  // r complete before the block preconditioner mixes components
        precond_publish(v);
      }
      mark(2);
      cg2_publish<CG2_THR>(cl, slotsA, 2, v, wred);
      mark(3);
      cl.sync();
      mark(4);
      const double gn = cg2_sum(slotsA, 0, G);
      rr = cg2_sum(slotsA, 1, G);
      if (sqrt(rr) <= rtol * bnorm) break;
      beta = gn / gam;
      v[0] = spmv(beta);
      mark(5);
      cg2_publish<CG2_THR>(cl, slotsB, 1, v, wred);  // its CTA barrier also completes r and s
      mark(6);
      if (CC) cc_restrict(true);
      mark(7);
      cl.barrier_arrive();
      mark(8);
      // the direction updates need beta (known) and local rows only: they run while the cluster
      // barrier of the (z.w) exchange completes
      if (OVL || dim != 2)
        for (int i = tid; i < nr; i += CG2_THR) {
          p[i] = zf[zown + i] + beta * p[i];
          if (!CC) sv[i] = w[i] + beta * sv[i];
        }
      mark(9);
      cl.barrier_wait();
      mark(10);
      del = cg2_sum(slotsB, 0, G);
      const double den = del - beta * gn / alpha;
      if (!(den > 0.0)) { status = 6; break; }
      alpha = gn / den;
      gam = gn;
    }
    if (status == 0 && it > max_iter) { status = 5; it = max_iter; }
  }
  for (int i = tid; i < nr; i += CG2_THR) {
    const int gi = r0 + i;
    xout[gi] = M.dmask[gi] ? scale * M.dval[gi] : x[i];
  }
  if (g == 0 && tid == 0) {
    st->iterations = it;
    st->status = status;
    st->rel_residual = bnorm > 0.0 ? sqrt(rr) / bnorm : 0.0;
    st->rhs_norm = bnorm;
  }
  cl.sync();  // no CTA exits while others may still write its shared memory
}

void cg2_windows(const MacroDev& M, const int* host_rowptr, const int* host_col, int G, int* win, int* wmax,
                 int* wok) {
  *wmax = 0;
  for (int g = 0; g < G; ++g) {  // node-aligned partition, as in k_macro_cg_cluster2
    const int r0 = (int)((long)M.n_nodes * g / G) * M.dim, r1 = (int)((long)M.n_nodes * (g + 1) / G) * M.dim;
    int lo = r0, hi = r1;
    for (int k = host_rowptr[r0]; k < host_rowptr[r1]; ++k) {
      lo = std::min(lo, host_col[k]);
      hi = std::max(hi, host_col[k] + 1);
    }
    win[2 * g] = lo;
    win[2 * g + 1] = hi;
    *wmax = std::max(*wmax, hi - lo);
  }
  *wok = 1;
  for (int g = 0; g < G; ++g) {  // windows (other than its own) that CTA g's rows reach
    const int r0 = (int)((long)M.n_nodes * g / G) * M.dim, r1 = (int)((long)M.n_nodes * (g + 1) / G) * M.dim;
    int nd = 0;
    for (int t = 0; t < G; ++t)
      if (t != g && std::max(r0, win[2 * t]) < std::min(r1, win[2 * t + 1])) ++nd;
    if (nd > CG_WDEST) *wok = 0;
  }
}

void cg2_slice_sizes(const MacroDev& M, const int* host_rowptr, int G, int* max_nr, int* max_nnz) {
  *max_nr = *max_nnz = 0;
  for (int g = 0; g < G; ++g) {  // node-aligned partition, as in k_macro_cg_cluster2
    const int nd0 = (int)((long)M.n_nodes * g / G), nd1 = (int)((long)M.n_nodes * (g + 1) / G);
    *max_nr = std::max(*max_nr, (nd1 - nd0) * M.dim);
    *max_nnz = std::max(*max_nnz, (nd1 - nd0) * M.dim * M.cg_ellw);  // ELL slice (k_macro_cg_cluster2)
  }
}

bool launch_macro_cg_cluster2(const MacroDev& M, const int (*slice)[2], const double* val, const double* rhs,
                              double scale, double rtol, int max_iter, double* x, CgState* st, cudaStream_t s,
                              int* extra_launches) {
  if (extra_launches) *extra_launches = 0;
  static const int force_G = [] {
    const char* e = getenv("HOM_CG_CLUSTER");  // experiment knob: 8 or 16
    return e ? atoi(e) : 0;
  }();
  static const int prefer_full = [] {
    const char* e = getenv("HOM_CG_FULLZ");  // experiment knob: 1 = try the full z copy first
    return e ? atoi(e) : 0;
  }();
  // preference: the two-level preconditioner, the whole ELL slice in shared memory, z windows
  // (fewer DSMEM stores), 16 CTAs
  bool cc_ready = false;
  for (int c = 0; c < 16; ++c) {
      const int use_cc = !(c >> 3), spill = (c >> 2) & 1, gi = c & 1, win = ((c >> 1) & 1) ^ (prefer_full ? 0 : 1);
      const int G = gi == 0 ? 16 : 8;
      if (use_cc && M.cc.nc <= 0) continue;
      if (force_G && G != force_G) continue;
      if (win && !M.cg_wok[gi]) continue;
      const int max_nr = slice[gi][0];
      const int zlen = win ? M.cg_wmax[gi] : M.ndof;
      size_t base = (size_t)(6 * CGC_MAXG + 96 + zlen + 5 * max_nr + max_nr * M.dim) * 8 +
                    (size_t)(max_nr + 1) * 4 + 64;
      if (use_cc) {  // k_macro_cg_cluster2's CC arrays
        const int nla = M.cc.nla_max[gi], nl = nla * M.cc.nm, nlp = (nl + 7) / 16 * 16 + 8;
        base += (size_t)nl * 16 + 16 + (size_t)(nl + M.cc.nc + max_nr + 2 * nl * CC_NCH) * 8 + (size_t)nlp * M.cc.nc * 4 +
                (size_t)(max_nr + 1 + nla + max_nr / M.dim + M.cc.nagg * (1 + M.cc.kmax[gi])) * 4;
      }
      const size_t cap = 227 * 1024;  // the sm_100 per-CTA opt-in maximum
      if (base > cap) continue;
      int js = (int)std::min<size_t>(M.cg_ellw, (cap - base) / ((size_t)max_nr * 12));
      if (js < M.cg_ellw) {
        if (!spill) continue;
        js &= ~1;  // may be 0: the whole ELL slice from L2
      } else if (spill) {
        continue;  // already tried without
      }
      const size_t sm = base + (size_t)max_nr * js * 12;
      const bool wide = max_nr > 768;
      decltype(&k_macro_cg_cluster2<true, 256, true>) k;
      if (use_cc)
        k = win ? (wide ? k_macro_cg_cluster2<true, 512, true> : k_macro_cg_cluster2<true, 256, true>)
                : (wide ? k_macro_cg_cluster2<false, 512, true> : k_macro_cg_cluster2<false, 256, true>);
      else
        k = win ? (wide ? k_macro_cg_cluster2<true, 512, false> : k_macro_cg_cluster2<true, 256, false>)
                : (wide ? k_macro_cg_cluster2<false, 512, false> : k_macro_cg_cluster2<false, 256, false>);
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (G > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(G, 1, 1);
      cfg.blockDim = dim3(wide ? 512 : 256, 1, 1);
      cfg.dynamicSmemBytes = sm;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = G;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, k, &cfg) != cudaSuccess || ncl < 1) {
        cudaGetLastError();
        continue;
      }
      if (use_cc && !cc_ready) {  // A_c and its inverse for these values, same stream
        if (!launch_coarse_setup(M, val, s)) {
          cudaGetLastError();
          continue;
        }
        cc_ready = true;
        if (extra_launches) *extra_launches = 2;  // k_coarse_assemble, k_coarse_invert
      }
      if (getenv("HOM_CG_VERBOSE"))
        fprintf(stderr, "cg2: cc %d G %d win %d wide %d js %d/%d smem %zu\n", use_cc, G, win, (int)wide, js, M.cg_ellw, sm);
      cudaError_t e = cudaLaunchKernelEx(&cfg, k, M, val, rhs, scale, rtol, max_iter, x, st, js);
      if (e == cudaSuccess) return true;
      cudaGetLastError();
    }
  return false;
}

// ---------------------------------------------------------------- persistent grid-wide PCG
// Meshes beyond one cluster (e.g. the config-3 macro mesh at N = 8, nel 181, 66k DOFs): one
// cooperative launch, one CTA per SM, the same Chronopoulos-Gear iteration and node-block Jacobi
// preconditioner as k_macro_cg_cluster2.  Each CTA owns a node range: its CSR slice as column-major
// ELL (shared memory, trailing slots in the global [slot][ndof] spill) and its x, r, p, s, w and
// block inverses in shared memory; z goes to a global array (L2) that the SpMV gathers read with
// ld.global.cg after the grid barrier.  Two grid barriers per iteration; the dot products are
// per-CTA partials in global memory summed by every CTA in CTA order (bitwise deterministic).
constexpr int CGG_THR = 512;
__device__ __forceinline__ double cgg_sum(const double* part, int G, int j, double* sred) {
  // every thread returns sum_g part[g * 4 + j] in g order (warp 0 sums, broadcast through sred)
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    double a = 0.0;
    for (int g = lane; g < G; g += 32) a += __ldcg(part + g * 4 + j);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) sred[j] = a;
  }
  __syncthreads();
  const double v = sred[j];
  return v;
}
template <bool CC>  // CC: the two-level preconditioner of k_macro_cg_cluster2, partials through L2
__global__ void __launch_bounds__(CGG_THR) k_macro_cg_grid(MacroDev M, const double* __restrict__ val,
                                                           const double* __restrict__ b, double scale, double rtol,
                                                           int max_iter, double* __restrict__ xout, CgState* st,
                                                           double* __restrict__ zg, double* __restrict__ part, int js) {
  cgx::grid_group grid = cgx::this_grid();
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = M.ndof, dim = M.dim;
  const int nd0 = (int)((long)M.n_nodes * g / G), nd1 = (int)((long)M.n_nodes * (g + 1) / G);
  const int r0 = nd0 * dim, nr = (nd1 - nd0) * dim;
  extern __shared__ __align__(16) double sm[];
  double* sred = sm;              // [8]
  double* wred = sred + 8;        // [3][32]
  double* x = wred + 96;
  double* r = x + nr;
  double* p = r + nr;
  double* sv = p + nr;
  double* w = sv + nr;
  double* zl = w + nr;
  double* mi = zl + nr;           // [nr][dim]
  const int nz0 = M.rowptr[r0], ew = M.cg_ellw, nell = js * nr;
  double* sval = mi + nr * dim;
  int* scol = reinterpret_cast<int*>(sval + nell);
  int* srow = scol + nell;
  double* gval = M.cg_gval + r0;
  int* gcol = M.cg_gcol + r0;
  // CC: zc [nl], rcf [nc] fp32, cpart [2 nl][CC_NCH], srel [nr], sainv [nc][nlp] fp32,
  // sq [nr], slnp [nla + 1], sln [nr / dim], sntch [nagg], stch [nagg][KC]
  constexpr int NWARP = CGG_THR / 32;
  const int NM = CC ? M.cc.nm : 1, nc = CC ? M.cc.nc : 1, KC = CC ? M.cc.kmax_g : 0;
  const int la0 = CC ? M.cc.lptr_g[g] : 0, nla = CC ? M.cc.lptr_g[g + 1] - la0 : 0;
  const int nl = nla * NM, nlp = CC ? (nl + 7) / 16 * 16 + 8 : 0, nlm = CC ? M.cc.nla_max_g * NM : 0;
  double* zc = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(srow + nr + 1) + 15) & ~uintptr_t(15));
  float* rcf = reinterpret_cast<float*>(zc + nl);
  double* cpart = zc + nl + (CC ? (nc + 1) / 2 : 0);
  double* srel = cpart + (CC ? 2 * nl * CC_NCH : 0);
  float* sainv = reinterpret_cast<float*>(srel + (CC ? nr : 0));
  int* sq = reinterpret_cast<int*>(sainv + (size_t)nlp * nc);
  int* slnp = sq + (CC ? nr : 0);
  int* sln = slnp + (CC ? nla + 1 : 0);
  int* sntch = sln + (CC ? nr / dim : 0);
  int* stch = sntch + (CC ? M.cc.nagg : 0);
  double2* gpart = CC ? M.cc.gpart : nullptr;
  for (int i = tid; i <= nr; i += CGG_THR) srow[i] = M.rowptr[r0 + i] - nz0;
  __syncthreads();
  for (int e = tid; e < ew * nr; e += CGG_THR) {
    const int j = e / nr, i = e - j * nr, k = srow[i] + j;
    const bool in = k < srow[i + 1];
    const double vv = in ? val[nz0 + k] : 0.0;
    const int cc = in ? M.col[nz0 + k] : r0 + i;  // padding points at the row's own z
    if (j < js) {
      sval[e] = vv;
      scol[e] = cc;
    } else {
      gval[(size_t)j * n + i] = vv;
      gcol[(size_t)j * n + i] = cc;
    }
  }
  __syncthreads();
  // node-block Jacobi (as k_macro_cg_cluster2)
  for (int nd = nd0 + tid; nd < nd1; nd += CGG_THR) {
    double a[3][3] = {}, inv[3][3] = {};
    bool fr[3] = {false, false, false};
    for (int ci = 0; ci < dim; ++ci) {
      const int row = nd * dim + ci;
      fr[ci] = !M.dmask[row];
      const int li = row - r0, len = srow[li + 1] - srow[li];
      for (int j = 0; j < len; ++j) {
        const int cc = (j < js ? scol[j * nr + li] : gcol[(size_t)j * n + li]) - nd * dim;
        if (cc >= 0 && cc < dim) a[ci][cc] = j < js ? sval[j * nr + li] : gval[(size_t)j * n + li];
      }
    }
    for (int ci = 0; ci < 3; ++ci)
      for (int cj = 0; cj < 3; ++cj)
        if (ci >= dim || cj >= dim || !fr[ci] || !fr[cj]) a[ci][cj] = (ci == cj) ? 1.0 : 0.0;
    const double det = a[0][0] * (a[1][1] * a[2][2] - a[1][2] * a[2][1]) -
                       a[0][1] * (a[1][0] * a[2][2] - a[1][2] * a[2][0]) +
                       a[0][2] * (a[1][0] * a[2][1] - a[1][1] * a[2][0]);
    inv[0][0] = (a[1][1] * a[2][2] - a[1][2] * a[2][1]) / det;
    inv[0][1] = (a[0][2] * a[2][1] - a[0][1] * a[2][2]) / det;
    inv[0][2] = (a[0][1] * a[1][2] - a[0][2] * a[1][1]) / det;
    inv[1][0] = (a[1][2] * a[2][0] - a[1][0] * a[2][2]) / det;
    inv[1][1] = (a[0][0] * a[2][2] - a[0][2] * a[2][0]) / det;
    inv[1][2] = (a[0][2] * a[1][0] - a[0][0] * a[1][2]) / det;
    inv[2][0] = (a[1][0] * a[2][1] - a[1][1] * a[2][0]) / det;
    inv[2][1] = (a[0][1] * a[2][0] - a[0][0] * a[2][1]) / det;
    inv[2][2] = (a[0][0] * a[1][1] - a[0][1] * a[1][0]) / det;
    for (int ci = 0; ci < dim; ++ci)
      for (int cj = 0; cj < dim; ++cj)
        mi[((nd - nd0) * dim + ci) * dim + cj] = (fr[ci] && fr[cj]) ? inv[ci][cj] : 0.0;
  }
  __syncthreads();
  for (int i = tid; i < nr; i += CGG_THR) {
    const int gi = r0 + i;
    x[i] = 0.0;
    r[i] = M.dmask[gi] ? 0.0 : b[gi];
    sv[i] = 0.0;
    if (M.dmask[gi])
      for (int j = 0; j < ew; ++j) {
        if (j < js) sval[j * nr + i] = 0.0;
        else gval[(size_t)j * n + i] = 0.0;
      }
  }
  if (CC) {
    const int e00 = M.cc.lnptr_g[la0];
    for (int i = tid; i < nr; i += CGG_THR) srel[i] = M.cc.rel[(size_t)r0 + i];
    for (int q = tid; q <= nla; q += CGG_THR) slnp[q] = M.cc.lnptr_g[la0 + q] - e00;
    for (int a = tid; a < M.cc.nagg; a += CGG_THR) sntch[a] = M.cc.ntch_g[a];
    for (int t = tid; t < M.cc.nagg * KC; t += CGG_THR) stch[t] = M.cc.tch_g[t];
    for (int q = warp; q < nla; q += NWARP)
      for (int e = M.cc.lnptr_g[la0 + q] + lane; e < M.cc.lnptr_g[la0 + q + 1]; e += 32) {
        const int l = M.cc.lnode_g[e];
        sln[e - e00] = l;
        for (int c = 0; c < dim; ++c) sq[l * dim + c] = M.dmask[r0 + l * dim + c] ? -1 : q;
      }
    for (int t = tid; t < nl * nc; t += CGG_THR) {
      const int cc = t / nl, rw = t - cc * nl, q = rw / NM, m = rw - q * NM;
      sainv[cc * nlp + rw] = (float)M.cc.Ainv[(size_t)(M.cc.lagg_g[la0 + q] * NM + m) * nc + cc];
    }
  }
  __syncthreads();
  // CC: (P^T r, P^T s) partials of this CTA's aggregates -> gpart (global, read after the grid barrier)
  auto cc_restrict = [&](bool with_s) {
    for (int u = tid; u < 2 * nl * CC_NCH; u += CGG_THR) {
      const int ch = u % CC_NCH, tv = u / CC_NCH, t = tv >> 1, q = t / NM, m = t - q * NM;
      const double* vec = (tv & 1) ? sv : r;
      const int e0 = slnp[q], L = slnp[q + 1] - e0;
      double acc = 0.0;
      if (!(tv & 1) || with_s)
        for (int e = e0 + L * ch / CC_NCH; e < e0 + L * (ch + 1) / CC_NCH; ++e) {
          const int l = sln[e];
          if (m < dim) {
            acc += vec[l * dim + m];
          } else {
            const double* d = srel + l * dim;
#pragma unroll
            for (int c = 0; c < 3; ++c)
              if (c < dim) acc += cc_coef(dim, c, m, d) * vec[l * dim + c];
          }
        }
      cpart[u] = acc;
    }
    __syncthreads();
    double* gp = reinterpret_cast<double*>(gpart + (size_t)g * nlm);
    for (int tv = tid; tv < 2 * nl; tv += CGG_THR) {
      double acc = 0.0;
#pragma unroll
      for (int ch = 0; ch < CC_NCH; ++ch) acc += cpart[tv * CC_NCH + ch];
      gp[tv] = acc;
    }
  };
  // CC: r_c from the partials of the CTAs touching each aggregate, then zc = A_c^-1 r_c (fp32)
  auto cc_solve = [&](double alpha) {
    for (int c = tid; c < nc; c += CGG_THR) {
      const int a = c / NM, m = c - a * NM, nt = sntch[a];
      double sr = 0.0, ss = 0.0;
      for (int k = 0; k < nt; ++k) {
        const int tk = stch[a * KC + k];
        const double2 t = __ldcg(gpart + (size_t)(tk >> 16) * nlm + (tk & 0xffff) * NM + m);
        sr += t.x;
        ss += t.y;
      }
      rcf[c] = (float)(sr - alpha * ss);
    }
    __syncthreads();
    for (int t0 = warp * 8; t0 < nl; t0 += NWARP * 8) {
      const int t = t0 + (lane & 7), cg = lane >> 3;
      float a0 = 0.0f, a1 = 0.0f;
      if (t < nl) {
        int c = cg;
        for (; c + 4 < nc; c += 8) {
          a0 = fmaf(sainv[c * nlp + t], rcf[c], a0);
          a1 = fmaf(sainv[(c + 4) * nlp + t], rcf[c + 4], a1);
        }
        if (c < nc) a0 = fmaf(sainv[c * nlp + t], rcf[c], a0);
      }
      float a = a0 + a1;
      a += __shfl_xor_sync(0xffffffffu, a, 8);
      a += __shfl_xor_sync(0xffffffffu, a, 16);
      if (cg == 0 && t < nl) zc[t] = (double)a;
    }
    __syncthreads();
  };
  if (CC) {
    cc_restrict(false);
    grid.sync();
    cc_solve(0.0);
  }
  // block reduction of up to 2 partials into part[g * 4 + j0 .. j0 + nv)
  auto publish = [&](double v0, double v1, int j0, int nv) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v0 += __shfl_xor_sync(0xffffffffu, v0, o);
      v1 += __shfl_xor_sync(0xffffffffu, v1, o);
    }
    if (lane == 0) { wred[warp] = v0; wred[32 + warp] = v1; }
    __syncthreads();
    if (tid < nv) {
      double a = 0.0;
      for (int k = 0; k < CGG_THR / 32; ++k) a += wred[32 * tid + k];
      part[g * 4 + j0 + tid] = a;
    }
  };
  // z = M^-1 r (local rows) -> zl, zg; (r.z, r.r) partials
  auto precond = [&]() {
    double rz = 0.0, rr = 0.0;
    for (int i = tid; i < nr; i += CGG_THR) {
      const int nd = i / dim;
      double z = 0.0;
      for (int cj = 0; cj < dim; ++cj) z += mi[i * dim + cj] * r[nd * dim + cj];
      if (CC) {
        const int q = sq[i];
        if (q >= 0)
#pragma unroll
          for (int m = 0; m < 6; ++m)
            if (m < NM) z += cc_coef(dim, i - nd * dim, m, srel + nd * dim) * zc[q * NM + m];
      }
      zl[i] = z;
      zg[r0 + i] = z;
      rz += r[i] * z;
      rr += r[i] * r[i];
    }
    publish(rz, rr, 0, 2);
  };
  // w = A z (gathers from zg through L2); (z.w) partial
  auto spmv = [&](double beta_s) {  // CC: also s = w + beta_s s
    double zw = 0.0;
    for (int i = tid; i < nr; i += CGG_THR) {
      double s0 = 0.0, s1 = 0.0;
      int j = 0;
      for (; j + 1 < js; j += 2) {
        s0 += sval[j * nr + i] * __ldcg(zg + scol[j * nr + i]);
        s1 += sval[(j + 1) * nr + i] * __ldcg(zg + scol[(j + 1) * nr + i]);
      }
      if (j < js) {
        s0 += sval[j * nr + i] * __ldcg(zg + scol[j * nr + i]);
        ++j;
      }
      for (; j < ew; ++j) s0 += __ldcg(gval + (size_t)j * n + i) * __ldcg(zg + __ldcg(gcol + (size_t)j * n + i));
      const double wi = s0 + s1;
      w[i] = wi;
      if (CC) sv[i] = wi + beta_s * sv[i];
      zw += zl[i] * wi;
    }
    publish(zw, 0.0, 2, 1);
    if (CC) cc_restrict(true);  // publish's CTA barrier also completes w and s
  };
  precond();
  grid.sync();
  double gam = cgg_sum(part, G, 0, sred), rr = cgg_sum(part, G, 1, sred);
  const double bnorm = sqrt(rr);
  int it = 0, status = 0;
  if (bnorm > 0.0) {
    spmv(0.0);
    grid.sync();
    double del = cgg_sum(part, G, 2, sred);
    if (!(del > 0.0)) status = 6;
    double alpha = gam / del;
    for (int i = tid; i < nr; i += CGG_THR) { p[i] = zl[i]; sv[i] = w[i]; }
    for (it = 1; it <= max_iter && status == 0; ++it) {
      if (CC) cc_solve(alpha);
      for (int i = tid; i < nr; i += CGG_THR) {
        x[i] += alpha * p[i];
        r[i] -= alpha * sv[i];
      }
      __syncthreads();  // r complete before the block preconditioner mixes components
      precond();
      grid.sync();
      const double gn = cgg_sum(part, G, 0, sred);
      rr = cgg_sum(part, G, 1, sred);
      if (sqrt(rr) <= rtol * bnorm) break;
      const double beta = gn / gam;
      spmv(beta);
      for (int i = tid; i < nr; i += CGG_THR) {
        p[i] = zl[i] + beta * p[i];
        if (!CC) sv[i] = w[i] + beta * sv[i];
      }
      grid.sync();
      del = cgg_sum(part, G, 2, sred);
      const double den = del - beta * gn / alpha;
      if (!(den > 0.0)) { status = 6; break; }
      alpha = gn / den;
      gam = gn;
    }
    if (status == 0 && it > max_iter) { status = 5; it = max_iter; }
  }
  for (int i = tid; i < nr; i += CGG_THR) {
    const int gi = r0 + i;
    xout[gi] = M.dmask[gi] ? scale * M.dval[gi] : x[i];
  }
  if (g == 0 && tid == 0) {
    st->iterations = it;
    st->status = status;
    st->rel_residual = bnorm > 0.0 ? sqrt(rr) / bnorm : 0.0;
    st->rhs_norm = bnorm;
  }
}

bool launch_macro_cg_grid(const MacroDev& M, const double* val, const double* rhs, double scale, double rtol,
                          int max_iter, double* x, double* zg, double* part, CgState* st, cudaStream_t s,
                          int* extra_launches) {
  if (extra_launches) *extra_launches = 0;
  int dev = 0, sms = 0, coop = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop || sms <= 0 || sms > 2 * 592) return false;
  const int G = sms;
  int max_nr = 0;
  for (int g = 0; g < G; ++g) {
    const int nd0 = (int)((long)M.n_nodes * g / G), nd1 = (int)((long)M.n_nodes * (g + 1) / G);
    max_nr = std::max(max_nr, (nd1 - nd0) * M.dim);
  }
  const size_t cap = 227 * 1024;
  for (int use_cc = (M.cc.nc > 0 && M.cc.ggrid == G) ? 1 : 0; use_cc >= 0; --use_cc) {
    size_t base = (size_t)(8 + 96 + 6 * max_nr + max_nr * M.dim) * 8 + (size_t)(max_nr + 1) * 4 + 64;
    if (use_cc) {
      const int nla = M.cc.nla_max_g, nl = nla * M.cc.nm, nlp = (nl + 7) / 16 * 16 + 8;
      base += 16 + (size_t)(nl + (M.cc.nc + 1) / 2 + nl * CC_NCH * 2 + max_nr) * 8 + (size_t)nlp * M.cc.nc * 4 +
              (size_t)(max_nr + nla + 1 + max_nr / M.dim + M.cc.nagg * (1 + M.cc.kmax_g)) * 4;
    }
    if (base > cap) continue;
    int js = (int)std::min<size_t>(M.cg_ellw, (cap - base) / ((size_t)max_nr * 12));
    if (js < M.cg_ellw) js &= ~1;
    const size_t sm = base + (size_t)max_nr * js * 12;
    auto k = use_cc ? k_macro_cg_grid<true> : k_macro_cg_grid<false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int per = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, CGG_THR, sm) != cudaSuccess || per < 1) {
      cudaGetLastError();
      continue;
    }
    if (use_cc) {
      if (!launch_coarse_setup(M, val, s)) {
        cudaGetLastError();
        continue;
      }
      if (extra_launches) *extra_launches = 2;
    }
    if (getenv("HOM_CG_VERBOSE")) fprintf(stderr, "cgg: cc %d G %d js %d/%d smem %zu\n", use_cc, G, js, M.cg_ellw, sm);
    MacroDev Mc = M;
    void* args[] = {&Mc, (void*)&val, (void*)&rhs, &scale, &rtol, &max_iter, &x, &st, &zg, &part, &js};
    cudaError_t e = cudaLaunchCooperativeKernel((void*)k, dim3(G), dim3(CGG_THR), args, sm, s);
    if (e == cudaSuccess) return true;
    cudaGetLastError();
  }
  return false;
}

// ---------------------------------------------------------------- K6 SpMV + large-problem PCG
// For macro problems too large for one cluster's shared memory (scaled meshes, multi-GPU
// weak scaling): grid-wide kernels.  K6 (k_spmv) streams the CSR matrix once per call --
// HBM-bound, 8 lanes per row (coalesced 64 B of values + 32 B of columns per step), the
// gathered x stays in L2.  Dot products are reduced per block and then in a fixed order by
// one block (deterministic); the PCG scalars never leave the device; the host checks
// convergence every CGL_CHECK iterations.
constexpr int SPMV_THR = 256, SPMV_LPR = 4, CGL_BLOCKS = 592, CGL_CHECK = 16;

// y = A x on the free rows (Dirichlet rows -> 0); optional partial sums of x.y per block.
// Latency-bound by construction (row -> rowptr -> col -> x are dependent loads), so the kernel
// keeps many bytes in flight: every lane issues all (up to SPMV_PASS per pass) value/column
// loads of its row before any gather, and the next row's rowptr/mask are prefetched under the
// current row.  SPMV_LPR lanes per row.
constexpr int SPMV_PASS = 5;
__global__ void __launch_bounds__(SPMV_THR) k_spmv(MacroDev M, const double* __restrict__ val,
                                                   const double* __restrict__ x, double* __restrict__ y,
                                                   double* __restrict__ part) {
  const int lane = threadIdx.x & (SPMV_LPR - 1);
  const long row0 = ((long)blockIdx.x * SPMV_THR + threadIdx.x) / SPMV_LPR;
  const long stride = (long)gridDim.x * SPMV_THR / SPMV_LPR;
  // warp-uniform trip count: every lane reaches the shuffles (rows of a warp are consecutive)
  const long wrow0 = row0 - (threadIdx.x & 31) / SPMV_LPR;
  const long n = M.ndof;
  double dot = 0.0;
  int kb = 0, ke = 0;
  bool act = false;
  if (row0 < n) {
    kb = __ldg(M.rowptr + row0);
    ke = __ldg(M.rowptr + row0 + 1);
    act = !M.dmask[row0];
  }
  for (long wr = wrow0, row = row0; wr < n; wr += stride, row += stride) {
    double v[SPMV_PASS];
    int c[SPMV_PASS];
    double s = 0.0;
    int k = kb + lane;
    const int kend = act ? ke : kb;
#pragma unroll
    for (int j = 0; j < SPMV_PASS; ++j) {  // all loads of the pass issued together
      const int kk = k + j * SPMV_LPR;
      v[j] = kk < kend ? __ldcs(val + kk) : 0.0;
      c[j] = kk < kend ? __ldcs(M.col + kk) : 0;
    }
    const long nrow = row + stride;  // prefetch the next row's range under the gathers
    int nkb = 0, nke = 0;
    bool nact = false;
    if (nrow < n) {
      nkb = __ldg(M.rowptr + nrow);
      nke = __ldg(M.rowptr + nrow + 1);
      nact = !M.dmask[nrow];
    }
#pragma unroll
    for (int j = 0; j < SPMV_PASS; ++j) s += v[j] * __ldg(x + c[j]);
    for (k += SPMV_PASS * SPMV_LPR; k < kend; k += SPMV_LPR) s += __ldcs(val + k) * __ldg(x + __ldcs(M.col + k));
#pragma unroll
    for (int o = SPMV_LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0 && row < n) {
      y[row] = s;
      dot += s * x[row];
    }
    kb = nkb;
    ke = nke;
    act = nact;
  }
  if (part) {
    __shared__ double red[SPMV_THR / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dot;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < SPMV_THR / 32; ++w) t += red[w];
      part[blockIdx.x] = t;
    }
  }
}
void launch_spmv(const MacroDev& M, const double* val, const double* x, double* y, cudaStream_t s) {
  k_spmv<<<CGL_BLOCKS * 4, SPMV_THR, 0, s>>>(M, val, x, y, nullptr);
}

// scalars sc: [0] rz, [1] alpha, [2] beta, [3] rr, [4] bnorm^2, [5] status
__global__ void k_cgl_reduce(const double* __restrict__ part, int nb, int nv, double* __restrict__ out) {
  __shared__ double red[4][32];
  for (int v = 0; v < nv; ++v) {
    double t = 0.0;
    for (int i = threadIdx.x; i < nb; i += 32) t += part[v * nb + i];  // fixed assignment and order
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) red[v][0] = t;
  }
  __syncwarp();
  if (threadIdx.x == 0)
    for (int v = 0; v < nv; ++v) out[v] = red[v][0];
}

// init: x = 0, r = b (free), z = D^-1 r, p = z; partials of (r.z, r.r)
__global__ void k_cgl_init(MacroDev M, const double* __restrict__ b, const double* __restrict__ diag,
                           double* __restrict__ x, double* __restrict__ r, double* __restrict__ p,
                           double* __restrict__ part) {
  double rz = 0.0, rr = 0.0;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < M.ndof; i += (long)gridDim.x * blockDim.x) {
    const bool d = M.dmask[i];
    const double ri = d ? 0.0 : b[i], zi = d ? 0.0 : ri / diag[i];
    x[i] = 0.0;
    r[i] = ri;
    p[i] = zi;
    rz += ri * zi;
    rr += ri * ri;
  }
  __shared__ double red[2][SPMV_THR / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    rz += __shfl_xor_sync(0xffffffffu, rz, o);
    rr += __shfl_xor_sync(0xffffffffu, rr, o);
  }
  if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = rz; red[1][threadIdx.x >> 5] = rr; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, c = 0.0;
    for (int w = 0; w < SPMV_THR / 32; ++w) { a += red[0][w]; c += red[1][w]; }
    part[blockIdx.x] = a;
    part[gridDim.x + blockIdx.x] = c;
  }
}

// alpha = rz / pq (sc[1]); breakdown -> status 6
__global__ void k_cgl_alpha(double* sc, const double* pq) {
  if (!(pq[0] > 0.0)) sc[5] = 6.0;
  sc[1] = sc[0] / pq[0];
}

// x += a p; r -= a q; z = D^-1 r (into q); partials of (r.z, r.r)
__global__ void k_cgl_update(MacroDev M, const double* __restrict__ diag, const double* __restrict__ sc,
                             double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                             double* __restrict__ q, double* __restrict__ part) {
  const double a = sc[1];
  double rz = 0.0, rr = 0.0;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < M.ndof; i += (long)gridDim.x * blockDim.x) {
    if (M.dmask[i]) { q[i] = 0.0; continue; }
    x[i] += a * p[i];
    const double ri = r[i] - a * q[i];
    r[i] = ri;
    const double zi = ri / diag[i];
    q[i] = zi;
    rz += ri * zi;
    rr += ri * ri;
  }
  __shared__ double red[2][SPMV_THR / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    rz += __shfl_xor_sync(0xffffffffu, rz, o);
    rr += __shfl_xor_sync(0xffffffffu, rr, o);
  }
  if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = rz; red[1][threadIdx.x >> 5] = rr; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a2 = 0.0, c = 0.0;
    for (int w = 0; w < SPMV_THR / 32; ++w) { a2 += red[0][w]; c += red[1][w]; }
    part[blockIdx.x] = a2;
    part[gridDim.x + blockIdx.x] = c;
  }
}

// beta = rz_new / rz; rz = rz_new; rr (sc[3])
__global__ void k_cgl_beta(double* sc, const double* red) {
  sc[2] = red[0] / sc[0];
  sc[0] = red[0];
  sc[3] = red[1];
}

// p = z + beta p
__global__ void k_cgl_p(MacroDev M, const double* __restrict__ sc, const double* __restrict__ z,
                        double* __restrict__ p) {
  const double be = sc[2];
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < M.ndof; i += (long)gridDim.x * blockDim.x)
    p[i] = z[i] + be * p[i];
}

__global__ void k_cgl_final(MacroDev M, const double* __restrict__ x, double scale, double* __restrict__ xout) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < M.ndof; i += (long)gridDim.x * blockDim.x)
    xout[i] = M.dmask[i] ? scale * M.dval[i] : x[i];
}

// work: [x | r | p | q] (4 n) ; sc: >= 6 + 4 doubles; part: >= 2 * CGL_BLOCKS * 4 doubles
void launch_macro_cg_large(const MacroDev& M, const double* val, const double* diag, const double* rhs,
                           double scale, double rtol, int max_iter, double* xout, double* work, double* sc,
                           double* part, CgState* st, cudaStream_t s) {
  const long n = M.ndof;
  double *x = work, *r = work + n, *p = work + 2 * n, *q = work + 3 * n;
  const int nbv = CGL_BLOCKS, nbs = CGL_BLOCKS * 4;
  double* red = sc + 6;
  cudaMemsetAsync(sc, 0, 6 * sizeof(double), s);
  k_cgl_init<<<nbv, SPMV_THR, 0, s>>>(M, rhs, diag, x, r, p, part);
  k_cgl_reduce<<<1, 32, 0, s>>>(part, nbv, 2, red);
  double h[2];
  cudaMemcpyAsync(h, red, 2 * sizeof(double), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  cudaMemcpyAsync(sc, red, sizeof(double), cudaMemcpyDeviceToDevice, s);  // rz
  const double bnorm = sqrt(h[1]);
  int it = 0, status = 0;
  double rr = h[1];
  if (bnorm > 0.0) {
    for (it = 1; it <= max_iter; ++it) {
      k_spmv<<<nbs, SPMV_THR, 0, s>>>(M, val, p, q, part);
      k_cgl_reduce<<<1, 32, 0, s>>>(part, nbs, 1, red + 2);
      k_cgl_alpha<<<1, 1, 0, s>>>(sc, red + 2);
      k_cgl_update<<<nbv, SPMV_THR, 0, s>>>(M, diag, sc, x, r, p, q, part);
      k_cgl_reduce<<<1, 32, 0, s>>>(part, nbv, 2, red);
      k_cgl_beta<<<1, 1, 0, s>>>(sc, red);
      k_cgl_p<<<nbv, SPMV_THR, 0, s>>>(M, sc, q, p);
      if (it % CGL_CHECK == 0 || it == max_iter) {
        double hs[6];
        cudaMemcpyAsync(hs, sc, 6 * sizeof(double), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        rr = hs[3];
        if (hs[5] != 0.0) { status = 6; break; }
        if (sqrt(rr) <= rtol * bnorm) break;
      }
    }
    if (status == 0 && it > max_iter) { status = 5; it = max_iter; }
  }
  k_cgl_final<<<nbv, SPMV_THR, 0, s>>>(M, x, scale, xout);
  CgState h_st{it, status, bnorm > 0.0 ? sqrt(rr) / bnorm : 0.0, bnorm};
  cudaMemcpyAsync(st, &h_st, sizeof(h_st), cudaMemcpyHostToDevice, s);
  cudaStreamSynchronize(s);
}

// ---------------------------------------------------------------- K8 recovery
// accumulate = 0: w = -X[:, :m] kin            (small strain, kin = eps)
// accumulate = 1: w += -(X[:, m] + X[:, :m] kin) (finite strain, kin = grad du)
__global__ void k_recover(RveDev R, int b0, int nb, const double* __restrict__ X, const double* __restrict__ kin,
                          double* __restrict__ w, int accumulate) {
  long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)nb * R.npad) return;
  int b = b0 + (int)(t / R.npad), i = (int)(t % R.npad);
  t += (long)b0 * R.npad;
  const double* xr = X + ((long)(b - R.xb0) * R.NT + i) * RHSW;
  const double* kb = kin + (long)b * R.m;
  double v = 0.0;
  for (int k = 0; k < R.m; ++k) v += xr[k] * kb[k];
  if (accumulate) w[t] -= xr[R.m] + v;
  else if (R.nat_of) {  // external (natural) layout
    const int dr = R.npad / R.n_indep;
    w[(long)b * R.npad + (long)__ldg(R.nat_of + i / dr) * dr + i % dr] = -v;
  } else w[t] = -v;
}

__global__ void k_permute_w(RveDev R, long n, const double* __restrict__ src, double* __restrict__ dst,
                            int to_api) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int dr = R.npad / R.n_indep;
  const long b = t / R.npad;
  const int i = (int)(t % R.npad);  // internal index
  const long e = b * R.npad + (long)__ldg(R.nat_of + i / dr) * dr + i % dr;
  if (to_api) dst[e] = src[t];
  else dst[t] = src[e];
}

__global__ void k_expand_kff(RveDev R, const double* __restrict__ Kb, double* __restrict__ out) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const int n = R.npad;
  if (t >= (long)n * n) return;
  const int i = (int)(t / n), j = (int)(t % n), dr = n / R.n_indep;
  int ii = i, jj = j;  // natural -> internal DOF
  if (R.int_of) {
    ii = __ldg(R.int_of + i / dr) * dr + i % dr;
    jj = __ldg(R.int_of + j / dr) * dr + j % dr;
  }
  if (ii < jj) { const int x = ii; ii = jj; jj = x; }  // lower tiles only (symmetric)
  const int I = ii / TILE, J = jj / TILE;
  double v = 0.0;
  const int slot = __ldg(R.tslot + I * R.nt + J);
  if (slot >= 0 && R.tile_nz[I * R.nt + J]) v = Kb[(long)slot * TILE_ELEMS + (ii % TILE) * TILE + jj % TILE];
  out[t] = v;
}

void launch_expand_kff(const RveDev& R, const double* Kb, double* out, cudaStream_t s) {
  const long n = (long)R.npad * R.npad;
  k_expand_kff<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(R, Kb, out);
}

void launch_permute_w(const RveDev& R, int B, const double* src, double* dst, int to_api, cudaStream_t s) {
  const long n = (long)B * R.npad;
  if (n <= 0) return;
  if (!R.nat_of) {
    cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDeviceToDevice, s);
    return;
  }
  k_permute_w<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(R, n, src, dst, to_api);
}

void launch_recover(const RveDev& R, int b0, int nb, const double* X, const double* kin, double* w,
                    int accumulate, cudaStream_t s) {
  long n = (long)nb * R.npad;
  if (n <= 0) return;
  k_recover<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(R, b0, nb, X, kin, w, accumulate);
}

}  // namespace hom
