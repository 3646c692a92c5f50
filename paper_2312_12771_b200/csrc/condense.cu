// condense.cu -- K2/K3/K4: batched blocked FP64 Cholesky, influence solves and
// Schur-complement epilogue, one CTA per RVE.
//
// For RVE b:
//   K_ff = G G^T                       (left-looking over 64x64 tiles, in place)
//   Y    = G^-1 [K_fe | r_f]            (fused into the diagonal step of each tile column)
//   C_eff = <C> - Y_e^T Y_e / |Omega|  (K4 epilogue; = <C> - K_ef K_ff^-1 K_fe / |Omega|,
//                                      eq:solution1/2 with the Dirac basis)
//   P_eff = <P> - Y_e^T Y_r / |Omega|  (finite strain, RHS of eq:solution2)
//   X    = G^-T Y = K_ff^-1 [K_fe | r_f] (backward pass; kept for recovery)
//
// Every 64^3 product runs on the FP64 tensor cores: mma.sync.m8n8k4.f64 (DMMA;
// sm_100a has no FP64 tcgen05 kind).  Operands are staged in
// shared memory with cp.async (16 B) into an XOR-swizzled layout that makes the
// DMMA fragment reads bank-conflict free; diagonal tiles are stored inverted
// (G_JJ^-1) so that the triangular solves are DMMA GEMMs too.
#include "hom_internal.cuh"

namespace hom {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// swizzled word index inside a [rows][32] k-chunk and a [64][64] tile
__device__ __forceinline__ int sw32(int r, int k) { return r * KC + (k ^ ((r & 3) << 2)); }
__device__ __forceinline__ int sw64(int r, int c) { return r * TILE + (c ^ ((r & 3) << 2)); }
// [rows][8] right-hand-side block
__device__ __forceinline__ int swy(int k, int n) { return k * RHSW + (n ^ (((k >> 1) & 1) << 2)); }

__device__ __forceinline__ const double* tile_ptr(const double* Kb, int I, int J) {
  return Kb + (long)(I * (I + 1) / 2 + J) * TILE_ELEMS;
}

// Stage a [64][32] k-chunk of a row-major 64x64 global tile into swizzled smem.
__device__ __forceinline__ void stage_chunk(double* dst, const double* src_tile, int kc, int tid) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int idx = tid + NTHR * i;  // 0..1023 16-byte pieces
    int r = idx >> 4, c2 = idx & 15;
    cp_async16(dst + sw32(r, 2 * c2), src_tile + r * TILE + kc * KC + 2 * c2);
  }
}
// Stage a full 64x64 tile into swizzled smem.
__device__ __forceinline__ void stage_tile(double* dst, const double* src_tile, int tid) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int idx = tid + NTHR * i;  // 0..2047
    int r = idx >> 5, c2 = idx & 31;
    cp_async16(dst + sw64(r, 2 * c2), src_tile + r * TILE + 2 * c2);
  }
}
// Stage rows [r0, r0+n) of an [NT][8] RHS block into swizzled [n][8] smem (n <= 64).
__device__ __forceinline__ void stage_rhs(double* dst, const double* src, int n, int tid) {
  int pieces = n * (RHSW / 2);
  for (int idx = tid; idx < pieces; idx += NTHR) {
    int k = idx >> 2, c2 = idx & 3;
    cp_async16(dst + swy(k, 2 * c2), src + k * RHSW + 2 * c2);
  }
}

// acc[4][2][2] += A(64x32 chunk) * B(64x32 chunk)^T for warp tile rows R0.., cols C0..
__device__ __forceinline__ void mma_chunk(double (&acc)[4][2][2], const double* sA, const double* sB,
                                          int R0, int C0, int lane) {
  const int lr = lane >> 2, lc = lane & 3;
#pragma unroll
  for (int k0 = 0; k0 < KC; k0 += 4) {
    double a[4], b[2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) a[mi] = sA[sw32(R0 + 8 * mi + lr, k0 + lc)];
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) b[ni] = sB[sw32(C0 + 8 * ni + lr, k0 + lc)];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
  }
}

// ------------------------------------------------------------------ diagonal tile
// One warp: Cholesky of the 16x16 block at (k0,k0) of the swizzled 64x64 tile sT
// (lower part, in registers, shuffles only) and its inverse into the same block of sX.
// Returns the first failing local pivot (16 = none); warp-uniform.
__device__ __forceinline__ int chol_inv16(double* sT, double* sX, int k0, int lane) {
  const unsigned FULL = 0xffffffffu;
  const int r = lane & 15;
  double a[16], ip[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) a[c] = (c <= r) ? sT[sw64(k0 + r, k0 + c)] : 0.0;
  int fail = 16;
  // Pivot chain: one rsqrt per pivot (no sqrt, no division); every lane keeps 1/L_kk.
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    double dkk = __shfl_sync(FULL, a[k], k);
    if (!(dkk > 0.0) && fail == 16) fail = k;
    ip[k] = rsqrt(dkk);
    a[k] = (r == k) ? dkk * ip[k] : a[k] * ip[k];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (j > k) {  // compile-time after unrolling: a[] stays in registers
        double ljk = __shfl_sync(FULL, a[k], j);
        if (r >= j) a[j] = fma(-a[k], ljk, a[j]);
      }
    }
  }
  if (lane < 16) {
#pragma unroll
    for (int c = 0; c < 16; ++c)
      if (c <= r) sT[sw64(k0 + r, k0 + c)] = a[c];
  }
  __syncwarp();
  // X = L^-1: lane c builds column c by forward substitution (L rows read as smem
  // broadcasts), two partial sums to halve the dependent FMA chain.
  const int c = lane & 15;
  double x[16];
#pragma unroll
  for (int rr = 0; rr < 16; ++rr) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int k = 0; k < 16; k += 2) {
      if (k < rr) s0 = fma(sT[sw64(k0 + rr, k0 + k)], x[k], s0);
      if (k + 1 < rr) s1 = fma(sT[sw64(k0 + rr, k0 + k + 1)], x[k + 1], s1);
    }
    x[rr] = (rr >= c) ? (((rr == c) ? 1.0 : 0.0) - (s0 + s1)) * ip[rr] : 0.0;
  }
  if (lane < 16) {
#pragma unroll
    for (int rr = 0; rr < 16; ++rr) sX[sw64(k0 + rr, k0 + c)] = x[rr];
  }
  return fail;
}

// 8x8 output tile: acc += A[r0.., k0..k0+nk) * B[c0.., k0..)^T   (both [row][k], sw64)
__device__ __forceinline__ void tile8_abt(double (&acc)[2], const double* A, int r0, const double* B, int c0,
                                          int k0, int nk, int lane, double sign) {
  const int lr = lane >> 2, lc = lane & 3;
  for (int k = k0; k < k0 + nk; k += 4)
    dmma(acc[0], acc[1], sign * A[sw64(r0 + lr, k + lc)], B[sw64(c0 + lr, k + lc)]);
}
// 8x8 output tile: acc += A[r0.., k..) * B[k.., c0..)   (A [row][k], B [k][col], sw64)
__device__ __forceinline__ void tile8_ab(double (&acc)[2], const double* A, int r0, const double* B, int c0,
                                         int k0, int nk, int lane, double sign) {
  const int lr = lane >> 2, lc = lane & 3;
  for (int k = k0; k < k0 + nk; k += 4)
    dmma(acc[0], acc[1], sign * A[sw64(r0 + lr, k + lc)], B[sw64(k + lc, c0 + lr)]);
}

// Blocked (16-wide) Cholesky of the 64x64 tile in sT followed by the blocked
// triangular inverse; on return sT holds G_JJ^-1 (exact zeros above the
// diagonal).  sX is 64x64 + 768 doubles of scratch.  All block updates run on
// DMMA; about 18 CTA barriers instead of one per column.
__device__ __forceinline__ bool factor_invert_diag(double* sT, double* sX, int* sFail, int J, int tid) {
  const int lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  for (int i = tid; i < TILE_ELEMS; i += NTHR) sX[i] = 0.0;
  __syncthreads();
  for (int kb = 0; kb < 4; ++kb) {
    const int k0 = 16 * kb;
    if (warp == 0) {
      int f = chol_inv16(sT, sX, k0, lane);
      if (f < 16 && lane == 0 && sFail[0] == 0) sFail[0] = J * TILE + k0 + f + 1;
    }
    __syncthreads();
    if (sFail[0]) return false;
    if (kb == 3) break;
    const int rb0 = k0 + 16, nrb = (TILE - rb0) / 8;  // row blocks below the panel
    // panel: L_ik = A_ik * Linv_kk^T, rows rb0..63, cols k0..k0+15 (nrb x 2 tiles)
    double pan[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    const int nt_pan = nrb * 2;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      int t = warp + 8 * u;
      if (t < nt_pan) tile8_abt(pan[u], sT, rb0 + 8 * (t >> 1), sX, k0 + 8 * (t & 1), k0, 16, lane, 1.0);
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      int t = warp + 8 * u;
      if (t < nt_pan) {
        int r = rb0 + 8 * (t >> 1) + lr, cc = k0 + 8 * (t & 1) + 2 * lc;
        sT[sw64(r, cc)] = pan[u][0];
        sT[sw64(r, cc + 1)] = pan[u][1];
      }
    }
    __syncthreads();
    // trailing: A_ij -= L_ik L_jk^T for lower 8x8 tiles of rows/cols rb0..63
    const int ntr = nrb * (nrb + 1) / 2;
    for (int t = warp; t < ntr; t += 8) {
      int ti = 0;
      while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
      int tj = t - ti * (ti + 1) / 2;
      int r = rb0 + 8 * ti, cb = rb0 + 8 * tj;
      double acc[2] = {sT[sw64(r + lr, cb + 2 * lc)], sT[sw64(r + lr, cb + 2 * lc + 1)]};
      tile8_abt(acc, sT, r, sT, cb, k0, 16, lane, -1.0);
      sT[sw64(r + lr, cb + 2 * lc)] = acc[0];
      sT[sw64(r + lr, cb + 2 * lc + 1)] = acc[1];
    }
    __syncthreads();
  }
  // off-diagonal blocks of the inverse: X_ik = -X_ii sum_{j=k}^{i-1} L_ij X_jk
  double* sTmp = sX + TILE_ELEMS;  // 3 blocks of 16x16, plain row-major
  for (int i = 1; i < 4; ++i) {
    const int ntile = 4 * i;  // blocks k = 0..i-1, 2x2 tiles each
    double tv[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      int t = warp + 8 * u;
      if (t < ntile) {
        int k = t >> 2, q = t & 3;
        tile8_ab(tv[u], sT, 16 * i + 8 * (q >> 1), sX, 16 * k + 8 * (q & 1), 16 * k, 16 * (i - k), lane, 1.0);
        int rr = 8 * (q >> 1) + lr, cc = 8 * (q & 1) + 2 * lc;
        sTmp[k * 256 + rr * 16 + cc] = tv[u][0];
        sTmp[k * 256 + rr * 16 + cc + 1] = tv[u][1];
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      int t = warp + 8 * u;
      if (t < ntile) {
        int k = t >> 2, q = t & 3;
        int r0 = 8 * (q >> 1), c0 = 8 * (q & 1);
        double acc[2] = {0.0, 0.0};
#pragma unroll
        for (int kk = 0; kk < 16; kk += 4)
          dmma(acc[0], acc[1], -sX[sw64(16 * i + r0 + lr, 16 * i + kk + lc)], sTmp[k * 256 + (kk + lc) * 16 + c0 + lr]);
        tv[u][0] = acc[0];
        tv[u][1] = acc[1];
      }
    }
    // X_ik written after all warps read X_ii / sTmp (X_ii is a different block: no hazard)
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      int t = warp + 8 * u;
      if (t < ntile) {
        int k = t >> 2, q = t & 3;
        int r = 16 * i + 8 * (q >> 1) + lr, cc = 16 * k + 8 * (q & 1) + 2 * lc;
        sX[sw64(r, cc)] = tv[u][0];
        sX[sw64(r, cc + 1)] = tv[u][1];
      }
    }
    __syncthreads();
  }
  for (int i = tid; i < TILE_ELEMS; i += NTHR) sT[i] = sX[i];
  __syncthreads();
  return true;
}

// Smem budget (doubles): sT 4096 | stage[2] x (A 2048 + B 2048 + Yc 256) | sY 512 | sY2 512 | misc
constexpr int STAGE_DBL = 2 * 64 * KC + KC * RHSW;
constexpr int SMEM_DBL = TILE_ELEMS + 2 * STAGE_DBL + 2 * 64 * RHSW + 64;

// ------------------------------------------------------------------ kernel
__global__ void __launch_bounds__(NTHR, 2)
k_condense(RveDev R, int b0, double* __restrict__ Kt, double* __restrict__ Y,
           const double* __restrict__ Cavg, const double* __restrict__ Pavg,
           double* __restrict__ Ceff, double* __restrict__ Peff, double* __restrict__ PavgOut,
           double* __restrict__ X, int* __restrict__ info) {
  extern __shared__ __align__(128) double smem[];
  double* sT = smem;                              // 64x64 swizzled: diag work / G_JJ^-1
  double* sStage = smem + TILE_ELEMS;             // 2 stages (also reused as a 64x64 tile)
  double* sY = sStage + 2 * STAGE_DBL;            // 64x8 swizzled
  double* sY2 = sY + 64 * RHSW;                   // 64x8 swizzled
  double* sMisc = sY2 + 64 * RHSW;                // flags
  int* sFail = reinterpret_cast<int*>(sMisc);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  const int R0 = (warp >> 2) * 32, C0 = (warp & 3) * 16;
  const int bl = blockIdx.x, b = b0 + bl;
  const int nt = R.nt, NT = R.NT;
  double* Kb = Kt + (long)bl * (nt * (nt + 1) / 2) * TILE_ELEMS;
  double* Yb = Y + (long)bl * NT * RHSW;
  double* Xb = X + (long)b * NT * RHSW;

  if (tid == 0) sFail[0] = 0;
  double Sacc = 0.0;  // thread (i,j) = (tid>>3, tid&7), tid < 64: sum_r Y[r][i] Y[r][j]

  // ======================= forward: factor + Y ==============================
  for (int J = 0; J < nt; ++J) {
    // ---------- diagonal tile: acc = sum_K G_JK G_JK^T, yacc = sum_K G_JK Y_K ----------
    double acc[4][2][2] = {};
    double yacc[2] = {0.0, 0.0};
    const int nk = J * 2;  // (K, kc) chunks
    if (nk > 0) {
      stage_chunk(sStage, tile_ptr(Kb, J, 0), 0, tid);
      stage_rhs(sStage + 2 * 64 * KC, Yb, KC, tid);
      cp_async_commit();
    }
    for (int c = 0; c < nk; ++c) {
      if (c + 1 < nk) {
        double* st = sStage + ((c + 1) & 1) * STAGE_DBL;
        int K = (c + 1) >> 1, kc = (c + 1) & 1;
        stage_chunk(st, tile_ptr(Kb, J, K), kc, tid);
        stage_rhs(st + 2 * 64 * KC, Yb + (long)(K * TILE + kc * KC) * RHSW, KC, tid);
        cp_async_commit();
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const double* st = sStage + (c & 1) * STAGE_DBL;
      mma_chunk(acc, st, st, R0, C0, lane);
      {  // yacc (rows 8*warp.., 8 RHS columns) += G_JK chunk * Y_K chunk
        const double* sYc = st + 2 * 64 * KC;
#pragma unroll
        for (int k0 = 0; k0 < KC; k0 += 4) {
          double a = st[sw32(8 * warp + lr, k0 + lc)];
          double bb = sYc[swy(k0 + lc, lr)];
          dmma(yacc[0], yacc[1], a, bb);
        }
      }
      __syncthreads();
    }
    // sT = A_JJ - acc ; sY = Kfe_J - yacc
    {
      const double* Ajj = tile_ptr(Kb, J, J);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) {
          int r = R0 + 8 * mi + lr, cc = C0 + 8 * ni + 2 * lc;
          double2 a = *reinterpret_cast<const double2*>(Ajj + r * TILE + cc);
          sT[sw64(r, cc)] = a.x - acc[mi][ni][0];
          sT[sw64(r, cc + 1)] = a.y - acc[mi][ni][1];
        }
      int r = 8 * warp + lr, cc = 2 * lc;
      double2 y = *reinterpret_cast<const double2*>(Yb + (long)(J * TILE + r) * RHSW + cc);
      sY[swy(r, cc)] = y.x - yacc[0];
      sY[swy(r, cc + 1)] = y.y - yacc[1];
    }
    __syncthreads();
    // ---------- blocked Cholesky + inverse of the 64x64 diagonal tile ----------
    if (!factor_invert_diag(sT, sStage, sFail, J, tid)) break;
    // ---------- Y_J = G_JJ^-1 (Kfe_J - sum) ; S += Y_J^T Y_J ----------
    {
      double y[2] = {0.0, 0.0};
      const int r = 8 * warp;
#pragma unroll
      for (int k0 = 0; k0 < TILE; k0 += 4) {
        double a = sT[sw64(r + lr, k0 + lc)];
        double bb = sY[swy(k0 + lc, lr)];
        dmma(y[0], y[1], a, bb);
      }
      int rr = r + lr, cc = 2 * lc;
      sY2[swy(rr, cc)] = y[0];
      sY2[swy(rr, cc + 1)] = y[1];
      *reinterpret_cast<double2*>(Yb + (long)(J * TILE + rr) * RHSW + cc) = make_double2(y[0], y[1]);
    }
    // store G_JJ^-1 as tile (J,J)
    {
      double* Gjj = Kb + (long)(J * (J + 1) / 2 + J) * TILE_ELEMS;
      for (int idx = tid; idx < TILE_ELEMS / 2; idx += NTHR) {
        int r = idx >> 5, cc = 2 * (idx & 31);
        *reinterpret_cast<double2*>(Gjj + r * TILE + cc) = make_double2(sT[sw64(r, cc)], sT[sw64(r, cc + 1)]);
      }
    }
    __syncthreads();
    if (tid < 64) {
      const int i = tid >> 3, j = tid & 7;
      double s = 0.0;
      for (int r = 0; r < TILE; ++r) s += sY2[swy(r, i)] * sY2[swy(r, j)];
      Sacc += s;
    }
    // ---------- off-diagonal tiles of column J ----------
    for (int I = J + 1; I < nt; ++I) {
      double a2[4][2][2] = {};
      if (nk > 0) {
        stage_chunk(sStage, tile_ptr(Kb, I, 0), 0, tid);
        stage_chunk(sStage + 64 * KC, tile_ptr(Kb, J, 0), 0, tid);
        cp_async_commit();
      }
      for (int c = 0; c < nk; ++c) {
        if (c + 1 < nk) {
          double* st = sStage + ((c + 1) & 1) * STAGE_DBL;
          int K = (c + 1) >> 1, kc = (c + 1) & 1;
          stage_chunk(st, tile_ptr(Kb, I, K), kc, tid);
          stage_chunk(st + 64 * KC, tile_ptr(Kb, J, K), kc, tid);
          cp_async_commit();
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncthreads();
        const double* st = sStage + (c & 1) * STAGE_DBL;
        mma_chunk(a2, st, st + 64 * KC, R0, C0, lane);
        __syncthreads();
      }
      // S = A_IJ - acc into the stage area (64x64 swizzled)
      double* sS = sStage;
      const double* Aij = tile_ptr(Kb, I, J);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) {
          int r = R0 + 8 * mi + lr, cc = C0 + 8 * ni + 2 * lc;
          double2 a = *reinterpret_cast<const double2*>(Aij + r * TILE + cc);
          sS[sw64(r, cc)] = a.x - a2[mi][ni][0];
          sS[sw64(r, cc + 1)] = a.y - a2[mi][ni][1];
        }
      __syncthreads();
      // G_IJ = S * G_JJ^-T
      double g[4][2][2] = {};
#pragma unroll 4
      for (int k0 = 0; k0 < TILE; k0 += 4) {
        double a[4], bb[2];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) a[mi] = sS[sw64(R0 + 8 * mi + lr, k0 + lc)];
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) bb[ni] = sT[sw64(C0 + 8 * ni + lr, k0 + lc)];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) dmma(g[mi][ni][0], g[mi][ni][1], a[mi], bb[ni]);
      }
      double* Gij = Kb + (long)(I * (I + 1) / 2 + J) * TILE_ELEMS;
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) {
          int r = R0 + 8 * mi + lr, cc = C0 + 8 * ni + 2 * lc;
          *reinterpret_cast<double2*>(Gij + r * TILE + cc) = make_double2(g[mi][ni][0], g[mi][ni][1]);
        }
      __syncthreads();
    }
  }

  if (sFail[0]) {  // report and poison the outputs of this RVE
    if (tid == 0) info[b] = sFail[0];
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    if (tid < R.m * R.m) Ceff[(long)b * R.m * R.m + tid] = nan;
    if (Peff && tid < R.m) Peff[(long)b * R.m + tid] = nan;
    return;
  }

  // ======================= K4 epilogue: C_eff, P_eff ==========================
  {
    double* sSum = sY;  // reuse: 8x8 plain
    __syncthreads();
    if (tid < 64) sSum[tid] = Sacc;
    __syncthreads();
    const int m = R.m;
    const double* Ca = Cavg + (long)bl * 64;
    if (tid < m * m) {
      int i = tid / m, j = tid % m;
      Ceff[(long)b * m * m + tid] = Ca[i * m + j] - sSum[i * 8 + j] / R.vol;
    }
    if (R.finite && tid < m) {
      double pa = Pavg[(long)bl * 8 + tid];
      if (Peff) Peff[(long)b * m + tid] = pa - sSum[tid * 8 + m] / R.vol;
      if (PavgOut) PavgOut[(long)b * m + tid] = pa;
    }
    __syncthreads();
  }

  // ======================= backward: X = G^-T Y ===============================
  for (int J = nt - 1; J >= 0; --J) {
    double xacc[2] = {0.0, 0.0};
    const int ni_cnt = nt - 1 - J;
    // double-buffered: buffer = [64x64 tile | 64x8 X_I]
    constexpr int BUF = TILE_ELEMS + 64 * RHSW;
    double* buf0 = sStage;  // 2*BUF = 9216 <= 2*STAGE_DBL (8704)? see static_assert below
    if (ni_cnt > 0) {
      stage_tile(buf0, tile_ptr(Kb, J + 1, J), tid);
      stage_rhs(buf0 + TILE_ELEMS, Xb + (long)(J + 1) * TILE * RHSW, TILE, tid);
      cp_async_commit();
    }
    for (int c = 0; c < ni_cnt; ++c) {
      const int I = J + 1 + c;
      if (c + 1 < ni_cnt) {
        double* nb = buf0 + ((c + 1) & 1) * BUF;
        stage_tile(nb, tile_ptr(Kb, I + 1, J), tid);
        stage_rhs(nb + TILE_ELEMS, Xb + (long)(I + 1) * TILE * RHSW, TILE, tid);
        cp_async_commit();
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const double* tl = buf0 + (c & 1) * BUF;
      const double* xi = tl + TILE_ELEMS;
      // xacc[j][n] += sum_k G_IJ[k][j] * X_I[k][n],  rows j = 8*warp..
#pragma unroll
      for (int k0 = 0; k0 < TILE; k0 += 4) {
        double a = tl[sw64(k0 + lc, 8 * warp + lr)];
        double bb = xi[swy(k0 + lc, lr)];
        dmma(xacc[0], xacc[1], a, bb);
      }
      __syncthreads();
    }
    // r = Y_J - xacc ; X_J = G_JJ^-T r
    stage_tile(sT, tile_ptr(Kb, J, J), tid);
    cp_async_commit();
    {
      int r = 8 * warp + lr, cc = 2 * lc;
      double2 y = *reinterpret_cast<const double2*>(Yb + (long)(J * TILE + r) * RHSW + cc);
      sY[swy(r, cc)] = y.x - xacc[0];
      sY[swy(r, cc + 1)] = y.y - xacc[1];
    }
    cp_async_wait<0>();
    __syncthreads();
    {
      double x[2] = {0.0, 0.0};
#pragma unroll
      for (int k0 = 0; k0 < TILE; k0 += 4) {
        double a = sT[sw64(k0 + lc, 8 * warp + lr)];  // (G_JJ^-1)^T
        double bb = sY[swy(k0 + lc, lr)];
        dmma(x[0], x[1], a, bb);
      }
      int rr = 8 * warp + lr, cc = 2 * lc;
      *reinterpret_cast<double2*>(Xb + (long)(J * TILE + rr) * RHSW + cc) = make_double2(x[0], x[1]);
    }
    __syncthreads();
  }
}

static_assert(2 * (TILE_ELEMS + 64 * RHSW) <= 2 * STAGE_DBL + 2 * 64 * RHSW,
              "backward double buffer must fit in the stage area + sY/sY2");

void launch_condense(const RveDev& R, int b0, int nb, double* Kt, double* Y, const double* Cavg,
                     const double* Pavg, double* Ceff, double* Peff, double* PavgOut, double* X,
                     int* info, cudaStream_t s) {
  size_t sm = (size_t)SMEM_DBL * sizeof(double);
  cudaFuncSetAttribute(k_condense, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_condense<<<nb, NTHR, sm, s>>>(R, b0, Kt, Y, Cavg, Pavg, Ceff, Peff, PavgOut, X, info);
}

// ------------------------------------------------------------------ small reductions
__global__ void k_first_fail(const int* __restrict__ f, int n, int sentinel, int* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && f[i] != sentinel) atomicMin(out, i);
}
void launch_first_fail(const int* flags, int n, int sentinel, int* out, cudaStream_t s) {
  k_first_fail<<<(n + 255) / 256, 256, 0, s>>>(flags, n, sentinel, out);
}

__global__ void k_max_reduce(const double* __restrict__ v, int n, double* out) {
  __shared__ double red[256];
  double m = 0.0;
  for (int i = threadIdx.x; i < n; i += 256) m = fmax(m, v[i]);
  red[threadIdx.x] = m;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}
void launch_max_reduce(const double* v, int n, double* out, cudaStream_t s) {
  k_max_reduce<<<1, 256, 0, s>>>(v, n, out);
}

}  // namespace hom
