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
#include <cuda.h>
#include <cstdlib>
#include <cudaTypedefs.h>

#include "hom_internal.cuh"

namespace hom {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
// -x by flipping the sign bit (integer op, keeps the FP64 pipe free for DMMA)
__device__ __forceinline__ double neg(double x) {
  return __longlong_as_double(__double_as_longlong(x) ^ (long long)0x8000000000000000ULL);
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---- TMA (cp.async.bulk.tensor) staging of the k-chunks, completion on mbarriers ----
__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(s_u32(bar)), "r"(parity)
                 : "memory");
}
// generic-proxy writes of this CTA (ordered by a preceding barrier) before async-proxy writes
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int r0, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          s_u32(dst)),
      "l"(map), "r"(c0), "r"(r0), "r"(s_u32(bar))
      : "memory");
}
// TMA 128-byte swizzle of a [rows][16] FP64 k-chunk (rows of 128 B, 16-byte units XOR row & 7)
__device__ __forceinline__ int swt(int r, int k) { return r * KC + ((((k >> 1) ^ (r & 7)) << 1) | (k & 1)); }

// swizzled word index inside a [rows][KC] k-chunk and a [rows][64] tile (row-chunk)
__device__ __forceinline__ int sw32(int r, int k) { return r * KC + (k ^ ((r & 3) << 2)); }
// k-chunk layout: TMA's 128-byte swizzle (dense, TMA-staged) or sw32 (tile-sparse, cp.async)
template <bool TS>
__device__ __forceinline__ int swk(int r, int k) { return TS ? swt(r, k) : sw32(r, k); }
__device__ __forceinline__ int sw64(int r, int c) { return r * TILE + (c ^ ((r & 3) << 2)); }
// Diagonal-tile buffer: only the 10 lower 16x16 blocks of the 64x64 tile, block (bi, bj <= bi) at
// (bi(bi+1)/2 + bj) * 256, each block row-major with the same XOR swizzle (2560 doubles instead of
// 4096 -> 4 CTAs per SM).  Callers never address a strictly upper block.
constexpr int SD_DBL = 10 * 256;
__device__ __forceinline__ int sd(int r, int c) {
  const int bi = r >> 4, bj = c >> 4;
  return (((bi * (bi + 1)) >> 1) + bj) * 256 + (r & 15) * 16 + ((c & 15) ^ ((r & 3) << 2));
}
__device__ __forceinline__ bool sd_upper(int r, int c) { return (c >> 4) > (r >> 4); }
// [rows][8] right-hand-side block
__device__ __forceinline__ int swy(int k, int n) { return k * RHSW + (n ^ (((k >> 1) & 1) << 2)); }

// Tile structure, MODE 0: every lower tile stored at the row-major lower slot I(I+1)/2 + J
// (dense; no lookups).  MODE 1: tile-sparse with nt <= 64, bitmasks in the kernel parameter
// space (TileMask).  MODE 2: tile-sparse, any nt, tables in global memory (g_nz, tslot).
template <int MODE>
__device__ __forceinline__ double* tile_ptr(double* Kb, const RveDev& R, const TileMask& tm, int I, int J) {
#ifdef HOM_DEBUG_BOUNDS
  HOM_DCHECK(I >= J && J >= 0 && I < R.nt);
  if (MODE == 2) HOM_DCHECK(__ldg(R.tslot + I * R.nt + J) >= 0 && __ldg(R.tslot + I * R.nt + J) < R.nslot);
  if (MODE == 1) HOM_DCHECK(((tm.row[I] >> J) & 1ull) && tm.rowstart[I] + __popcll(tm.row[I] & ((1ull << J) - 1ull)) < R.nslot);
  if (MODE == 0) HOM_DCHECK(((I * (I + 1)) >> 1) + J < R.nslot);
#endif
  if (MODE == 2) return Kb + (long)__ldg(R.tslot + I * R.nt + J) * TILE_ELEMS;
  if (MODE == 1) return Kb + (long)(tm.rowstart[I] + __popcll(tm.row[I] & ((1ull << J) - 1ull))) * TILE_ELEMS;
  return Kb + (long)(((I * (I + 1)) >> 1) + J) * TILE_ELEMS;
}
template <int MODE>
__device__ __forceinline__ int tile_slot(const RveDev& R, const TileMask& tm, int I, int J) {
  if (MODE == 2) return __ldg(R.tslot + I * R.nt + J);
  if (MODE == 1) return tm.rowstart[I] + __popcll(tm.row[I] & ((1ull << J) - 1ull));
  return ((I * (I + 1)) >> 1) + J;
}
// G(I,J) structurally nonzero
template <int MODE>
__device__ __forceinline__ bool gnz(const RveDev& R, const TileMask& tm, int I, int J) {
  if (MODE == 2) return __ldg(R.g_nz + I * R.nt + J);
  if (MODE == 1) return (tm.row[I] >> J) & 1ull;
  return true;
}
// first K' >= K, K' < J, with G(I,K') and G(J,K') both structurally nonzero (J if none)
template <int MODE>
__device__ __forceinline__ int next_pair(const RveDev& R, const TileMask& tm, int I, int J, int K) {
  if (MODE == 0 || K >= J) return K;
  if (MODE == 1) {
    const unsigned long long m = tm.row[I] & tm.row[J] & ((1ull << J) - 1ull) & (~0ull << K);
    return m ? __ffsll((long long)m) - 1 : J;
  } else {
    while (K < J && !(__ldg(R.g_nz + I * R.nt + K) && __ldg(R.g_nz + J * R.nt + K))) ++K;
    return K;
  }
}
// first I' >= I with G(I',J) structurally nonzero (nt if none)
template <int MODE>
__device__ __forceinline__ int next_row(const RveDev& R, const TileMask& tm, int J, int I) {
  if (MODE == 0 || I >= R.nt) return I;
  if (MODE == 1) {
    const unsigned long long m = tm.col[J] & (~0ull << I);
    return m ? min(__ffsll((long long)m) - 1, R.nt) : R.nt;
  } else {
    while (I < R.nt && !__ldg(R.g_nz + I * R.nt + J)) ++I;
    return I;
  }
}

// ------------------------------------------------------------------ CTA shape
// One CTA per RVE, 4 warps; each warp owns a 32x32 quadrant of a 64x64 output tile
// (16 independent DMMA accumulators, 8 fragment loads per 16 DMMAs).  ~72 KB of
// shared memory and <= 168 registers give 3 co-resident CTAs per SM: while one CTA
// is in the latency-bound pivot chain of its diagonal tile (one warp, 64 dependent
// rsqrt steps), the other two keep the FP64 tensor pipe busy
// (profiles/r01/ncu_v6_cfg2.md: 30% of samples were warps waiting on that chain).
constexpr int NTC = 128;          // threads per CTA
constexpr int CPT = TILE / KC;    // k-chunks per tile

// Phase timestamps for tools/condense_timing.cu only (HOM_TIMING build).
#ifdef HOM_TIMING
__device__ long long g_tm[64][40][8];
__device__ __forceinline__ long long clk_ordered() {
  long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
  return t;
}
#define TMARK(slot)                                                                   \
  do {                                                                                \
    if (blockIdx.x < 64 && J < 40 && threadIdx.x == 0) g_tm[blockIdx.x][J][slot] = clk_ordered(); \
  } while (0)
#define TMARK_T(slot, t)                                                                    \
  do {                                                                                      \
    if (blockIdx.x < 64 && J < 40 && threadIdx.x == (t)) g_tm[blockIdx.x][J][slot] = clk_ordered(); \
  } while (0)
#else
#define TMARK(slot) do {} while (0)
#define TMARK_T(slot, t) do {} while (0)
#endif

// Stage the [64][KC] k-chunk kc (columns kc*KC..) of a row-major 64x64 global tile into swizzled smem.
__device__ __forceinline__ void stage_chunk(double* dst, const double* src_tile, int kc, int tid) {
  constexpr int PPR = KC / 2;  // 16-byte pieces per row
#pragma unroll
  for (int i = 0; i < 64 * PPR / NTC; ++i) {
    int idx = tid + NTC * i;
    int r = idx / PPR, c2 = idx % PPR;
    cp_async16(dst + sw32(r, 2 * c2), src_tile + r * TILE + kc * KC + 2 * c2);
  }
}
// Stage rows [r0, r0+n) of a row-major 64x64 global tile into swizzled [n][64] smem (sw64, local rows).
__device__ __forceinline__ void stage_rows(double* dst, const double* src_tile, int r0, int n, int tid) {
  for (int idx = tid; idx < n * 32; idx += NTC) {
    int r = idx >> 5, c2 = idx & 31;
    cp_async16(dst + sw64(r, 2 * c2), src_tile + (r0 + r) * TILE + 2 * c2);
  }
}
// Stage rows [0, n) of an [.][8] RHS block into swizzled [n][8] smem.
__device__ __forceinline__ void stage_rhs(double* dst, const double* src, int n, int tid) {
  for (int idx = tid; idx < n * (RHSW / 2); idx += NTC) {
    int k = idx >> 2, c2 = idx & 3;
    cp_async16(dst + swy(k, 2 * c2), src + k * RHSW + 2 * c2);
  }
}

// ------------------------------------------------------------------ diagonal tile
// Cholesky of the 16x16 block at (k0,k0) of sD (lower part; lanes hold rows,
// shuffles only), then its inverse written over the block (zeros above the
// diagonal).  Returns the first failing local pivot (16 = none); warp-uniform.
__device__ __forceinline__ int chol16_inv_inplace(double* sD, int k0, int lane) {
  const unsigned FULL = 0xffffffffu;
  const int r = lane & 15;
  const int lr = lane >> 2, lc = lane & 3;
  double ip[16];
  int fail = 16;
  // Right-looking in four 4-column panels: the pivot chain and the in-panel updates on the
  // registers of lane r = row r (one rsqrt per pivot, every lane keeps 1/L_kk), the rank-4
  // update of the trailing rows/columns on DMMA (k = 4 = the panel) -- the FP64 pipe is shared
  // with the other CTAs' DMMA, so the chain is kept to as few FP64 instructions as possible.
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int c0 = 4 * p;
    double a[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) a[q] = (r >= c0 + q) ? sD[sd(k0 + r, k0 + c0 + q)] : 0.0;
#pragma unroll
    for (int k = 0; k < 4; k += 2) {
      // two pivots at a time: the 2x2 pivot block [A B; B C] gives L_kk = sqrt(A) and
      // L_k+1,k+1 = sqrt(det / A), det = AC - B^2 -- the two rsqrt are independent, so the chain
      // has one rsqrt level per two columns
      const double A = __shfl_sync(FULL, a[k], c0 + k);
      const double Bv = __shfl_sync(FULL, a[k], c0 + k + 1);
      const double Cv = __shfl_sync(FULL, a[k + 1], c0 + k + 1);
      const double det = fma(A, Cv, -(Bv * Bv));
      if (!(A > 0.0) && fail == 16) fail = c0 + k;
      if (!(det > 0.0) && fail == 16) fail = c0 + k + 1;
      const double ia = rsqrt(A), id = rsqrt(det);
      const double ip1 = (A * ia) * id;  // 1 / L_k+1,k+1 = sqrt(A) / sqrt(det)
      ip[c0 + k] = ia;
      ip[c0 + k + 1] = ip1;
      const double l10 = Bv * ia;  // L_k+1,k
      const double lk = a[k] * ia;  // column k of row r (row k: sqrt(A); row k+1: l10)
      const double lk1 = fma(-lk, l10, a[k + 1]) * ip1;  // column k+1 (row k+1: sqrt(det / A))
      a[k] = lk;
      if (r >= c0 + k + 1) a[k + 1] = lk1;
#pragma unroll
      for (int j = k + 2; j < 4; ++j) {
        const double ljk = __shfl_sync(FULL, a[k], c0 + j), ljk1 = __shfl_sync(FULL, a[k + 1], c0 + j);
        if (r >= c0 + j) a[j] = fma(-a[k], ljk, fma(-a[k + 1], ljk1, a[j]));
      }
    }
    if (lane < 16 && r >= c0) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (c0 + q <= r) sD[sd(k0 + r, k0 + c0 + q)] = a[q];
    }
    __syncwarp();
    if (p < 3) {  // trailing rows/cols >= c0 + 4: C -= L_panel L_panel^T (rows above masked to 0)
      const int t0 = c0 + 4;
#pragma unroll
      for (int blk = 0; blk < 3; ++blk) {
        const int bi = blk == 0 ? 0 : 1, bj = blk == 2 ? 1 : 0;
        if (8 * bi + 7 < t0 || 8 * bj + 7 < t0) continue;  // block outside the trailing part
        const int ra = 8 * bi + lr, rb = 8 * bj + lr;
        const double av = ra >= t0 ? neg(sD[sd(k0 + ra, k0 + c0 + lc)]) : 0.0;
        const double bv = rb >= t0 ? sD[sd(k0 + rb, k0 + c0 + lc)] : 0.0;
        const int cc = 8 * bj + 2 * lc;
        double c0v = sD[sd(k0 + ra, k0 + cc)], c1v = sD[sd(k0 + ra, k0 + cc + 1)];
        dmma(c0v, c1v, av, bv);
        __syncwarp();
        if (ra >= t0) {
          sD[sd(k0 + ra, k0 + cc)] = c0v;
          sD[sd(k0 + ra, k0 + cc + 1)] = c1v;
        }
      }
      __syncwarp();
    }
  }
  __syncwarp();
  // X = L^-1 blockwise (8x8 blocks): X00 = L00^-1 and X11 = L11^-1 together (lane c builds column
  // c & 7 of block c >> 3 by forward substitution, L rows read as smem broadcasts), then
  // X10 = -X11 (L10 X00) as two 8x8x8 DMMA products (T = L10 X00 is parked over L10).
  {
    const int c = lane & 15, bq = c >> 3, cb = c & 7, o = 8 * bq;
    double x[8];
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        if (k < rr) s0 = fma(sD[sd(k0 + o + rr, k0 + o + k)], x[k], s0);
        if (k + 1 < rr) s1 = fma(sD[sd(k0 + o + rr, k0 + o + k + 1)], x[k + 1], s1);
      }
      const double ipr = bq ? ip[8 + rr] : ip[rr];
      x[rr] = (rr >= cb) ? (((rr == cb) ? 1.0 : 0.0) - (s0 + s1)) * ipr : 0.0;
    }
    __syncwarp();
    if (lane < 16) {
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) {
        sD[sd(k0 + o + rr, k0 + c)] = x[rr];
        if (bq) sD[sd(k0 + rr, k0 + c)] = 0.0;  // strictly upper 8x8 block
      }
    }
    __syncwarp();
    double t0 = 0.0, t1 = 0.0;  // T = L10 X00 (rows 8..15, cols 0..7)
#pragma unroll
    for (int kk = 0; kk < 8; kk += 4)
      dmma(t0, t1, sD[sd(k0 + 8 + lr, k0 + kk + lc)], sD[sd(k0 + kk + lc, k0 + lr)]);
    __syncwarp();
    sD[sd(k0 + 8 + lr, k0 + 2 * lc)] = t0;
    sD[sd(k0 + 8 + lr, k0 + 2 * lc + 1)] = t1;
    __syncwarp();
    double y0 = 0.0, y1 = 0.0;  // X10 = -X11 T
#pragma unroll
    for (int kk = 0; kk < 8; kk += 4)
      dmma(y0, y1, neg(sD[sd(k0 + 8 + lr, k0 + 8 + kk + lc)]), sD[sd(k0 + 8 + kk + lc, k0 + lr)]);
    __syncwarp();
    sD[sd(k0 + 8 + lr, k0 + 2 * lc)] = y0;
    sD[sd(k0 + 8 + lr, k0 + 2 * lc + 1)] = y1;
  }
  __syncwarp();
  return fail;
}


// Blocked (16-wide) Cholesky of the SPD 64x64 tile in sD followed by the blocked
// triangular inverse, in place, by NW warps (warp index `warp` < NW; `sync` is their
// barrier): the 16x16 pivot blocks on warp 0 (registers + shuffles), panels, trailing
// updates and the off-diagonal inverse blocks on DMMA over the NW warps.  On return
// sD = G_JJ^-1 (lower, exact zeros above the diagonal: the caller zeroes the strict upper
// part).  sScr: 3 x 16x20.  Returns false (sFail set to the 1-based failing row of the RVE)
// on a non-positive pivot.  NW = 4: k_condense (all warps of the CTA); NW = 1: the factor
// warp of k_condense_ws, which runs this while the MMA warps accumulate the column's
// off-diagonal tiles.
struct NoSide {
  __device__ void operator()(int) const {}
};
template <int NW, typename Sync, typename Side = NoSide>
__device__ __forceinline__ bool factor_invert_diag(double* sD, double* sScr, int* sFail, int J, int warp,
                                                   int lane, Sync sync, Side side = Side()) {
  const int lr = lane >> 2, lc = lane & 3;
#pragma unroll 1
  for (int kb = 0; kb < 4; ++kb) {
    const int k0 = 16 * kb;
    if (warp == 0) {
      const int f = chol16_inv_inplace(sD, k0, lane);  // block (kb,kb) := L_kk^-1
      if (f < 16 && lane == 0) sFail[0] = J * TILE + k0 + f + 1;
    } else {
      side(kb);  // the other warps' work in the pivot-chain window (tile-sparse: diagonal lookahead)
    }
    sync();
    if (kb == 0) TMARK(5);
    if (sFail[0]) return false;
    if (kb == 3) break;
    const int rb0 = k0 + 16, nrt = (TILE - rb0) / 8;
    // panel: L_ik = A_ik X_kk^T (X_kk lower: col tile 0 needs k < 8 only); row tiles over warps
    if constexpr (NW == 1) {  // one warp: each row tile reads and then overwrites only its own rows
#pragma unroll 1
      for (int ti = 0; ti < nrt; ++ti) {
        const int r = rb0 + 8 * ti + lr;
        double q[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int kk = 0; kk < 16; kk += 4) {
          const double a = sD[sd(r, k0 + kk + lc)];
          if (kk < 8) dmma(q[0], q[1], a, sD[sd(k0 + lr, k0 + kk + lc)]);
          dmma(q[2], q[3], a, sD[sd(k0 + 8 + lr, k0 + kk + lc)]);
        }
        __syncwarp();
        sD[sd(r, k0 + 2 * lc)] = q[0];
        sD[sd(r, k0 + 2 * lc + 1)] = q[1];
        sD[sd(r, k0 + 8 + 2 * lc)] = q[2];
        sD[sd(r, k0 + 8 + 2 * lc + 1)] = q[3];
        __syncwarp();
      }
    } else {
      double p[2][4];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int ti = warp + NW * u;
        if (ti < nrt) {
          const int r = rb0 + 8 * ti + lr;
          p[u][0] = p[u][1] = p[u][2] = p[u][3] = 0.0;
#pragma unroll
          for (int kk = 0; kk < 16; kk += 4) {
            const double a = sD[sd(r, k0 + kk + lc)];
            if (kk < 8) dmma(p[u][0], p[u][1], a, sD[sd(k0 + lr, k0 + kk + lc)]);
            dmma(p[u][2], p[u][3], a, sD[sd(k0 + 8 + lr, k0 + kk + lc)]);
          }
        }
      }
      sync();
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int ti = warp + NW * u;
        if (ti < nrt) {
          const int r = rb0 + 8 * ti + lr;
          sD[sd(r, k0 + 2 * lc)] = p[u][0];
          sD[sd(r, k0 + 2 * lc + 1)] = p[u][1];
          sD[sd(r, k0 + 8 + 2 * lc)] = p[u][2];
          sD[sd(r, k0 + 8 + 2 * lc + 1)] = p[u][3];
        }
      }
      sync();
    }
    // trailing: A_ij -= L_ik L_jk^T on the lower 8x8 tiles of rows/cols rb0..63 (reads the
    // panel columns, writes disjoint columns: no hazard between warps)
    const int ntr = nrt * (nrt + 1) / 2;
    for (int t = warp; t < ntr; t += NW) {
      int ti = 0;
      while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
      const int tj = t - ti * (ti + 1) / 2;
      const int r = rb0 + 8 * ti, cb = rb0 + 8 * tj;
      double acc0 = sD[sd(r + lr, cb + 2 * lc)], acc1 = sD[sd(r + lr, cb + 2 * lc + 1)];
#pragma unroll
      for (int kk = 0; kk < 16; kk += 4)
        dmma(acc0, acc1, neg(sD[sd(r + lr, k0 + kk + lc)]), sD[sd(cb + lr, k0 + kk + lc)]);
      sD[sd(r + lr, cb + 2 * lc)] = acc0;
      sD[sd(r + lr, cb + 2 * lc + 1)] = acc1;
    }
    sync();
  }
  TMARK(6);
  // off-diagonal blocks of the inverse, in place, block rows i ascending:
  //   T_k = sum_{j=k}^{i-1} L_ij X_jk (all k < i in parallel; X_jk of rows j < i are final),
  //   X_ik = -X_ii T_k written over L_ik after every T_k is formed.
#pragma unroll 1
  for (int i = 1; i < 4; ++i) {
    const int ntile = 4 * i;  // (k, tr, tc)
    for (int t = warp; t < ntile; t += NW) {
      const int k = t >> 2, tr = (t >> 1) & 1, tc = t & 1;
      double t0 = 0.0, t1 = 0.0;
      for (int j = k; j < i; ++j) {
#pragma unroll
        for (int kk = 0; kk < 16; kk += 4) {
          if (j == k && tc == 1 && kk < 8) continue;  // X_kk[kk][8+n] = 0 for kk < 8
          dmma(t0, t1, sD[sd(16 * i + 8 * tr + lr, 16 * j + kk + lc)],
               sD[sd(16 * j + kk + lc, 16 * k + 8 * tc + lr)]);
        }
      }
      double* W = sScr + k * 320;
      W[(8 * tr + lr) * 20 + 8 * tc + 2 * lc] = t0;
      W[(8 * tr + lr) * 20 + 8 * tc + 2 * lc + 1] = t1;
    }
    sync();
    for (int t = warp; t < ntile; t += NW) {
      const int k = t >> 2, tr = (t >> 1) & 1, tc = t & 1;
      const double* W = sScr + k * 320;
      double o0 = 0.0, o1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < 16; kk += 4) {
        if (tr == 0 && kk >= 8) continue;  // X_ii lower
        dmma(o0, o1, neg(sD[sd(16 * i + 8 * tr + lr, 16 * i + kk + lc)]), W[(kk + lc) * 20 + 8 * tc + lr]);
      }
      const int r = 16 * i + 8 * tr + lr, cc = 16 * k + 8 * tc + 2 * lc;
      sD[sd(r, cc)] = o0;  // only X_ii and sScr are read in this phase: in-place write is safe
      sD[sd(r, cc + 1)] = o1;
    }
    sync();
  }
  return true;
}

// ------------------------------------------------------------------ MMA helpers
// acc[4][4][2] += (-A(64xKC chunk)) * B(64xKC chunk)^T for the warp quadrant (R0, C0): acc starts
// as the original tile, so the result is A_IJ - sum_K G_IK G_JK^T.  DIAG: skip the 8x8 blocks
// strictly above the diagonal (the upper half is never used; frees the pipe for the other CTAs).
template <bool DIAG, bool TS>
__device__ __forceinline__ void mma_chunk(double (&acc)[4][4][2], const double* sA, const double* sB,
                                          int R0, int C0, int lane) {
  if (DIAG && C0 > R0 + 24) return;  // quadrant entirely above the diagonal
  const int lr = lane >> 2, lc = lane & 3;
#pragma unroll
  for (int k0 = 0; k0 < KC; k0 += 4) {
    double a[4], b[4];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) a[mi] = neg(sA[swk<TS>(R0 + 8 * mi + lr, k0 + lc)]);
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = sB[swk<TS>(C0 + 8 * ni + lr, k0 + lc)];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
        if (!DIAG || C0 + 8 * ni <= R0 + 8 * mi) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
  }
}

// Diagonal tile S_JJ = A_JJ - sum_K G_JK G_JK^T balanced over the 4 warps: warp W owns the lower
// 8x8 blocks of block rows W and 7-W (9 blocks each; 32x32 quadrants would give 16/10/10/0).
// A and B fragments of a chunk are the same words (G_JK against itself): 8-W loads per k-step.
template <int W>
__device__ __forceinline__ void diag_load(double (&acc)[9][2], const double* T, int lane) {
  const int lr = lane >> 2, lc = lane & 3;
  int t = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = h ? 7 - W : W;
#pragma unroll
    for (int c = 0; c <= r; ++c, ++t) {
      const double2 v = __ldcg(reinterpret_cast<const double2*>(T + (8 * r + lr) * TILE + 8 * c + 2 * lc));
      acc[t][0] = v.x;
      acc[t][1] = v.y;
    }
  }
}
template <int W, bool TS>
__device__ __forceinline__ void diag_chunk(double (&acc)[9][2], const double* sA, int lane) {
  const int lr = lane >> 2, lc = lane & 3;
#pragma unroll
  for (int k0 = 0; k0 < KC; k0 += 4) {
    double b[8 - W];
#pragma unroll
    for (int c = 0; c < 8 - W; ++c) b[c] = sA[swk<TS>(8 * c + lr, k0 + lc)];
    const double a0 = neg(b[W]), a1 = neg(b[7 - W]);
    int t = 0;
#pragma unroll
    for (int c = 0; c <= W; ++c, ++t) dmma(acc[t][0], acc[t][1], a0, b[c]);
#pragma unroll
    for (int c = 0; c <= 7 - W; ++c, ++t) dmma(acc[t][0], acc[t][1], a1, b[c]);
  }
}
// sT = lower(S_JJ): exact zeros above the diagonal inside the stored 16x16 blocks
template <int W>
__device__ __forceinline__ void diag_store(const double (&acc)[9][2], double* sT, int lane) {
  const int lr = lane >> 2, lc = lane & 3;
  int t = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = h ? 7 - W : W, row = 8 * r + lr;
#pragma unroll
    for (int c = 0; c <= r; ++c, ++t) {
      const int cc = 8 * c + 2 * lc;
      sT[sd(row, cc)] = (c < r || cc <= row) ? acc[t][0] : 0.0;
      sT[sd(row, cc + 1)] = (c < r || cc + 1 <= row) ? acc[t][1] : 0.0;
    }
  }
  const int row = 16 * W + lr, cc = 16 * W + 8 + 2 * lc;  // upper 8x8 half of diagonal block W
  sT[sd(row, cc)] = 0.0;
  sT[sd(row, cc + 1)] = 0.0;
}
#define DIAG_DISPATCH(fn, ...)           \
  switch (warp) {                        \
    case 0: fn<0>(__VA_ARGS__); break;   \
    case 1: fn<1>(__VA_ARGS__); break;   \
    case 2: fn<2>(__VA_ARGS__); break;   \
    default: fn<3>(__VA_ARGS__); break;  \
  }

// acc := this thread's accumulator-layout fragment of the quadrant of a row-major 64x64 global tile
__device__ __forceinline__ void load_frag(double (&acc)[4][4][2], const double* T, int R0, int C0, int lane) {
  const int lr = lane >> 2, lc = lane & 3;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      double2 v = __ldcg(reinterpret_cast<const double2*>(T + (R0 + 8 * mi + lr) * TILE + C0 + 8 * ni + 2 * lc));
      acc[mi][ni][0] = v.x;
      acc[mi][ni][1] = v.y;
    }
}

// ------------------------------------------------------------------ diagonal lookahead (tile-sparse)
// While warp 0 runs the pivot chain of diagonal tile J, warps 1-3 accumulate the first k-chunks of the
// NEXT column's diagonal step, S_J+1,J+1 = A_J+1,J+1 - sum_K G_J+1,K G_J+1,K^T and
// yacc_J+1 = sum_K G_J+1,K Y_K over the structurally nonzero K < J (final; K = J needs tile (J+1, J) of
// this column).  The partial sums are parked in place -- the pool slot of tile (J+1, J+1) and the X rows
// of tile row J+1 (written only by the backward pass) -- and the diagonal step of column J+1 continues
// from them with the remaining chunks: the same DMMAs in the same order, so the result is bitwise the
// one without the lookahead (and the dense path's).  Warp W = warp - 1 owns the lower 8x8 block rows
// {7, 3}, {6, 4} or {5, 2, 1, 0} (12 blocks each) and the same RHS rows; chunks are staged by 16-byte
// cp.async of the three warps into stage 1 (idle during the factor of the tile-sparse modes) and a
// 2 x [KC][8] area after sY, buffer reuse ordered by a named barrier of the three warps.
// (The dense path measured slower with it: there the co-resident CTAs already fill
// the pivot-chain windows.)
__device__ __forceinline__ void nbar_sync96() { asm volatile("bar.sync 1, 96;" ::: "memory"); }
template <int W>
__device__ __forceinline__ int la_row(int i) {
  return W == 0 ? (i == 0 ? 7 : 3) : W == 1 ? (i == 0 ? 6 : 4) : (i == 0 ? 5 : 3 - i);
}
// chunks of the lookahead of column J: 4 per structurally nonzero K < J of row J + 1, at most 4 la_q
template <int MODE>
__device__ __forceinline__ int la_count(const RveDev& R, const TileMask& tm, int J, int nt, int la_q) {
  if (MODE == 0 || la_q <= 0 || J < 1 || J + 1 >= nt) return 0;
  int n = 0;
  for (int K = next_pair<MODE>(R, tm, J + 1, J + 1, 0); K < J && n < 4 * la_q;
       K = next_pair<MODE>(R, tm, J + 1, J + 1, K + 1))
    n += CPT;
  return n;
}
// chunks [c0, c1) of the lookahead; (K, kc) = the position of chunk c0 on entry, of chunk c1 on return
template <int W, int MODE>
__device__ __forceinline__ void la_run(const RveDev& R, const TileMask& tm, double* Kb, const double* Yb,
                                       double* Xb, int J, int c0, int c1, int& K, int& kc, double* sG,
                                       double* sYl, int tid, int lane) {
  constexpr int NR = W == 2 ? 4 : 2, NB = W == 0 ? 8 : (W == 1 ? 7 : 6);
  const int lr = lane >> 2, lc = lane & 3, t96 = tid - 32;
  double* Tn = tile_ptr<MODE>(Kb, R, tm, J + 1, J + 1);
  double* Xn = Xb + (long)(J + 1) * TILE * RHSW;
  double d[12][2], y[NR][2];
  {
    int t = 0;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const int r = la_row<W>(i);
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c <= r) {
          const double2 v = __ldcg(reinterpret_cast<const double2*>(Tn + (8 * r + lr) * TILE + 8 * c + 2 * lc));
          d[t][0] = v.x;
          d[t][1] = v.y;
          ++t;
        }
      if (c0 > 0) {
        const double2 v = __ldcg(reinterpret_cast<const double2*>(Xn + (8 * r + lr) * RHSW + 2 * lc));
        y[i][0] = v.x;
        y[i][1] = v.y;
      } else {
        y[i][0] = y[i][1] = 0.0;
      }
    }
  }
  auto issue = [&](int bf, int K, int kc) {  // G_J+1,K chunk kc + Y_K rows, the three warps
    double* dg = sG + bf * 64 * KC;
    const double* src = tile_ptr<MODE>(Kb, R, tm, J + 1, K);
    for (int idx = t96; idx < 64 * (KC / 2); idx += 96) {
      const int r = idx / (KC / 2), c2 = idx % (KC / 2);
      cp_async16(dg + sw32(r, 2 * c2), src + r * TILE + kc * KC + 2 * c2);
    }
    double* dy = sYl + bf * KC * RHSW;
    const double* ys = Yb + (long)(K * TILE + kc * KC) * RHSW;
    for (int idx = t96; idx < KC * (RHSW / 2); idx += 96) {
      const int k = idx >> 2, c2 = idx & 3;
      cp_async16(dy + swy(k, 2 * c2), ys + k * RHSW + 2 * c2);
    }
    cp_async_commit();
  };
  issue(c0 & 1, K, kc);
#pragma unroll 1
  for (int c = c0; c < c1; ++c) {
    int K2 = K, kc2 = kc + 1;
    if (kc2 == CPT) { kc2 = 0; K2 = next_pair<MODE>(R, tm, J + 1, J + 1, K + 1); }
    if (c + 1 < c1) { issue((c + 1) & 1, K2, kc2); cp_async_wait<1>(); }
    else cp_async_wait<0>();
    nbar_sync96();  // every thread's copies of chunk c landed
    const double* st = sG + (c & 1) * 64 * KC;
    const double* sy = sYl + (c & 1) * KC * RHSW;
#pragma unroll
    for (int k0 = 0; k0 < KC; k0 += 4) {
      double b[NB];
#pragma unroll
      for (int cc = 0; cc < NB; ++cc) b[cc] = st[sw32(8 * cc + lr, k0 + lc)];
      const double bb = sy[swy(k0 + lc, lr)];
      int t = 0;
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        const int r = la_row<W>(i);
        const double a = neg(b[r]);
#pragma unroll
        for (int cc = 0; cc < 8; ++cc)
          if (cc <= r) { dmma(d[t][0], d[t][1], a, b[cc]); ++t; }
        dmma(y[i][0], y[i][1], b[r], bb);  // yacc += G Y as in the diagonal step
      }
    }
    nbar_sync96();  // the buffer of chunk c may be refilled (chunk c + 2)
    K = K2;
    kc = kc2;
  }
  {
    int t = 0;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const int r = la_row<W>(i);
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c <= r) {
          __stcg(reinterpret_cast<double2*>(Tn + (8 * r + lr) * TILE + 8 * c + 2 * lc), make_double2(d[t][0], d[t][1]));
          ++t;
        }
      __stcg(reinterpret_cast<double2*>(Xn + (8 * r + lr) * RHSW + 2 * lc), make_double2(y[i][0], y[i][1]));
    }
  }
}

// Smem (doubles): sT (packed lower 16x16 blocks) | stage[2] x (A 64xKC + B 64xKC + Yc KCx8) | misc.
// The stage area doubles as: factor scratch (3 x 16x20 at 0), Y_J (64x8 at 0), Kfe_J - sum (64x8
// at SY_F, forward) / Y_J - xacc (at SY_B, backward), the full S_IJ tile of the TRSM (64x64) and
// the backward row chunks -- never two of them at the same time.
constexpr int STAGE_DBL = 2 * 64 * KC + KC * RHSW;
constexpr int SY_F = 1024, SY_B = 3456;
constexpr int SMEM_DBL = SD_DBL + 2 * STAGE_DBL + 64;
static_assert(SMEM_DBL * 8 + 1024 <= 57 * 1024, "four CTAs per SM");
static_assert(3 * 320 <= SY_F && SY_F + 64 * RHSW <= 2 * STAGE_DBL, "forward stage-area aliases");
static_assert(STAGE_DBL + 16 * TILE + 16 * RHSW <= SY_B && SY_B + 64 * RHSW <= 2 * STAGE_DBL, "backward aliases");
static_assert(TILE_ELEMS <= 2 * STAGE_DBL, "S tile fits in the stage area");
static_assert(16 * TILE + 16 * RHSW <= STAGE_DBL, "backward row chunk fits in a stage");

// ------------------------------------------------------------------ kernel
template <int MODE>
__global__ void __launch_bounds__(NTC, 4)
k_condense(RveDev R, const __grid_constant__ TileMask tm, const __grid_constant__ CUtensorMap kmap,
           const __grid_constant__ CUtensorMap ymap, int b0, double* __restrict__ Kt, double* __restrict__ Y,
           const double* __restrict__ Cavg, const double* __restrict__ Pavg,
           double* __restrict__ Ceff, double* __restrict__ Peff, double* __restrict__ PavgOut,
           double* __restrict__ X, int* __restrict__ info, int la_q) {
  extern __shared__ __align__(1024) double smem[];
  double* sT = smem;                        // packed lower 64x64 (sd): S_JJ -> G_JJ^-1
  double* sStage = sT + SD_DBL;             // 2 stages | S tile | factor scratch | Y_J | sY
  double* sY = sStage + SY_F;               // 64x8 swizzled: Kfe_J - sum_K G_JK Y_K (forward)
  int* sFail = reinterpret_cast<int*>(sStage + 2 * STAGE_DBL);
  double* sY2 = sStage;                     // Y_J (after the factorisation, before the off-diagonal tiles)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  const int R0 = (warp >> 1) * 32, C0 = (warp & 1) * 32;  // accumulation quadrant
  const int cLo = warp, cHi = 7 - warp;                    // TRSM column-block pair (balanced)
  const int bl = blockIdx.x, b = b0 + bl;
  const int nt = R.nt, NT = R.NT;
  double* Kb = Kt + (long)bl * R.nslot * TILE_ELEMS;
  double* Yb = Y + (long)bl * NT * RHSW;
  double* Xb = X + (long)(b - R.xb0) * NT * RHSW;  // X holds the context's local RVE range only

  // two k-chunk stages filled by TMA: full[s] completes when the stage's bytes have landed
  uint64_t* full = reinterpret_cast<uint64_t*>(sStage + 2 * STAGE_DBL + 8);
  uint32_t ph0 = 0, ph1 = 0;  // parity of the next completion of full[0], full[1]
  if (tid == 0) {
    sFail[0] = 0;
    sFail[3] = 0;  // tile-sparse lookahead: chunks parked for the next column (none yet)
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto wait_stage = [&](int st) {
    if (st == 0) { mbar_wait(&full[0], ph0); ph0 ^= 1u; }
    else { mbar_wait(&full[1], ph1); ph1 ^= 1u; }
  };
  // k-chunks: TMA + mbarriers for the dense structure (long pipelines); 16-byte cp.async for the
  // tile-sparse modes (one or two chunks per tile: the TMA round trip measured slower there)
  constexpr bool TMA_STAGING = MODE == 0;
  const long krow0 = (long)bl * R.nslot * TILE;  // first pool row of this RVE (kmap rows)
  const long yrow0 = (long)bl * NT;              // first Y row of this RVE (ymap rows)
  // Schur sum S = sum_J Y_J^T Y_J (8x8) on DMMA by warp 0: lane (lr, lc) holds S[lr][2lc], S[lr][2lc+1]
  double Sacc0 = 0.0, Sacc1 = 0.0;

  // ======================= forward: factor + Y ==============================
  for (int J = 0; J < nt; ++J) {
    TMARK(0);
    // ---------- S_JJ = A_JJ - sum_K G_JK G_JK^T ; yacc = sum_K G_JK Y_K ----------
    // k-chunks (K, kc) run over the K < J with G_JK != 0, two-stage cp.async pipeline
    {
      double dacc[9][2];
      double yacc[2][2] = {};
      DIAG_DISPATCH(diag_load, dacc, tile_ptr<MODE>(Kb, R, tm, J, J), lane);
      int K = next_pair<MODE>(R, tm, J, J, 0), kc = 0, par = 0;
      if (MODE != 0 && sFail[3] > 0) {  // the lookahead of column J - 1 accumulated chunks; resume after them
        {
          K = sFail[2];
          kc = 0;
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const double2 v = __ldcg(reinterpret_cast<const double2*>(
                Xb + (long)(J * TILE + 16 * warp + 8 * u + lr) * RHSW + 2 * lc));
            yacc[u][0] = v.x;
            yacc[u][1] = v.y;
          }
        }
      }
      auto issue_d = [&](int stg, int KK, int kcc) {  // G_JK chunk kcc + Y_K rows, one thread
        double* st = sStage + stg * STAGE_DBL;
        fence_proxy_async();
        mbar_expect(&full[stg], (64 * KC + KC * RHSW) * 8);
        tma_load_2d(st, &kmap, kcc * KC, (int)(krow0 + (long)tile_slot<MODE>(R, tm, J, KK) * TILE), &full[stg]);
        tma_load_2d(st + 2 * 64 * KC, &ymap, 0, (int)(yrow0 + KK * TILE + kcc * KC), &full[stg]);
      };
      auto stage_d = [&](int stg, int KK, int kcc) {  // cp.async variant (tile-sparse modes)
        double* st = sStage + stg * STAGE_DBL;
        stage_chunk(st, tile_ptr<MODE>(Kb, R, tm, J, KK), kcc, tid);
        stage_rhs(st + 2 * 64 * KC, Yb + (long)(KK * TILE + kcc * KC) * RHSW, KC, tid);
        cp_async_commit();
      };
      if (K < J) {
        if (TMA_STAGING) { if (tid == 0) issue_d(0, K, 0); }
        else stage_d(0, K, 0);
      }
      while (K < J) {
        int K2 = K, kc2 = kc + 1;
        if (kc2 == CPT) { kc2 = 0; K2 = next_pair<MODE>(R, tm, J, J, K + 1); }
        if (TMA_STAGING) {
          if (K2 < J && tid == 0) issue_d(par ^ 1, K2, kc2);
          wait_stage(par);
        } else {
          if (K2 < J) { stage_d(par ^ 1, K2, kc2); cp_async_wait<1>(); }
          else cp_async_wait<0>();
          __syncthreads();
        }
        const double* st = sStage + par * STAGE_DBL;
        switch (warp) {
          case 0: diag_chunk<0, TMA_STAGING>(dacc, st, lane); break;
          case 1: diag_chunk<1, TMA_STAGING>(dacc, st, lane); break;
          case 2: diag_chunk<2, TMA_STAGING>(dacc, st, lane); break;
          default: diag_chunk<3, TMA_STAGING>(dacc, st, lane); break;
        }
        const double* sYc = st + 2 * 64 * KC;  // yacc rows 16*warp.. (2 blocks) x 8 RHS columns
#pragma unroll
        for (int k0 = 0; k0 < KC; k0 += 4) {
          // TMA chunk unswizzled [KC][8]; cp.async chunk in the swy layout
          const double bb = TMA_STAGING ? sYc[(k0 + lc) * RHSW + lr] : sYc[swy(k0 + lc, lr)];
#pragma unroll
          for (int u = 0; u < 2; ++u)
            dmma(yacc[u][0], yacc[u][1], st[swk<TMA_STAGING>(16 * warp + 8 * u + lr, k0 + lc)], bb);
        }
        __syncthreads();
        K = K2; kc = kc2; par ^= 1;
      }
      DIAG_DISPATCH(diag_store, dacc, sT, lane);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int r = 16 * warp + 8 * u + lr, cc = 2 * lc;
        const double2 y = __ldcg(reinterpret_cast<const double2*>(Yb + (long)(J * TILE + r) * RHSW + cc));
        sY[swy(r, cc)] = y.x - yacc[u][0];
        sY[swy(r, cc + 1)] = y.y - yacc[u][1];
      }
    }
    __syncthreads();
    TMARK(1);
    // dense (TMA): the first chunk of the first off-diagonal tile (J+1, J) is fetched into stage 1
    // now -- stage 1 is untouched by the factor and Y phases -- so it lands under the pivot chain
    const bool pre_o = TMA_STAGING && J > 0 && J + 1 < nt;
    if (pre_o && tid == 0) {
      double* st = sStage + STAGE_DBL;
      fence_proxy_async();
      mbar_expect(&full[1], 2 * 64 * KC * 8);
      tma_load_2d(st, &kmap, 0, (int)(krow0 + (long)tile_slot<MODE>(R, tm, J + 1, 0) * TILE), &full[1]);
      tma_load_2d(st + 64 * KC, &kmap, 0, (int)(krow0 + (long)tile_slot<MODE>(R, tm, J, 0) * TILE), &full[1]);
    }
    // ---------- blocked Cholesky + inverse of the diagonal tile ----------
    // tile-sparse lookahead of column J + 1's diagonal step (warps 1-3, pivot-chain windows); the resume
    // point (K after the last chunk, chunk count) for column J + 1 goes to sFail[2], sFail[3]
    if (MODE != 0 && tid == 0) sFail[3] = 0;  // phase A of this column has read it (barrier above)
    int LAc = -1, laK = 0, lakc = 0;
    auto side = [&](int kb) {
      if (MODE == 0) return;
      if (LAc < 0) {
        LAc = la_count<MODE>(R, tm, J, nt, la_q);
        laK = next_pair<MODE>(R, tm, J + 1, J + 1, 0);
      }
      const int c0 = (LAc * kb) >> 2, c1 = (LAc * (kb + 1)) >> 2;
      if (c0 >= c1) return;
      double* sLaG = sStage + STAGE_DBL;         // 2 x [64][KC] in stage 1
      double* sLaY = sStage + SY_F + 64 * RHSW;  // 2 x [KC][8] after sY
      switch (warp) {
        case 1: la_run<0, MODE>(R, tm, Kb, Yb, Xb, J, c0, c1, laK, lakc, sLaG, sLaY, tid, lane); break;
        case 2: la_run<1, MODE>(R, tm, Kb, Yb, Xb, J, c0, c1, laK, lakc, sLaG, sLaY, tid, lane); break;
        default: la_run<2, MODE>(R, tm, Kb, Yb, Xb, J, c0, c1, laK, lakc, sLaG, sLaY, tid, lane); break;
      }
      if (c1 == LAc && tid == 32) { sFail[2] = laK; sFail[3] = LAc; }
    };
    if (!factor_invert_diag<4>(sT, sStage, sFail, J, warp, lane, [] { __syncthreads(); }, side)) {
      if (pre_o) wait_stage(1);  // no TMA left in flight into this CTA's shared memory
      break;
    }
    TMARK(2);
    // ---------- Y_J = G_JJ^-1 (Kfe_J - sum) ; S += Y_J^T Y_J ; store G_JJ^-1 ----------
    {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int r = 16 * warp + 8 * u;
        double y0 = 0.0, y1 = 0.0;
        for (int k0 = 0; k0 < r + 8; k0 += 4)  // G_JJ^-1 lower
          dmma(y0, y1, sT[sd(r + lr, k0 + lc)], sY[swy(k0 + lc, lr)]);
        const int rr = r + lr, cc = 2 * lc;
        sY2[swy(rr, cc)] = y0;
        sY2[swy(rr, cc + 1)] = y1;
        *reinterpret_cast<double2*>(Yb + (long)(J * TILE + rr) * RHSW + cc) = make_double2(y0, y1);
      }
      double* Gjj = tile_ptr<MODE>(Kb, R, tm, J, J);
      for (int idx = tid; idx < TILE_ELEMS / 2; idx += NTC) {
        const int r = idx >> 5, cc = 2 * (idx & 31);
        *reinterpret_cast<double2*>(Gjj + r * TILE + cc) =
            sd_upper(r, cc) ? make_double2(0.0, 0.0) : make_double2(sT[sd(r, cc)], sT[sd(r, cc + 1)]);
      }
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int k0 = 0; k0 < TILE; k0 += 4)  // A = Y_J^T (8 x 64), B' = Y_J^T (rows j, k = r)
        dmma(Sacc0, Sacc1, sY2[swy(k0 + lc, lr)], sY2[swy(k0 + lc, lr)]);
    }
    __syncthreads();  // sY2 (stage area) free again
    TMARK(3);
    // ---------- off-diagonal tiles of column J: S_IJ, then G_IJ = S_IJ G_JJ^-T ----------
    for (int I = J + 1; I < nt; ++I) {
      if (!gnz<MODE>(R, tm, I, J)) continue;  // structurally zero tile of G (tile-sparse path)
      double acc[4][4][2];
      double* Aij = tile_ptr<MODE>(Kb, R, tm, I, J);
      if (__ldg(R.tile_nz + I * nt + J)) {
        load_frag(acc, Aij, R0, C0, lane);
      } else {  // fill tile: A_IJ = 0 (never written by K1)
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
      }
      int K = next_pair<MODE>(R, tm, I, J, 0), kc = 0, par = 0;
      const bool prefetched = pre_o && I == J + 1;  // chunk (K = 0, kc = 0) already in stage 1
      if (prefetched) par = 1;
      auto issue_o = [&](int stg, int KK, int kcc) {  // G_IK and G_JK chunks kcc, one thread
        double* st = sStage + stg * STAGE_DBL;
        fence_proxy_async();
        mbar_expect(&full[stg], 2 * 64 * KC * 8);
        tma_load_2d(st, &kmap, kcc * KC, (int)(krow0 + (long)tile_slot<MODE>(R, tm, I, KK) * TILE), &full[stg]);
        tma_load_2d(st + 64 * KC, &kmap, kcc * KC, (int)(krow0 + (long)tile_slot<MODE>(R, tm, J, KK) * TILE),
                    &full[stg]);
      };
      auto stage_o = [&](int stg, int KK, int kcc) {  // cp.async variant (tile-sparse modes)
        double* st = sStage + stg * STAGE_DBL;
        stage_chunk(st, tile_ptr<MODE>(Kb, R, tm, I, KK), kcc, tid);
        stage_chunk(st + 64 * KC, tile_ptr<MODE>(Kb, R, tm, J, KK), kcc, tid);
        cp_async_commit();
      };
      if (K < J && !prefetched) {
        if (TMA_STAGING) { if (tid == 0) issue_o(0, K, 0); }
        else stage_o(0, K, 0);
      }
      while (K < J) {
        int K2 = K, kc2 = kc + 1;
        if (kc2 == CPT) { kc2 = 0; K2 = next_pair<MODE>(R, tm, I, J, K + 1); }
        if (TMA_STAGING) {
          if (K2 < J && tid == 0) issue_o(par ^ 1, K2, kc2);
          wait_stage(par);
        } else {
          if (K2 < J) { stage_o(par ^ 1, K2, kc2); cp_async_wait<1>(); }
          else cp_async_wait<0>();
          __syncthreads();
        }
        const double* st = sStage + par * STAGE_DBL;
        mma_chunk<false, TMA_STAGING>(acc, st, st + 64 * KC, R0, C0, lane);
        __syncthreads();
        K = K2; kc = kc2; par ^= 1;
      }
      // S_IJ into the stage area (full 64x64, sw64)
      double* sS = sStage;
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
          const int r = R0 + 8 * mi + lr, cc = C0 + 8 * ni + 2 * lc;
          sS[sw64(r, cc)] = acc[mi][ni][0];
          sS[sw64(r, cc + 1)] = acc[mi][ni][1];
        }
      __syncthreads();
      // G_IJ = S_IJ (G_JJ^-1)^T: warp owns column blocks cLo, cHi (all rows); G_JJ^-1 lower, so
      // column block c needs k < 8(c+1): 72 k-steps per warp for every warp.
      double g[8][2][2] = {};
      int k0 = 0;
      for (; k0 < 8 * (cLo + 1); k0 += 4) {
        const double bl0 = sT[sd(8 * cLo + lr, k0 + lc)], bh0 = sT[sd(8 * cHi + lr, k0 + lc)];
#pragma unroll
        for (int mi = 0; mi < 8; ++mi) {
          const double a = sS[sw64(8 * mi + lr, k0 + lc)];
          dmma(g[mi][0][0], g[mi][0][1], a, bl0);
          dmma(g[mi][1][0], g[mi][1][1], a, bh0);
        }
      }
      for (; k0 < 8 * (cHi + 1); k0 += 4) {
        const double bh0 = sT[sd(8 * cHi + lr, k0 + lc)];
#pragma unroll
        for (int mi = 0; mi < 8; ++mi) dmma(g[mi][1][0], g[mi][1][1], sS[sw64(8 * mi + lr, k0 + lc)], bh0);
      }
      double* Gij = Aij;
#pragma unroll
      for (int mi = 0; mi < 8; ++mi) {
        const int r = 8 * mi + lr;
        *reinterpret_cast<double2*>(Gij + r * TILE + 8 * cLo + 2 * lc) = make_double2(g[mi][0][0], g[mi][0][1]);
        *reinterpret_cast<double2*>(Gij + r * TILE + 8 * cHi + 2 * lc) = make_double2(g[mi][1][0], g[mi][1][1]);
      }
      __syncthreads();
    }
    TMARK(4);
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
    double* sSum = sStage;  // reuse: 8x8 plain
    __syncthreads();
    if (warp == 0) {
      sSum[lr * 8 + 2 * lc] = Sacc0;
      sSum[lr * 8 + 2 * lc + 1] = Sacc1;
    }
    __syncthreads();
    const int m = R.m;
    const double* Ca = Cavg + (long)bl * 64;
    if (tid < m * m) {
      const int i = tid / m, j = tid % m;
      Ceff[(long)b * m * m + tid] = Ca[i * m + j] - sSum[i * 8 + j] / R.vol;
    }
    if (R.finite && tid < m) {
      const double pa = Pavg[(long)bl * 8 + tid];
      if (Peff) Peff[(long)b * m + tid] = pa - sSum[tid * 8 + m] / R.vol;
      if (PavgOut) PavgOut[(long)b * m + tid] = pa;
    }
    __syncthreads();
  }

  // ======================= backward: X = G^-T Y ===============================
  // xacc[j][n] = sum_{I>J} sum_k G_IJ[k][j] X_I[k][n], streamed in 16-row chunks of G_IJ;
  // warp owns rows j = 16*warp .. +15 (2 blocks).
#ifdef HOM_TIMING
  if (blockIdx.x < 64 && threadIdx.x == 0) g_tm[blockIdx.x][39][0] = clk_ordered();
#endif
  constexpr int RC = 16, RPT = TILE / RC;
  constexpr int NSTB = 4, BST = RC * TILE + RC * RHSW;  // backward stages (doubles each)
  static_assert(NSTB * BST <= SD_DBL + SY_B, "backward stages overlap sY");
  auto next_row = [&](int J, int I) { return hom::next_row<MODE>(R, tm, J, I); };
  for (int J = nt - 1; J >= 0; --J) {
    double xacc[2][2] = {};
    // 16-row chunks (I, rq) of the G_IJ column, NSTB-deep cp.async pipeline in the diagonal-tile
    // buffer + stage area (sT is reloaded with G_JJ^-1 only after the chunks; sY at SY_B is free)
    int I = next_row(J, J + 1), rq = 0;
    int nis = 0, ncon = 0;
    auto issue_b = [&]() {
      double* nb = smem + (nis % NSTB) * BST;
      stage_rows(nb, tile_ptr<MODE>(Kb, R, tm, I, J), rq * RC, RC, tid);
      stage_rhs(nb + RC * TILE, Xb + (long)(I * TILE + rq * RC) * RHSW, RC, tid);
      cp_async_commit();
      ++nis;
      if (++rq == RPT) { rq = 0; I = next_row(J, I + 1); }
    };
    while (nis < NSTB - 1 && I < nt) issue_b();
    while (ncon < nis) {
      if (I < nt) {
        issue_b();
        cp_async_wait<NSTB - 1>();
      } else {
        const int ahead = nis - ncon - 1;  // groups allowed to stay in flight
        if (ahead >= 2) cp_async_wait<2>();
        else if (ahead == 1) cp_async_wait<1>();
        else cp_async_wait<0>();
      }
      __syncthreads();
      const double* tl = smem + (ncon % NSTB) * BST;
      const double* xi = tl + RC * TILE;
#pragma unroll
      for (int k0 = 0; k0 < RC; k0 += 4) {
        const double bb = xi[swy(k0 + lc, lr)];
#pragma unroll
        for (int u = 0; u < 2; ++u)
          dmma(xacc[u][0], xacc[u][1], tl[sw64(k0 + lc, 16 * warp + 8 * u + lr)], bb);
      }
      __syncthreads();
      ++ncon;
    }
    // r = Y_J - xacc ; X_J = G_JJ^-T r
    {  // G_JJ^-1 (lower 16x16 blocks) into the packed buffer
      const double* src = tile_ptr<MODE>(Kb, R, tm, J, J);
      for (int idx = tid; idx < TILE * 32; idx += NTC) {
        const int r = idx >> 5, c2 = 2 * (idx & 31);
        if (!sd_upper(r, c2)) cp_async16(sT + sd(r, c2), src + r * TILE + c2);
      }
    }
    cp_async_commit();
    sY = sStage + SY_B;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int r = 16 * warp + 8 * u + lr, cc = 2 * lc;
      const double2 y = __ldcg(reinterpret_cast<const double2*>(Yb + (long)(J * TILE + r) * RHSW + cc));
      sY[swy(r, cc)] = y.x - xacc[u][0];
      sY[swy(r, cc + 1)] = y.y - xacc[u][1];
    }
    cp_async_wait<0>();
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int r = 16 * warp + 8 * u;
      double x0 = 0.0, x1 = 0.0;
      for (int k0 = r; k0 < TILE; k0 += 4)  // (G_JJ^-1)^T upper: row j needs k >= j
        dmma(x0, x1, sT[sd(k0 + lc, r + lr)], sY[swy(k0 + lc, lr)]);
      const int rr = r + lr, cc = 2 * lc;
      *reinterpret_cast<double2*>(Xb + (long)(J * TILE + rr) * RHSW + cc) = make_double2(x0, x1);
    }
    __syncthreads();
  }
#ifdef HOM_TIMING
  if (blockIdx.x < 64 && threadIdx.x == 0) g_tm[blockIdx.x][39][1] = clk_ordered();
#endif
}

// ====================================================================================
// k_condense_ws: the same factorisation with a dedicated factor warp (dense structure).
//
// k_condense runs the 64x64 diagonal factor + inverse (a serial pivot chain on one warp, ~30% of
// a CTA's time at config 2, profiles/r02/) while its other three warps wait at a barrier.  Here a
// fifth warp owns that chain and the four MMA warps keep the FP64 tensor pipe busy meanwhile: for
// column J they accumulate S_IJ = A_IJ - sum_{K<J} G_IK G_JK^T of every off-diagonal tile (which
// does not depend on G_JJ) and park S_IJ in the tile's pool slot; once the factor warp has
// published G_JJ^-1 they stream the parked tiles back in 16-row chunks and form
// G_IJ = S_IJ (G_JJ^-1)^T.  The factor warp also forms Y_J = G_JJ^-1 (K_fe,J - sum_K G_JK Y_K), the
// Schur sum Y^T Y and the C_eff / P_eff epilogue.  Hand-offs are named barriers:
//   BAR_S: MMA warps arrive after writing S_JJ (sT) and K_fe,J - yacc (sY); the factor warp syncs.
//   BAR_G: the factor warp arrives after G_JJ^-1 (sT, pool), Y_J (pool); the MMA warps sync.
// The backward pass X = G^-T Y (MMA warps) is the one of k_condense.
// ====================================================================================
constexpr int NTC_WS = NTC + 32;
constexpr int BAR_MMA = 1, BAR_S = 2, BAR_G = 3;
__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// generic-proxy global writes of this thread before later async-proxy (TMA) reads of them
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// smem (doubles): stages[2] (TMA k-chunks; the TRSM / backward row-chunk ring) | factor scratch |
// sY (K_fe,J - yacc; backward: Y_J - xacc) | sY2 (Y_J) | sT (packed diagonal tile) | misc
constexpr int WS_STAGES = 2 * STAGE_DBL;
constexpr int WS_SCR = WS_STAGES, WS_SY = WS_SCR + 3 * 320, WS_SY2 = WS_SY + 64 * RHSW, WS_ST = WS_SY2 + 64 * RHSW;
constexpr int WS_MISC = WS_ST + SD_DBL, WS_SMEM_DBL = WS_MISC + 64;
constexpr int WS_RC = 16, WS_NCH = 4, WS_CH = WS_RC * TILE;  // TRSM row chunks: 16 rows, 4-deep ring
static_assert(WS_NCH * WS_CH <= WS_STAGES, "TRSM chunk ring fits the stage area");
static_assert(4 * (16 * TILE + 16 * RHSW) <= WS_SY, "backward ring fits stages + scratch");
static_assert(WS_SMEM_DBL * 8 + 1024 <= 76 * 1024, "three CTAs per SM");

__global__ void __launch_bounds__(NTC_WS, 3)
k_condense_ws(RveDev R, const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap ymap, int b0,
              double* __restrict__ Kt, double* __restrict__ Y, const double* __restrict__ Cavg,
              const double* __restrict__ Pavg, double* __restrict__ Ceff, double* __restrict__ Peff,
              double* __restrict__ PavgOut, double* __restrict__ X, int* __restrict__ info) {
  extern __shared__ __align__(1024) double smem[];
  double* sStage = smem;
  double* sScr = smem + WS_SCR;
  double* sY = smem + WS_SY;
  double* sY2 = smem + WS_SY2;
  double* sT = smem + WS_ST;
  int* sFail = reinterpret_cast<int*>(smem + WS_MISC);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + WS_MISC + 8);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  const int bl = blockIdx.x, b = b0 + bl;
  const int nt = R.nt, NT = R.NT;
  double* Kb = Kt + (long)bl * R.nslot * TILE_ELEMS;
  double* Yb = Y + (long)bl * NT * RHSW;
  double* Xb = X + (long)(b - R.xb0) * NT * RHSW;
  const TileMask tm{};  // unused (dense structure)
  if (tid == 0) {
    sFail[0] = 0;
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 4) {
    // ============================ factor warp ============================
    double Sacc0 = 0.0, Sacc1 = 0.0;  // Schur sum Y^T Y (8x8 DMMA fragment)
    for (int J = 0; J < nt; ++J) {
      nbar_sync(BAR_S, NTC_WS);
      TMARK_T(5, 128);
#ifdef HOM_WS_FAKE  // timing experiment only: identity instead of the factor (wrong results)
      for (int idx = lane; idx < SD_DBL; idx += 32) sT[idx] = 0.0;
      __syncwarp();
      for (int r = lane; r < TILE; r += 32) sT[sd(r, r)] = 1.0;
      __syncwarp();
      const bool ok = true;
#else
      const bool ok = factor_invert_diag<1>(sT, sScr, sFail, J, 0, lane, [] { __syncwarp(); });
#endif
      TMARK_T(6, 128);
      if (ok) {
        // Y_J = G_JJ^-1 (K_fe,J - sum_K G_JK Y_K): 8 row blocks, G_JJ^-1 lower (k < 8 (rb + 1))
#pragma unroll 1
        for (int rb = 0; rb < 8; ++rb) {
          double y0 = 0.0, y1 = 0.0;
          for (int k0 = 0; k0 < 8 * rb + 8; k0 += 4) dmma(y0, y1, sT[sd(8 * rb + lr, k0 + lc)], sY[swy(k0 + lc, lr)]);
          const int rr = 8 * rb + lr, cc = 2 * lc;
          sY2[swy(rr, cc)] = y0;
          sY2[swy(rr, cc + 1)] = y1;
          *reinterpret_cast<double2*>(Yb + (long)(J * TILE + rr) * RHSW + cc) = make_double2(y0, y1);
        }
        __syncwarp();
#pragma unroll
        for (int k0 = 0; k0 < TILE; k0 += 4)  // S += Y_J^T Y_J
          dmma(Sacc0, Sacc1, sY2[swy(k0 + lc, lr)], sY2[swy(k0 + lc, lr)]);
        double* Gjj = tile_ptr<0>(Kb, R, tm, J, J);
        for (int idx = lane; idx < TILE_ELEMS / 2; idx += 32) {
          const int r = idx >> 5, cc = 2 * (idx & 31);
          *reinterpret_cast<double2*>(Gjj + r * TILE + cc) =
              sd_upper(r, cc) ? make_double2(0.0, 0.0) : make_double2(sT[sd(r, cc)], sT[sd(r, cc + 1)]);
        }
        fence_proxy_async_global();  // Y_J is read by TMA in later columns
      }
      __syncwarp();
      TMARK_T(7, 128);
      nbar_arrive(BAR_G, NTC_WS);
      if (!ok) return;
    }
    // K4 epilogue: C_eff = <C> - Y_e^T Y_e / |Omega|, P_eff = <P> - Y_e^T Y_r / |Omega|
    // (sY2: the MMA warps' backward ring may already cover the scratch area)
    double* sSum = sY2;
    sSum[lr * 8 + 2 * lc] = Sacc0;
    sSum[lr * 8 + 2 * lc + 1] = Sacc1;
    __syncwarp();
    const int m = R.m;
    const double* Ca = Cavg + (long)bl * 64;
    for (int t = lane; t < m * m; t += 32) {
      const int i = t / m, j = t % m;
      Ceff[(long)b * m * m + t] = Ca[i * m + j] - sSum[i * 8 + j] / R.vol;
    }
    if (R.finite && lane < m) {
      const double pa = Pavg[(long)bl * 8 + lane];
      if (Peff) Peff[(long)b * m + lane] = pa - sSum[lane * 8 + m] / R.vol;
      if (PavgOut) PavgOut[(long)b * m + lane] = pa;
    }
    return;
  }

  // ============================ MMA warps (tid < 128) ============================
  auto gsync = [] { nbar_sync(BAR_MMA, NTC); };
  const int R0 = (warp >> 1) * 32, C0 = (warp & 1) * 32;  // accumulation quadrant
  const int cLo = warp, cHi = 7 - warp;                    // TRSM column-block pair (balanced)
  uint32_t ph0 = 0, ph1 = 0;
  auto wait_stage = [&](int st) {
    if (st == 0) { mbar_wait(&full[0], ph0); ph0 ^= 1u; }
    else { mbar_wait(&full[1], ph1); ph1 ^= 1u; }
  };
  const long krow0 = (long)bl * R.nslot * TILE;
  const long yrow0 = (long)bl * NT;
  bool failed = false;

  for (int J = 0; J < nt; ++J) {
    TMARK(0);
    // ---------- S_JJ = A_JJ - sum_K G_JK G_JK^T ; yacc = sum_K G_JK Y_K (as k_condense) ----------
    {
      double dacc[9][2];
      double yacc[2][2] = {};
      DIAG_DISPATCH(diag_load, dacc, tile_ptr<0>(Kb, R, tm, J, J), lane);
      int K = 0, kc = 0, par = 0;
      auto issue_d = [&](int stg, int KK, int kcc) {
        double* st = sStage + stg * STAGE_DBL;
        fence_proxy_async();
        mbar_expect(&full[stg], (64 * KC + KC * RHSW) * 8);
        tma_load_2d(st, &kmap, kcc * KC, (int)(krow0 + (long)tile_slot<0>(R, tm, J, KK) * TILE), &full[stg]);
        tma_load_2d(st + 2 * 64 * KC, &ymap, 0, (int)(yrow0 + KK * TILE + kcc * KC), &full[stg]);
      };
      if (K < J && tid == 0) issue_d(0, K, 0);
      while (K < J) {
        int K2 = K, kc2 = kc + 1;
        if (kc2 == CPT) { kc2 = 0; K2 = K + 1; }
        if (K2 < J && tid == 0) issue_d(par ^ 1, K2, kc2);
        wait_stage(par);
        const double* st = sStage + par * STAGE_DBL;
        switch (warp) {
          case 0: diag_chunk<0, true>(dacc, st, lane); break;
          case 1: diag_chunk<1, true>(dacc, st, lane); break;
          case 2: diag_chunk<2, true>(dacc, st, lane); break;
          default: diag_chunk<3, true>(dacc, st, lane); break;
        }
        const double* sYc = st + 2 * 64 * KC;
#pragma unroll
        for (int k0 = 0; k0 < KC; k0 += 4) {
          const double bb = sYc[(k0 + lc) * RHSW + lr];
#pragma unroll
          for (int u = 0; u < 2; ++u) dmma(yacc[u][0], yacc[u][1], st[swt(16 * warp + 8 * u + lr, k0 + lc)], bb);
        }
        gsync();
        K = K2; kc = kc2; par ^= 1;
      }
      DIAG_DISPATCH(diag_store, dacc, sT, lane);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int r = 16 * warp + 8 * u + lr, cc = 2 * lc;
        const double2 y = __ldcg(reinterpret_cast<const double2*>(Yb + (long)(J * TILE + r) * RHSW + cc));
        sY[swy(r, cc)] = y.x - yacc[u][0];
        sY[swy(r, cc + 1)] = y.y - yacc[u][1];
      }
    }
    nbar_arrive(BAR_S, NTC_WS);  // sT, sY ready: the factor warp starts the pivot chain
    TMARK(1);
    // ---------- off-diagonal accumulation of column J under the chain; park S_IJ in its slot ----------
    if (J > 0) {
      for (int I = J + 1; I < nt; ++I) {
        double acc[4][4][2];
        double* Aij = tile_ptr<0>(Kb, R, tm, I, J);
        if (__ldg(R.tile_nz + I * nt + J)) {
          load_frag(acc, Aij, R0, C0, lane);
        } else {  // fill tile: A_IJ = 0 (never written by K1)
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
        }
        int K = 0, kc = 0, par = 0;
        auto issue_o = [&](int stg, int KK, int kcc) {
          double* st = sStage + stg * STAGE_DBL;
          fence_proxy_async();
          mbar_expect(&full[stg], 2 * 64 * KC * 8);
          tma_load_2d(st, &kmap, kcc * KC, (int)(krow0 + (long)tile_slot<0>(R, tm, I, KK) * TILE), &full[stg]);
          tma_load_2d(st + 64 * KC, &kmap, kcc * KC, (int)(krow0 + (long)tile_slot<0>(R, tm, J, KK) * TILE),
                      &full[stg]);
        };
        if (tid == 0) issue_o(0, 0, 0);
        while (K < J) {
          int K2 = K, kc2 = kc + 1;
          if (kc2 == CPT) { kc2 = 0; K2 = K + 1; }
          if (K2 < J && tid == 0) issue_o(par ^ 1, K2, kc2);
          wait_stage(par);
          const double* st = sStage + par * STAGE_DBL;
          mma_chunk<false, true>(acc, st, st + 64 * KC, R0, C0, lane);
          gsync();
          K = K2; kc = kc2; par ^= 1;
        }
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni)
            *reinterpret_cast<double2*>(Aij + (R0 + 8 * mi + lr) * TILE + C0 + 8 * ni + 2 * lc) =
                make_double2(acc[mi][ni][0], acc[mi][ni][1]);
      }
    } else {  // J = 0: S_I0 = A_I0 is already in place; fill tiles need explicit zeros
      for (int I = 1; I < nt; ++I) {
        if (__ldg(R.tile_nz + I * nt)) continue;
        double* Ai0 = tile_ptr<0>(Kb, R, tm, I, 0);
        for (int idx = tid; idx < TILE_ELEMS / 2; idx += NTC)
          reinterpret_cast<double2*>(Ai0)[idx] = make_double2(0.0, 0.0);
      }
    }
    gsync();  // every parked S_IJ written before any warp streams it back
    TMARK(2);
    nbar_sync(BAR_G, NTC_WS);
    TMARK(3);
    if (sFail[0]) { failed = true; break; }
    // ---------- G_IJ = S_IJ (G_JJ^-1)^T, streamed in 16-row chunks of the parked tiles ----------
    {
      const int nch = (nt - 1 - J) * (TILE / WS_RC);
      int nis = 0;
      auto issue_c = [&]() {  // chunk nis: tile I = J + 1 + nis / 4, rows 16 (nis % 4)
        const int I = J + 1 + nis / (TILE / WS_RC), rq = nis % (TILE / WS_RC);
        stage_rows(sStage + (nis % WS_NCH) * WS_CH, tile_ptr<0>(Kb, R, tm, I, J), rq * WS_RC, WS_RC, tid);
        cp_async_commit();
        ++nis;
      };
      while (nis < WS_NCH - 1 && nis < nch) issue_c();
      for (int c = 0; c < nch; ++c) {
        if (nis < nch) {
          issue_c();
          cp_async_wait<WS_NCH - 1>();
        } else {
          const int ahead = nis - c - 1;
          if (ahead >= 2) cp_async_wait<2>();
          else if (ahead == 1) cp_async_wait<1>();
          else cp_async_wait<0>();
        }
        gsync();
        const double* sS = sStage + (c % WS_NCH) * WS_CH;
        // warp: column blocks cLo, cHi (all 16 rows = 2 row blocks); G_JJ^-1 lower: block c needs k < 8(c+1)
        double g[2][2][2] = {};
        int k0 = 0;
        for (; k0 < 8 * (cLo + 1); k0 += 4) {
          const double bl0 = sT[sd(8 * cLo + lr, k0 + lc)], bh0 = sT[sd(8 * cHi + lr, k0 + lc)];
#pragma unroll
          for (int mi = 0; mi < 2; ++mi) {
            const double a = sS[sw64(8 * mi + lr, k0 + lc)];
            dmma(g[mi][0][0], g[mi][0][1], a, bl0);
            dmma(g[mi][1][0], g[mi][1][1], a, bh0);
          }
        }
        for (; k0 < 8 * (cHi + 1); k0 += 4) {
          const double bh0 = sT[sd(8 * cHi + lr, k0 + lc)];
#pragma unroll
          for (int mi = 0; mi < 2; ++mi) dmma(g[mi][1][0], g[mi][1][1], sS[sw64(8 * mi + lr, k0 + lc)], bh0);
        }
        const int I = J + 1 + c / (TILE / WS_RC), rq = c % (TILE / WS_RC);
        double* Gij = tile_ptr<0>(Kb, R, tm, I, J) + (long)rq * WS_RC * TILE;
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
          const int r = 8 * mi + lr;
          *reinterpret_cast<double2*>(Gij + r * TILE + 8 * cLo + 2 * lc) = make_double2(g[mi][0][0], g[mi][0][1]);
          *reinterpret_cast<double2*>(Gij + r * TILE + 8 * cHi + 2 * lc) = make_double2(g[mi][1][0], g[mi][1][1]);
        }
        gsync();  // ring slot c % 4 free before it is refilled
      }
      fence_proxy_async_global();  // G_IJ is read by TMA in later columns
    }
    gsync();
    TMARK(4);
  }

  if (failed) {  // report and poison the outputs of this RVE (the factor warp has returned)
    if (tid == 0) info[b] = sFail[0];
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    if (tid < R.m * R.m) Ceff[(long)b * R.m * R.m + tid] = nan;
    if (Peff && tid < R.m) Peff[(long)b * R.m + tid] = nan;
    return;
  }

  // ======================= backward: X = G^-T Y (as k_condense, MMA warps) ===================
  constexpr int RC = 16, RPT = TILE / RC;
  constexpr int NSTB = 4, BST = RC * TILE + RC * RHSW;
  for (int J = nt - 1; J >= 0; --J) {
    double xacc[2][2] = {};
    int I = J + 1, rq = 0;
    int nis = 0, ncon = 0;
    auto issue_b = [&]() {
      double* nb = smem + (nis % NSTB) * BST;
      stage_rows(nb, tile_ptr<0>(Kb, R, tm, I, J), rq * RC, RC, tid);
      stage_rhs(nb + RC * TILE, Xb + (long)(I * TILE + rq * RC) * RHSW, RC, tid);
      cp_async_commit();
      ++nis;
      if (++rq == RPT) { rq = 0; ++I; }
    };
    {  // G_JJ^-1 (lower 16x16 blocks) into the packed buffer: the oldest cp.async group, so every
       // wait of the chunk ring below also covers it
      const double* src = tile_ptr<0>(Kb, R, tm, J, J);
      for (int idx = tid; idx < TILE * 32; idx += NTC) {
        const int r = idx >> 5, c2 = 2 * (idx & 31);
        if (!sd_upper(r, c2)) cp_async16(sT + sd(r, c2), src + r * TILE + c2);
      }
      cp_async_commit();
    }
    while (nis < NSTB - 1 && I < nt) issue_b();
    while (ncon < nis) {
      if (I < nt) {
        issue_b();
        cp_async_wait<NSTB - 1>();
      } else {
        const int ahead = nis - ncon - 1;
        if (ahead >= 2) cp_async_wait<2>();
        else if (ahead == 1) cp_async_wait<1>();
        else cp_async_wait<0>();
      }
      gsync();
      const double* tl = smem + (ncon % NSTB) * BST;
      const double* xi = tl + RC * TILE;
#pragma unroll
      for (int k0 = 0; k0 < RC; k0 += 4) {
        const double bb = xi[swy(k0 + lc, lr)];
#pragma unroll
        for (int u = 0; u < 2; ++u) dmma(xacc[u][0], xacc[u][1], tl[sw64(k0 + lc, 16 * warp + 8 * u + lr)], bb);
      }
      gsync();
      ++ncon;
    }
    cp_async_wait<0>();
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int r = 16 * warp + 8 * u + lr, cc = 2 * lc;
      const double2 y = __ldcg(reinterpret_cast<const double2*>(Yb + (long)(J * TILE + r) * RHSW + cc));
      sY[swy(r, cc)] = y.x - xacc[u][0];
      sY[swy(r, cc + 1)] = y.y - xacc[u][1];
    }
    gsync();
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int r = 16 * warp + 8 * u;
      double x0 = 0.0, x1 = 0.0;
      for (int k0 = r; k0 < TILE; k0 += 4) dmma(x0, x1, sT[sd(k0 + lc, r + lr)], sY[swy(k0 + lc, lr)]);
      const int rr = r + lr, cc = 2 * lc;
      *reinterpret_cast<double2*>(Xb + (long)(J * TILE + rr) * RHSW + cc) = make_double2(x0, x1);
    }
    gsync();
  }
}

__global__ void k_first_fail(const int* __restrict__ f, int n, int sentinel, int* out);

// Dense-structure kernel: 0 = k_condense (default), 1 = k_condense_ws (factor warp + 4 MMA warps, 3 CTAs/SM;
// HOM_CONDENSE=ws, for A/B measurements; its 4-CTA/SM version with 8-wide cp.async chunks was measured
// slower still and lives in git history, commit e0bd4eb -- DESIGN.md §5.1).
// Off by default: measured slower (profiles/r02/condense_variants.md).  Its code is kept
// compiled into the tile-sparse instantiations: with it ptxas allocates k_condense<1> without the 96 B of
// spills the factor's panel phase had otherwise (tile-sparse configs 2 / 3 5 % faster in a same-box A/B,
// dense unchanged).
constexpr int LA_Q_DEFAULT = 0;
static int condense_variant() {
  static const int v = [] {
    const char* e = getenv("HOM_CONDENSE");
    return (e && e[0] == 'w') ? 1 : 0;
  }();
  return v;
}

void launch_condense(const RveDev& R, int b0, int nb, double* Kt, double* Y, const double* Cavg,
                     const double* Pavg, double* Ceff, double* Peff, double* PavgOut, double* X,
                     int* info, cudaStream_t s, const TileMask* tm) {
  size_t sm = (size_t)SMEM_DBL * sizeof(double);
  static const TileMask none{};
  // tensor maps of this launch's K_ff pool ([rows][64] FP64, 16x64 boxes, 128-byte swizzle) and
  // right-hand sides ([rows][8], 8x16 boxes)
  CUtensorMap kmap, ymap;
  {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        fn = nullptr;
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode) {  // surfaces as a launch error through the caller's error check
      cudaLaunchKernel((const void*)k_first_fail, dim3(0), dim3(0), nullptr, 0, s);
      return;
    }
    const cuuint64_t kdim[2] = {(cuuint64_t)TILE, (cuuint64_t)nb * R.nslot * TILE};
    const cuuint64_t kstr[1] = {(cuuint64_t)TILE * sizeof(double)};
    const cuuint32_t kbox[2] = {(cuuint32_t)KC, (cuuint32_t)TILE}, one[2] = {1, 1};
    encode(&kmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, Kt, kdim, kstr, kbox, one, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const cuuint64_t ydim[2] = {(cuuint64_t)RHSW, (cuuint64_t)nb * R.NT};
    const cuuint64_t ystr[1] = {(cuuint64_t)RHSW * sizeof(double)};
    const cuuint32_t ybox[2] = {(cuuint32_t)RHSW, (cuuint32_t)KC};
    encode(&ymap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, Y, ydim, ystr, ybox, one, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (R.dense_tiles && condense_variant() == 1) {
    const size_t smw = (size_t)WS_SMEM_DBL * sizeof(double);
    cudaFuncSetAttribute(k_condense_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smw);
    k_condense_ws<<<nb, NTC_WS, smw, s>>>(R, kmap, ymap, b0, Kt, Y, Cavg, Pavg, Ceff, Peff, PavgOut, X, info);
    return;
  }
  auto k = R.dense_tiles ? k_condense<0> : (tm ? k_condense<1> : k_condense<2>);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const char* la_env = getenv("HOM_LA");  // tile-sparse diagonal lookahead: chunks per pivot-chain window (0 = off)
  const int la_q = la_env ? atoi(la_env) : LA_Q_DEFAULT;
  k<<<nb, NTC, sm, s>>>(R, tm ? *tm : none, kmap, ymap, b0, Kt, Y, Cavg, Pavg, Ceff, Peff, PavgOut, X, info, la_q);
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
