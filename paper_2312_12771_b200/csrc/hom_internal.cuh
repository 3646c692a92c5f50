// hom_internal.cuh -- device-side data structures and kernel entry points of libhom.so.
// Product path only; shares nothing with oracle/ (DESIGN.md §2).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/hom.h"

// Device-side bounds checks of the shared-memory tables and pool slots, compiled in only for debug builds
// (HOM_NVCC_EXTRA=-DHOM_DEBUG_BOUNDS; compute-sanitizer is not available on the B200 pool): a failed check
// prints its location and traps, so the launch fails with an error the caller reports.
#ifdef HOM_DEBUG_BOUNDS
#include <cstdio>
#define HOM_DCHECK(c)                                                                      \
  do {                                                                                     \
    if (!(c)) {                                                                            \
      printf("HOM_DCHECK %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, (int)blockIdx.x, \
             (int)threadIdx.x, #c);                                                        \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define HOM_DCHECK(c) ((void)0)
#endif

namespace hom {

constexpr int TILE = 64;          // K_ff tile edge (rows and columns)
constexpr int TILE_ELEMS = TILE * TILE;
constexpr int KC = 16;            // k-chunk staged per pipeline stage (condense.cu)
constexpr int RHSW = 8;           // right-hand-side columns kept per RVE (m <= 6, +1 for r_f)
constexpr int NTHR = 256;         // threads per CTA of the RVE kernels
constexpr int MAX_K1_CLASSES = 64;  // K1 stencil classes (RveDev::ncls) kept in shared memory

// Geometry + topology of the (shared) RVE mesh and the per-RVE phase/material tables.
struct RveDev {
  int dim, nen, nq, ne;           // spatial dim, nodes/elem, qps/elem, elements
  int n_indep, npad, nt, NT;      // independent nodes, dim*n_indep, tiles, nt*64
  int corner;                     // fixed independent node (corner class)
  int m, ncol, finite;            // tangent size, RHS columns used, finite strain flag
  double vol;                     // |Omega|
  const int* elem_indep;          // [ne][nen]
  const double* grad;             // [ne][nq][nen][dim]  dN/dx at the qps
  const double* wdet;             // [ne][nq]            Gauss weight * det J
  const int* inc_ptr;             // [n_indep+1] incidences (e<<4 | a) of each independent node
  const int* inc;
  const int* nbr_ptr;             // [n_indep+1] neighbour list of each independent node
  const int* nbr;                 // neighbour independent node
  const int* nbr_owner;           // owner node of each neighbour entry
  const int* sh_ptr;              // [n_nbr+1] shared (e<<8 | a<<4 | b) triples per neighbour entry
  const int* sh;
  const uint8_t* phase;           // [B|1][ne]
  int phase_per_rve;
  const double* mat;              // [B|1][n_phase][mat_stride]
  int mat_per_rve, n_phase, mat_stride;  // stride 2 (E, nu) / (alpha, kappa); 3 (alpha, beta, kappa)
  // geometry-only element matrices of the isotropic closed form (small strain):
  // K_e = lam_e * Klam_e + mu_e * Kmu_e, K_fe rows = lam_e * Flam_e + mu_e * Fmu_e
  const double* Klam;             // [ntype][nen*dim][nen*dim] (element type = identical geometry)
  const double* Kmu;
  const int* etype;               // [ne] element -> type
  const double* FlamT;            // [ntype][nen*dim][m] K_fe tables per element type
  const double* FmuT;
  int ntype;
  int fs_ks, fs_ke_off;            // finite strain: K_e of the RVE kept in K1's shared memory (2 CTAs/SM), its offset
  // finite strain, K_e in shared memory: qp geometry per element type (identical grad / wdet), staged
  // with the RVE's w, phases and connectivity in the material pass (fs_ntype = 0: not staged)
  int fs_ntype;
  const double* fs_tgeo;          // [fs_ntype][nq][nen * dim + 1] (dN/dx at the qp, then Gauss weight * det J)
  const int* fs_etype;            // [ne]
  int gtab;                       // 1: the (type, phase) tables exceed shared memory; K1 reads Klam/Kmu/FlamT/FmuT
                                  // from global memory and combines them with (lam, mu) per phase on the fly
  int npw;                        // K1: row-buffer capacity in RVE nodes per warp (12 / dim)
  const double* Flam;             // [ne][nen*dim][m]
  const double* Fmu;
  const double* evol;             // [ne] element volume
  const uint8_t* tile_nz;         // [nt*nt] 1 if lower tile (I,J) of K_ff has a structural nonzero
  // Tile structure of the factor: g_nz[I*nt+J] = 1 if lower tile (I,J) of G is
  // processed -- every lower tile (dense path) or the symbolic tile fill of tile_nz
  // (tile-sparse path); tslot[I*nt+J] = its slot in the per-RVE pool (-1: not stored).
  const uint8_t* g_nz;
  const int* tslot;
  int nslot;                      // pool slots (64x64 tiles) per RVE
  int dense_tiles;                // 1: every lower tile stored at slot I(I+1)/2 + J (no table lookups)
  const int* a_list;              // [n_a] (I << 16 | J) of the structurally nonzero lower tiles (K1)
  int n_a;
  // K1 gather records: node p, neighbour slot j < maxdeg -> rs4 int4s
  // {q (-1: none / corner), n_sh, code_0 .. code_{n_sh-1}, -1 ...}, code = e<<8 | a<<4 | b
  const int4* nrec;
  int maxdeg, rs4;
  // K1 warp work items: {tile code I<<16|J, first row node p0, node count nn, pool slot}, and per item one record
  // per lane: (g << 24 | record index) for node p0 + g, -1 = idle lane (<= 32 records, <= npw nodes)
  const int4* witem;
  const int* wlist;
  int n_witem;
  int xb0;                        // first RVE of the influence store X (the context's local range)
  const int* nat_of;              // [n_indep] internal node -> natural (API) node; nullptr = identity
  const int* int_of;              // [n_indep] natural node -> internal node; nullptr = identity
  // K1 stencil classes (small strain, shared-memory tables): record word 1 = n_sh | (class + 1) << 16; a
  // class is the sorted list of element-local pairs (a << 4 | b) cls_ab[cls_ptr[c] .. cls_ptr[c + 1])
  int ncls;
  const int* cls_ptr;
  const int* cls_ab;
  const int* wcov;                // [n_witem][32]: bit 2n + b = column 2 lane + b of item node n covered
};

// Two-level additive macro preconditioner (coarse.cu): aggregates of macro
// nodes with their rigid-body modes, nc = nagg * nm coarse DOFs (nc = 0: one-level only).
constexpr int CC_MIN_DOF = 1024, CC_NA2 = 8, CC_NA3 = 3, CC_NC_MAX = 192, CC_NB_MAX = 27,
              CC_ROWMAX = 96,  // longest CSR row the coarse assembly stages (3-D: 81)
              CC_NCH = 8;      // chunks per aggregate node list in the PCG's restriction
struct CoarseDev {
  int nc, nm, nagg, nbmax;
  const int* agg;      // [n_nodes] aggregate of each node
  const double* rel;   // [n_nodes][dim] (x - centroid of its aggregate) / h
  const int* aptr;     // [nagg+1] nodes of each aggregate: anode[aptr[a] .. aptr[a+1])
  const int* anode;
  const int* nbr;      // [nagg][nbmax] aggregates coupled through K_M (-1 padded)
  double* Ac;          // [nc][nc] P^T K_M P (per solve)
  double* Ainv;        // [nc][nc] its inverse (dropped modes: zero rows / columns)
  // per cluster size of k_macro_cg_cluster2 (index 0: G = 16, 1: G = 8)
  int nla_max[2], kmax[2];
  const int* lptr[2];   // [G+1] CTA g's aggregates: lagg[lptr[g] .. lptr[g+1])
  const int* lagg[2];
  const int* tch[2];    // [nagg][kmax] the CTAs touching each aggregate: g << 16 | its local index there
  const int* lnptr[2];  // node list of each local aggregate: lnode[lnptr[q] .. lnptr[q+1]) (CTA-local node ids)
  const int* lnode[2];
  const int* ntch[2];   // [nagg] number of CTAs touching each aggregate
  // the same for k_macro_cg_grid's partition (G = ggrid CTAs, one per SM)
  int ggrid, nla_max_g, kmax_g;
  const int *lptr_g, *lagg_g, *tch_g, *lnptr_g, *lnode_g, *ntch_g;
  double2* gpart;       // [ggrid][nla_max[2] * nm] k_macro_cg_grid's restriction partials
};
struct CoarseHost {
  int nc = 0, nm = 0, nagg = 0, nbmax = 0;
  std::vector<int> agg, aptr, anode, nbr;
  std::vector<double> rel;
  struct Loc {
    int nla_max = 0, kmax = 0;
    std::vector<int> lptr, lagg, tch, lnptr, lnode, ntch;
  } loc[3];
  int ggrid = 0;
};
// host side, once per macro mesh (Dirichlet rows of P are zeroed on the device through dmask)
CoarseHost coarse_build(int dim, int n_nodes, const double* coords, const int* rowptr, const int* col,
                        int one_level, int ggrid);
// coefficient of coarse mode m (0..dim-1: translations, then the rotations) in DOF component
// c of a node at scaled position d relative to its aggregate centroid: the column of P
__host__ __device__ __forceinline__ double cc_coef(int dim, int c, int m, const double* d) {
  if (m < dim) return c == m ? 1.0 : 0.0;
  if (dim == 2) return c == 0 ? -d[1] : d[0];  // u = w e_z x d
  switch (m - 3) {                              // 3-D: rotations about x, y, z
    case 0: return c == 1 ? -d[2] : (c == 2 ? d[1] : 0.0);
    case 1: return c == 0 ? d[2] : (c == 2 ? -d[0] : 0.0);
    default: return c == 0 ? -d[1] : (c == 1 ? d[0] : 0.0);
  }
}

struct MacroDev {
  int dim, nen, nq, ne, n_nodes, ndof, m, finite, nnz;
  const int* conn;                // [ne][nen]
  const double* grad;             // [ne][nq][nen][dim]
  const double* shp;              // [nq][nen]
  const double* wdet;             // [ne][nq]
  const int* rowptr;              // [ndof+1] scalar CSR
  const int* col;                 // [nnz]
  const int* nz_blk;              // [nnz] node-pair block of each entry
  const uint8_t* nz_cc;           // [nnz] ci*4 + cj
  const int* blk_ptr;             // [n_blk+1] shared (E<<8 | a<<4 | b) per node-pair block
  const int* blk_sh;
  const int* ninc_ptr;            // [n_nodes+1] incidences (E<<4 | a)
  const int* ninc;
  const uint8_t* dmask;           // [ndof] 1 = Dirichlet
  const double* dval;             // [ndof] prescribed value (0 where free)
  const double* fbody;            // [ndof] external load: consistent body load + nodal forces
  double load_factor;             // multiplies fbody (load stepping, hom_set_load_factor)
  int constant_basis;             // 1: one RVE per element (eq:constSolution1/2), D = C_eff per element
  const double* Cavg_e;           // [ne][m][m] <C> per element (constant basis)
  const double* evol;             // [ne] element volume |B_e|
  // cluster PCG with z windows (meshes whose full z copy does not fit a CTA): for cluster size
  // G = 16 (index 0) and 8 (index 1), CTA g reads z only on its CSR slice's column range
  // cg_win[(idx*16 + g)*2 + 0..1] = [lo, hi); cg_wmax = largest window; cg_wok = every CTA's rows
  // fall in at most CG_WDEST other windows
  const int* cg_win;
  int cg_wmax[2], cg_wok[2];
  int cg_ellw;  // k_macro_cg_cluster2: ELL width (longest CSR row)
  double* cg_gval;  // [cg_ellw][ndof] ELL slots that do not fit shared memory (L2-resident spill)
  int* cg_gcol;
  CoarseDev cc;
  unsigned long long* cg_prof;  // HOM_CG_PROF=1: clock64 phase sums of k_macro_cg_cluster2, [16 CTAs][16]
};
constexpr int CG_WDEST = 4;

// Tile structure of a tile-sparse factor with nt <= 64, passed to k_condense by value (kernel
// parameter space = constant bank: warp-uniform lookups without global loads): bit J of row[I] /
// bit I of col[J] = G(I,J) stored; rowstart[I] = slot of row I's first stored tile.
struct TileMask {
  unsigned long long row[64], col[64];
  int rowstart[64];
};

struct CgState {
  int iterations;
  int status;                     // 0 ok, 5 not converged, 6 breakdown
  double rel_residual;
  double rhs_norm;
};

// ---- kernels (launch wrappers; all enqueue on `s`) ----
size_t rve_assemble_smem(const RveDev& R, int npw);  // K1 dynamic shared memory
int rve_assemble_npw(const RveDev& R);              // K1 row-buffer nodes per warp
// small strain (and dim 1): one CTA per RVE of [b0, b0 + nb)
void launch_rve_assemble(const RveDev& R, int b0, int nb, double* Kt, double* Y, double* Cavg,
                         double* Pavg, double* rfn, cudaStream_t s);
// finite strain, fused material pass + tile writer: `slots` persistent CTAs, each with a scratch
// slice of ne * FS_RECORD doubles (rve_assemble_fs_slots() = resident CTAs on the device)
constexpr int FS_RECORD = 76;  // element record (rve_assembly.cu EL_STRIDE)
int rve_assemble_fs_slots(const RveDev& R);
void launch_rve_assemble_fs(const RveDev& R, int b0, int nb, const double* F, const double* w, double* Kt,
                            double* Y, double* Cavg, double* Pavg, double* rfn, double* scratch, int slots,
                            int* jflag, cudaStream_t s);
void launch_condense(const RveDev& R, int b0, int nb, double* Kt, double* Y, const double* Cavg,
                     const double* Pavg, double* Ceff, double* Peff, double* PavgOut, double* X,
                     int* info, cudaStream_t s,
                     const struct TileMask* tm = nullptr);
void launch_first_fail(const int* flags, int n, int sentinel, int* out, cudaStream_t s);
void launch_max_reduce(const double* v, int n, double* out, cudaStream_t s);

void launch_macro_kin(const MacroDev& M, const double* u, double* kin, int add_identity,
                      cudaStream_t s);
void launch_macro_assemble(const MacroDev& M, const double* D, double* val, double* diag,
                           cudaStream_t s);
void launch_macro_rhs(const MacroDev& M, const double* val, const double* S, double scale,
                      double* rhs, double* Rfree, cudaStream_t s);
void launch_macro_cg(const MacroDev& M, const double* val, const double* diag, const double* rhs,
                     double scale, double rtol, int max_iter, double* x, double* work,
                     CgState* st, cudaStream_t s);
bool launch_macro_cg_cluster(const MacroDev& M, int max_slice_nnz, const double* val, const double* diag,
                             const double* rhs, double scale, double rtol, int max_iter, double* x, double* p,
                             CgState* st, cudaStream_t s);
void launch_norm(const double* v, int n, double* out, cudaStream_t s);
void launch_spmv(const MacroDev& M, const double* val, const double* x, double* y, cudaStream_t s);
// persistent cooperative PCG for meshes beyond one cluster (one CTA per SM); false if it does not fit
bool launch_macro_cg_grid(const MacroDev& M, const double* val, const double* rhs, double scale, double rtol,
                          int max_iter, double* x, double* zg, double* part, CgState* st, cudaStream_t s,
                          int* extra_launches = nullptr);
void launch_macro_cg_large(const MacroDev& M, const double* val, const double* diag, const double* rhs,
                           double scale, double rtol, int max_iter, double* xout, double* work, double* sc,
                           double* part, CgState* st, cudaStream_t s);
// column windows of the node-aligned CSR slices for cluster size G (see MacroDev::cg_win)
void cg2_windows(const MacroDev& M, const int* host_rowptr, const int* host_col, int G, int* win, int* wmax,
                 int* wok);
void cg2_slice_sizes(const MacroDev& M, const int* host_rowptr, int G, int* max_nr, int* max_nnz);
bool launch_macro_cg_cluster2(const MacroDev& M, const int (*slice)[2], const double* val, const double* rhs,
                              double scale, double rtol, int max_iter, double* x, CgState* st, cudaStream_t s,
                              int* extra_launches = nullptr);
// A_c = P^T K_M P and its inverse for the current values (enqueued before the cluster PCG)
bool launch_coarse_setup(const MacroDev& M, const double* val, cudaStream_t s);
void launch_axpy(double* y, const double* x, double a, int n, cudaStream_t s);
// w between the natural (API) and the internal node order (to_api: internal -> natural)
void launch_permute_w(const RveDev& R, int B, const double* src, double* dst, int to_api, cudaStream_t s);
// dense natural-layout K_ff [npad][npad] from the lower tiles of one RVE's pool (Kb)
void launch_expand_kff(const RveDev& R, const double* Kb, double* out, cudaStream_t s);
void launch_recover(const RveDev& R, int b0, int nb, const double* X, const double* kin, double* w,
                    int accumulate, cudaStream_t s);

}  // namespace hom
