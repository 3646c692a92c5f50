/*
 * oracle/hom_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU oracle for the batched RVE condensation
 * and macro solve of Hesch, Schmidt & Schuss, arXiv 2312.12771 ("PAPER.md").
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no source, header,
 * table or generator with the CUDA path (paper_2312_12771_b200/csrc).
 *
 * What it computes:
 *  - per RVE, the effective tangent by the *textbook FE^2 route*: for every
 *    unit macro strain e_j solve the periodic fluctuation problem
 *    K_ff w_j = -K_fe e_j (eq:reduction) with a skyline
 *    (profile) Cholesky, then volume-average the stress (eq:averageStress,
 *    P:136-142): C_eff e_j = |Omega|^-1 sum_qp eta~ C (e_j + B w_j).
 *    This is algebraically the Schur complement of eq:solution1/2
 *     but computed by a different formula and order.
 *  - the finite-strain version: tangent A_eff by the
 *    same unit-gradient route and P_eff = <P + A G z>, z = -K_ff^-1 r_f.
 *  - the macro problem (eq:linSys): K_M = sum eta B^T C_eff B,
 *    Dirichlet DOFs eliminated, solved *directly* by skyline Cholesky.
 *
 * Numbering conventions (shared with the GPU path only through DESIGN.md):
 *  structured grids on [0,L]^d, nodes lexicographic x fastest; local element
 *  node order counter-clockwise (2-D) / bottom-then-top face (3-D); 2-point
 *  Gauss per direction at +-1/sqrt(3), qp order x fastest; Voigt order
 *  [e11,e22,g12] (2-D), [e11,e22,e33,g23,g13,g12] (3-D), engineering shear;
 *  full gradient row-major [11,12,21,22].  Periodic independent node
 *  p = (i mod r) + r (j mod r) + r^2 (k mod r); its DOF is dim*p + comp; the
 *  corner class p = 0 is fixed.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_ARG 1
#define ORC_ERR_NOT_SPD 3
#define ORC_ERR_JACOBIAN 4
#define ORC_ERR_OOM 8

#define MAXNEN 8  /* hex8 */
#define MAXM 6    /* 3-D Voigt */
#define MAXQ 8

/* ------------------------------------------------------------------------ */
/* Reference element: multilinear Lagrange on [-1,1]^d.          */
/* ------------------------------------------------------------------------ */

static int nen_of(int dim) { return 1 << dim; }

/* sign of local node a in reference direction k */
static double node_sign(int dim, int a, int k) {
  if (dim == 1) return a == 0 ? -1.0 : 1.0;
  int a2 = a & 3; /* position in the (x,y) face, counter-clockwise */
  if (k == 0) return (a2 == 1 || a2 == 2) ? 1.0 : -1.0;
  if (k == 1) return (a2 >= 2) ? 1.0 : -1.0;
  return (a >= 4) ? 1.0 : -1.0; /* k == 2 */
}

/* integer offset (0 or 1) of local node a in direction k within its cell */
static int node_off(int dim, int a, int k) { return node_sign(dim, a, k) > 0 ? 1 : 0; }

static void gauss_point(int dim, int q, double* xi) {
  const double g = 1.0 / sqrt(3.0);
  for (int k = 0; k < dim; ++k) xi[k] = ((q >> k) & 1) ? g : -g;
}

static void shape(int dim, const double* xi, double* N, double dNdxi[][3]) {
  int nen = nen_of(dim);
  for (int a = 0; a < nen; ++a) {
    double f[3];
    for (int k = 0; k < dim; ++k) f[k] = 0.5 * (1.0 + node_sign(dim, a, k) * xi[k]);
    double n = 1.0;
    for (int k = 0; k < dim; ++k) n *= f[k];
    N[a] = n;
    for (int k = 0; k < dim; ++k) {
      double d = 0.5 * node_sign(dim, a, k);
      for (int l = 0; l < dim; ++l)
        if (l != k) d *= f[l];
      dNdxi[a][k] = d;
    }
  }
}

/* Physical derivatives dN/dx at one point of an element with nodal coords x. */
static double element_derivs(int dim, const double x[][3], const double* xi, double* N,
                             double dNdx[][3]) {
  int nen = nen_of(dim);
  double dNdxi[MAXNEN][3];
  shape(dim, xi, N, dNdxi);
  double J[3][3] = {{0}};
  for (int a = 0; a < nen; ++a)
    for (int i = 0; i < dim; ++i)
      for (int j = 0; j < dim; ++j) J[i][j] += x[a][i] * dNdxi[a][j]; /* dx_i/dxi_j */
  double det, Ji[3][3];
  if (dim == 1) {
    det = J[0][0];
    Ji[0][0] = 1.0 / det;
  } else if (dim == 2) {
    det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    Ji[0][0] = J[1][1] / det; Ji[0][1] = -J[0][1] / det;
    Ji[1][0] = -J[1][0] / det; Ji[1][1] = J[0][0] / det;
  } else {
    det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
          J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
          J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
    Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
    Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
    Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
    Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
    Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
    Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
    Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
    Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
  }
  /* dN/dx_i = sum_j dN/dxi_j (J^-1)_{j i} */
  for (int a = 0; a < nen; ++a)
    for (int i = 0; i < dim; ++i) {
      double s = 0;
      for (int j = 0; j < dim; ++j) s += dNdxi[a][j] * Ji[j][i];
      dNdx[a][i] = s;
    }
  return det;
}

/* ------------------------------------------------------------------------ */
/* Strain operators.                                                         */
/* kind 0: small-strain Voigt (m = 1, 3, 6); kind 1: full gradient (m = d^2) */
/* ------------------------------------------------------------------------ */

static int m_of(int dim, int kind) {
  if (kind == 1) return dim * dim;
  return dim == 1 ? 1 : (dim == 2 ? 3 : 6);
}

/* Bm[row][a*dim + c]: strain component `row` per unit nodal value (a, c). */
static void strain_operator(int dim, int kind, const double dNdx[][3], double Bm[][MAXNEN * 3]) {
  int nen = nen_of(dim), m = m_of(dim, kind), nd = nen * dim;
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < nd; ++j) Bm[i][j] = 0.0;
  for (int a = 0; a < nen; ++a) {
    const double* g = dNdx[a];
    if (kind == 1) { /* grad u (i,J) = du_i/dX_J, row-major i*dim+J */
      for (int i = 0; i < dim; ++i)
        for (int J = 0; J < dim; ++J) Bm[i * dim + J][a * dim + i] = g[J];
    } else if (dim == 1) {
      Bm[0][a] = g[0];
    } else if (dim == 2) {
      Bm[0][a * 2 + 0] = g[0];
      Bm[1][a * 2 + 1] = g[1];
      Bm[2][a * 2 + 0] = g[1];
      Bm[2][a * 2 + 1] = g[0];
    } else {
      Bm[0][a * 3 + 0] = g[0];
      Bm[1][a * 3 + 1] = g[1];
      Bm[2][a * 3 + 2] = g[2];
      Bm[3][a * 3 + 1] = g[2]; Bm[3][a * 3 + 2] = g[1]; /* g23 */
      Bm[4][a * 3 + 0] = g[2]; Bm[4][a * 3 + 2] = g[0]; /* g13 */
      Bm[5][a * 3 + 0] = g[1]; Bm[5][a * 3 + 1] = g[0]; /* g12 */
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Materials.                                                                */
/* ------------------------------------------------------------------------ */

/* Isotropic linear elasticity, plane strain in 2-D (reading R7):
 * C = lambda 1(x)1 + 2 mu I_sym in Voigt form with engineering shear. */
int orc_linear_C(int dim, double E, double nu, double* C) {
  double lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
  double mu = E / (2.0 * (1.0 + nu));
  int m = m_of(dim, 0), nn = dim; /* normal components come first */
  if (dim == 1) { C[0] = E; return ORC_OK; }
  for (int i = 0; i < m * m; ++i) C[i] = 0.0;
  for (int i = 0; i < nn; ++i)
    for (int j = 0; j < nn; ++j) C[i * m + j] = lam + (i == j ? 2.0 * mu : 0.0);
  for (int i = nn; i < m; ++i) C[i * m + i] = mu;
  return ORC_OK;
}

/* The paper's Cook energy, written out:
 *   Psi = alpha (F:F - 2) + beta (F:F + J^2 - 3) + kappa/2 (J-1)^2 - 2 (alpha + 2 beta) ln J,
 * 2-D, J = det F.  Differentiated term by term with dJ/dF = H = cof F:
 *   P = 2 alpha F + beta (2 F + 2 J H) + kappa (J-1) H - 2 (alpha + 2 beta) / J H,
 *   A = dP/dF,  both row-major (i,J).  beta = 0 is the config-5 reading R11. */
int orc_mr_material(const double* F, double alpha, double beta, double kappa, double* psi, double* P,
                    double* A) {
  double J = F[0] * F[3] - F[1] * F[2];
  if (!(J > 0.0)) return ORC_ERR_JACOBIAN;
  /* cofactor H = dJ/dF, 2-D specialisation of (1/2) F xx F */
  double H[4] = {F[3], -F[2], -F[1], F[0]};
  double FF = F[0] * F[0] + F[1] * F[1] + F[2] * F[2] + F[3] * F[3];
  if (psi)
    *psi = alpha * (FF - 2.0) + beta * (FF + J * J - 3.0) + 0.5 * kappa * (J - 1.0) * (J - 1.0) -
           2.0 * (alpha + 2.0 * beta) * log(J);
  /* s = dPsi/dJ of the J-dependent terms: 2 beta J + kappa (J-1) - 2 (alpha + 2 beta)/J */
  double s = 2.0 * beta * J + kappa * (J - 1.0) - 2.0 * (alpha + 2.0 * beta) / J;
  /* P = dPsi/dF = 2 alpha F + 2 beta F + s H, term by term as differentiated above (plain form;
   * at F = I the terms cancel to round-off, which the parity tests allow for, R23) */
  for (int i = 0; i < 4; ++i) P[i] = 2.0 * alpha * F[i] + 2.0 * beta * F[i] + s * H[i];
  if (A) {
    double t = 2.0 * beta + kappa + 2.0 * (alpha + 2.0 * beta) / (J * J); /* d2Psi/dJ2 */
    /* dH/dF: H11=F22, H12=-F21, H21=-F12, H22=F11 */
    double dH[4][4] = {{0, 0, 0, 1}, {0, 0, -1, 0}, {0, -1, 0, 0}, {1, 0, 0, 0}};
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j)
        A[i * 4 + j] = (i == j ? 2.0 * (alpha + beta) : 0.0) + t * H[i] * H[j] + s * dH[i][j];
  }
  return ORC_OK;
}
int orc_nh_material(const double* F, double alpha, double kappa, double* psi, double* P, double* A) {
  return orc_mr_material(F, alpha, 0.0, kappa, psi, P, A);
}

/* ------------------------------------------------------------------------ */
/* Skyline (profile) symmetric storage + Cholesky.                           */
/* Row j stores columns first[j]..j.                                         */
/* ------------------------------------------------------------------------ */

typedef struct {
  int n;
  int* first;
  long* off;
  double* a;
} sky_t;

static void sky_free(sky_t* s) {
  free(s->first); free(s->off); free(s->a);
  s->first = NULL; s->off = NULL; s->a = NULL;
}

static int sky_alloc(sky_t* s) {
  s->off = (long*)malloc(sizeof(long) * (s->n + 1));
  if (!s->off) return ORC_ERR_OOM;
  s->off[0] = 0;
  for (int j = 0; j < s->n; ++j) s->off[j + 1] = s->off[j] + (j - s->first[j] + 1);
  s->a = (double*)calloc((size_t)s->off[s->n] + 1, sizeof(double));
  return s->a ? ORC_OK : ORC_ERR_OOM;
}

static double* sky_at(sky_t* s, int i, int j) { /* requires first[max] <= min */
  if (i < j) { int t = i; i = j; j = t; }
  return &s->a[s->off[i] + (j - s->first[i])];
}

static int sky_cholesky(sky_t* s) {
  for (int j = 0; j < s->n; ++j) {
    double* Lj = &s->a[s->off[j] - s->first[j]]; /* Lj[k] = L(j,k) */
    for (int i = s->first[j]; i < j; ++i) {
      double* Li = &s->a[s->off[i] - s->first[i]];
      int k0 = s->first[i] > s->first[j] ? s->first[i] : s->first[j];
      double v = Lj[i];
      for (int k = k0; k < i; ++k) v -= Li[k] * Lj[k];
      Lj[i] = v / Li[i];
    }
    double d = Lj[j];
    for (int k = s->first[j]; k < j; ++k) d -= Lj[k] * Lj[k];
    if (!(d > 0.0)) return -(j + 1);
    Lj[j] = sqrt(d);
  }
  return 0;
}

static void sky_solve(const sky_t* s, double* x) {
  for (int j = 0; j < s->n; ++j) { /* L y = b */
    const double* Lj = &s->a[s->off[j] - s->first[j]];
    double v = x[j];
    for (int k = s->first[j]; k < j; ++k) v -= Lj[k] * x[k];
    x[j] = v / Lj[j];
  }
  for (int j = s->n - 1; j >= 0; --j) { /* L^T x = y */
    const double* Lj = &s->a[s->off[j] - s->first[j]];
    x[j] /= Lj[j];
    for (int k = s->first[j]; k < j; ++k) x[k] -= Lj[k] * x[j];
  }
}

/* ------------------------------------------------------------------------ */
/* Structured grids.                                                         */
/* ------------------------------------------------------------------------ */

typedef struct {
  int dim, r, nen, nnode, nelem;
  double L;
  const double* xc; /* explicit mesh (macro problems on mapped / unstructured meshes) or NULL */
  const int* conn;
  const double* axes; /* tensor-product grid: node coordinate k along axis d at axes[d*(r+1)+k]; NULL = uniform */
} grid_t;

static void grid_init(grid_t* g, int dim, int r, double L) {
  g->dim = dim; g->r = r; g->L = L; g->nen = nen_of(dim);
  g->xc = NULL; g->conn = NULL; g->axes = NULL;
  g->nnode = 1; g->nelem = 1;
  for (int k = 0; k < dim; ++k) { g->nnode *= (r + 1); g->nelem *= r; }
}

static void mesh_init(grid_t* g, int dim, int nnode, int nelem, const double* xc, const int* conn) {
  g->axes = NULL;
  g->dim = dim; g->r = -1; g->L = 0.0; g->nen = nen_of(dim);
  g->nnode = nnode; g->nelem = nelem; g->xc = xc; g->conn = conn;
}

static void grid_elem(const grid_t* g, int e, int* nodes, double x[][3]) {
  if (g->conn) { /* explicit mesh: same local node order as the structured grid */
    for (int a = 0; a < g->nen; ++a) {
      nodes[a] = g->conn[e * g->nen + a];
      for (int k = 0; k < 3; ++k) x[a][k] = k < g->dim ? g->xc[(size_t)nodes[a] * g->dim + k] : 0.0;
    }
    return;
  }
  int idx[3] = {0, 0, 0}, t = e;
  for (int k = 0; k < g->dim; ++k) { idx[k] = t % g->r; t /= g->r; }
  double h = g->L / g->r;
  for (int a = 0; a < g->nen; ++a) {
    int n = 0, stride = 1;
    for (int k = 0; k < g->dim; ++k) {
      int ik = idx[k] + node_off(g->dim, a, k);
      n += ik * stride;
      stride *= (g->r + 1);
      x[a][k] = g->axes ? g->axes[k * (g->r + 1) + ik] : ik * h;
    }
    nodes[a] = n;
  }
}

static void grid_node_ijk(const grid_t* g, int n, int* ijk) {
  for (int k = 0; k < 3; ++k) ijk[k] = 0;
  for (int k = 0; k < g->dim; ++k) { ijk[k] = n % (g->r + 1); n /= (g->r + 1); }
}

/* ------------------------------------------------------------------------ */
/* RVE equation numbering.                                                   */
/* mode 0: periodic (iii) + corner fix; mode 1: w = 0 on boundary (ii);      */
/* mode 2: w = 0 everywhere (i, Taylor).  (eq:Con)     */
/* ------------------------------------------------------------------------ */

static int fold(int i, int r) { return (i <= r - 1 - i) ? 2 * i : 2 * (r - 1 - i) + 1; }

typedef struct {
  int neq;
  int* eq;    /* [nnode*dim] equation number of full-grid DOF, -1 if fixed */
  int* indep; /* [nnode] periodic independent node (mode 0) */
} rvemap_t;

static int rvemap_build(const grid_t* g, int mode, rvemap_t* mp) {
  int dim = g->dim, r = g->r;
  mp->eq = (int*)malloc(sizeof(int) * g->nnode * dim);
  mp->indep = (int*)malloc(sizeof(int) * g->nnode);
  if (!mp->eq || !mp->indep) return ORC_ERR_OOM;
  int nind = 1;
  for (int k = 0; k < dim; ++k) nind *= r;
  if (mode == 0) {
    /* equation numbers by folded lexicographic order of independent nodes */
    int* eqp = (int*)malloc(sizeof(int) * nind);
    int* order = (int*)malloc(sizeof(int) * nind);
    for (int p = 0; p < nind; ++p) {
      int t = p, f = 0, stride = 1;
      for (int k = 0; k < dim; ++k) { f += fold(t % r, r) * stride; t /= r; stride *= r; }
      order[f] = p;
    }
    int cnt = 0;
    for (int f = 0; f < nind; ++f) {
      int p = order[f];
      if (p == 0) { eqp[p] = -1; continue; } /* corner class fixed */
      eqp[p] = cnt++;
    }
    mp->neq = cnt * dim;
    for (int n = 0; n < g->nnode; ++n) {
      int ijk[3]; grid_node_ijk(g, n, ijk);
      int p = 0, stride = 1;
      for (int k = 0; k < dim; ++k) { p += (ijk[k] % r) * stride; stride *= r; }
      mp->indep[n] = p;
      for (int c = 0; c < dim; ++c) mp->eq[n * dim + c] = eqp[p] < 0 ? -1 : eqp[p] * dim + c;
    }
    free(eqp); free(order);
  } else {
    int cnt = 0;
    for (int n = 0; n < g->nnode; ++n) {
      int ijk[3]; grid_node_ijk(g, n, ijk);
      int bnd = (mode == 2);
      for (int k = 0; k < dim; ++k) bnd |= (ijk[k] == 0 || ijk[k] == r);
      mp->indep[n] = -1;
      for (int c = 0; c < dim; ++c) mp->eq[n * dim + c] = bnd ? -1 : cnt * dim + c;
      if (!bnd) cnt++;
    }
    mp->neq = cnt * dim;
  }
  return ORC_OK;
}

static void rvemap_free(rvemap_t* mp) { free(mp->eq); free(mp->indep); }

static int sky_profile_from_grid(const grid_t* g, const int* eqmap, int neq, sky_t* s) {
  s->n = neq;
  s->first = (int*)malloc(sizeof(int) * (neq > 0 ? neq : 1));
  if (!s->first) return ORC_ERR_OOM;
  for (int j = 0; j < neq; ++j) s->first[j] = j;
  for (int e = 0; e < g->nelem; ++e) {
    int nodes[MAXNEN]; double x[MAXNEN][3];
    grid_elem(g, e, nodes, x);
    int mn = neq, eqs[MAXNEN * 3], ne = 0;
    for (int a = 0; a < g->nen; ++a)
      for (int c = 0; c < g->dim; ++c) {
        int q = eqmap[nodes[a] * g->dim + c];
        if (q >= 0) { eqs[ne++] = q; if (q < mn) mn = q; }
      }
    for (int i = 0; i < ne; ++i)
      if (s->first[eqs[i]] > mn) s->first[eqs[i]] = mn;
  }
  return sky_alloc(s);
}

/* ------------------------------------------------------------------------ */
/* Linear RVE: effective tangent by unit strains + stress average.           */
/* ------------------------------------------------------------------------ */

/*
 * orc_rve_condense_linear
 *   dim, r, L  : RVE [0,L]^dim with r cells per direction
 *   mode       : 0 periodic+corner, 1 boundary w=0, 2 Taylor
 *   Cq         : [nelem][2^dim][m][m] material tangent at each micro qp
 *   C_eff      : out [m][m]
 *   W          : out (mode 0 only, may be NULL) [m][dim*r^dim]: fluctuation
 *                for unit strain e_j at periodic independent DOF dim*p+c
 *                (i.e. W[j] = -X e_j in the GPU notation)
 * returns 0, ORC_ERR_NOT_SPD, ORC_ERR_OOM
 */
static int rve_condense_linear_ax(int dim, int r, double L, const double* axes, int mode, const double* Cq,
                                  double* C_eff, double* W);
int orc_rve_condense_linear(int dim, int r, double L, int mode, const double* Cq, double* C_eff,
                            double* W) {
  return rve_condense_linear_ax(dim, r, L, NULL, mode, Cq, C_eff, W);
}
/* the same on a tensor-product RVE grid with arbitrary (graded) node coordinates per axis,
 * axes [dim][r+1] ascending (axes[d][0] and axes[d][r] are the periodic faces) */
int orc_rve_condense_linear_axes(int dim, int r, const double* axes, int mode, const double* Cq, double* C_eff,
                                 double* W) {
  return rve_condense_linear_ax(dim, r, 1.0, axes, mode, Cq, C_eff, W);
}
static int rve_condense_linear_ax(int dim, int r, double L, const double* axes, int mode, const double* Cq,
                                  double* C_eff, double* W) {
  if (dim < 1 || dim > 3 || r < 1 || mode < 0 || mode > 2) return ORC_ERR_ARG;
  grid_t g; grid_init(&g, dim, r, L);
  g.axes = axes;
  int m = m_of(dim, 0), nq = 1 << dim, nd = g.nen * dim;
  rvemap_t mp;
  int rc = rvemap_build(&g, mode, &mp);
  if (rc) return rc;
  sky_t K = {0};
  rc = sky_profile_from_grid(&g, mp.eq, mp.neq, &K);
  double* Kfe = (double*)calloc((size_t)(mp.neq > 0 ? mp.neq : 1) * m, sizeof(double));
  double* wj = (double*)malloc(sizeof(double) * (mp.neq > 0 ? mp.neq : 1) * m);
  if (rc || !Kfe || !wj) { rc = ORC_ERR_OOM; goto done; }

  /* assembly of K_ff and K_fe (eq:discreteSys_D, eq:discreteSys_L) */
  double vol = 0.0;
  for (int e = 0; e < g.nelem; ++e) {
    int nodes[MAXNEN]; double x[MAXNEN][3];
    grid_elem(&g, e, nodes, x);
    int eqs[MAXNEN * 3];
    for (int a = 0; a < g.nen; ++a)
      for (int c = 0; c < dim; ++c) eqs[a * dim + c] = mp.eq[nodes[a] * dim + c];
    for (int q = 0; q < nq; ++q) {
      double xi[3], N[MAXNEN], dNdx[MAXNEN][3], Bm[MAXM][MAXNEN * 3];
      gauss_point(dim, q, xi);
      double w = element_derivs(dim, x, xi, N, dNdx); /* Gauss weights are 1 */
      strain_operator(dim, 0, dNdx, Bm);
      const double* C = &Cq[((size_t)e * nq + q) * m * m];
      vol += w;
      double CB[MAXM][MAXNEN * 3];
      for (int i = 0; i < m; ++i)
        for (int j = 0; j < nd; ++j) {
          double v = 0;
          for (int k = 0; k < m; ++k) v += C[i * m + k] * Bm[k][j];
          CB[i][j] = v;
        }
      for (int i = 0; i < nd; ++i) {
        if (eqs[i] < 0) continue;
        for (int j = 0; j < nd; ++j) {
          if (eqs[j] < 0 || eqs[j] > eqs[i]) continue;
          double v = 0;
          for (int k = 0; k < m; ++k) v += Bm[k][i] * CB[k][j];
          *sky_at(&K, eqs[i], eqs[j]) += w * v;
        }
        for (int j = 0; j < m; ++j) {
          double v = 0;
          for (int k = 0; k < m; ++k) v += Bm[k][i] * C[k * m + j];
          Kfe[(size_t)eqs[i] * m + j] += w * v;
        }
      }
    }
  }

  if (mp.neq > 0) {
    int info = sky_cholesky(&K);
    if (info) { rc = ORC_ERR_NOT_SPD; goto done; }
  }
  /* unit strains e_j: K w_j = -K_fe e_j (eq:reduction) */
  for (int j = 0; j < m; ++j) {
    double* v = &wj[(size_t)j * (mp.neq > 0 ? mp.neq : 1)];
    for (int i = 0; i < mp.neq; ++i) v[i] = -Kfe[(size_t)i * m + j];
    if (mp.neq > 0) sky_solve(&K, v);
  }
  /* stress average (eq:averageStress) */
  for (int i = 0; i < m * m; ++i) C_eff[i] = 0.0;
  for (int e = 0; e < g.nelem; ++e) {
    int nodes[MAXNEN]; double x[MAXNEN][3];
    grid_elem(&g, e, nodes, x);
    for (int q = 0; q < nq; ++q) {
      double xi[3], N[MAXNEN], dNdx[MAXNEN][3], Bm[MAXM][MAXNEN * 3];
      gauss_point(dim, q, xi);
      double w = element_derivs(dim, x, xi, N, dNdx);
      strain_operator(dim, 0, dNdx, Bm);
      const double* C = &Cq[((size_t)e * nq + q) * m * m];
      for (int j = 0; j < m; ++j) {
        const double* v = &wj[(size_t)j * (mp.neq > 0 ? mp.neq : 1)];
        double eps[MAXM];
        for (int k = 0; k < m; ++k) eps[k] = (k == j) ? 1.0 : 0.0;
        for (int a = 0; a < g.nen; ++a)
          for (int c = 0; c < dim; ++c) {
            int qe = mp.eq[nodes[a] * dim + c];
            if (qe < 0) continue;
            for (int k = 0; k < m; ++k) eps[k] += Bm[k][a * dim + c] * v[qe];
          }
        for (int i = 0; i < m; ++i) {
          double sig = 0;
          for (int k = 0; k < m; ++k) sig += C[i * m + k] * eps[k];
          C_eff[i * m + j] += w * sig / vol;
        }
      }
    }
  }
  if (W && mode == 0) {
    int nind = 1;
    for (int k = 0; k < dim; ++k) nind *= r;
    int npad = nind * dim;
    for (int j = 0; j < m; ++j) {
      const double* v = &wj[(size_t)j * (mp.neq > 0 ? mp.neq : 1)];
      for (int i = 0; i < npad; ++i) W[(size_t)j * npad + i] = 0.0;
      for (int n = 0; n < g.nnode; ++n)
        for (int c = 0; c < dim; ++c) {
          int qe = mp.eq[n * dim + c];
          W[(size_t)j * npad + mp.indep[n] * dim + c] = qe < 0 ? 0.0 : v[qe];
        }
    }
  }
done:
  free(Kfe); free(wj); sky_free(&K); rvemap_free(&mp);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* Finite-strain RVE (2-D, full gradient, m = 4): one Newton linearisation.  */
/* ------------------------------------------------------------------------ */

/*
 * orc_rve_condense_nh
 *   r, L       : RVE [0,L]^2 with r x r cells, periodic + corner fix
 *   mstride    : 2: mat [n_phase][2] = (alpha, kappa) (beta = 0); 3: (alpha, beta, kappa)
 *   phase      : [r*r] phase per element
 *   Fbar       : [4] macro deformation gradient (row-major)
 *   w          : [2 r^2] current fluctuation (independent DOF 2p+c), or NULL = 0
 * outputs (any may be NULL except A_eff):
 *   A_eff [16] : |Omega|^-1 sum A (e_j + G W_j), W_j = -K^-1 K_fF e_j
 *   P_eff [4]  : |Omega|^-1 sum (P + A G z),     z  = -K^-1 r_f
 *   P_avg [4]  : <P>  (eq:averageStress)
 *   z     [2 r^2], Wout [4][2 r^2] in the independent-DOF layout
 *   rf_norm    : || r_f ||_2 over free DOFs (R_micro)
 * returns 0, ORC_ERR_JACOBIAN (J <= 0 at a micro qp), ORC_ERR_NOT_SPD
 */
int orc_rve_condense_nh(int r, double L, int mstride, const uint8_t* phase, const double* mat,
                        const double* Fbar, const double* w, double* A_eff, double* P_eff, double* P_avg,
                        double* z, double* Wout, double* rf_norm) {
  const int dim = 2, m = 4, nq = 4;
  grid_t g; grid_init(&g, dim, r, L);
  int nd = g.nen * dim, npad = r * r * dim;
  rvemap_t mp;
  int rc = rvemap_build(&g, 0, &mp);
  if (rc) return rc;
  sky_t K = {0};
  rc = sky_profile_from_grid(&g, mp.eq, mp.neq, &K);
  int ne = mp.neq;
  double* KfF = (double*)calloc((size_t)ne * m, sizeof(double));
  double* rf = (double*)calloc((size_t)ne, sizeof(double));
  double* sol = (double*)malloc(sizeof(double) * (size_t)ne * (m + 1));
  if (rc || !KfF || !rf || !sol) { rc = ORC_ERR_OOM; goto done; }
  double vol = 0.0, Aavg[16] = {0}, Pavg[4] = {0};
  for (int e = 0; e < g.nelem; ++e) {
    int nodes[MAXNEN]; double x[MAXNEN][3];
    grid_elem(&g, e, nodes, x);
    int eqs[MAXNEN * 3];
    double we[MAXNEN * 3];
    for (int a = 0; a < g.nen; ++a)
      for (int c = 0; c < dim; ++c) {
        eqs[a * dim + c] = mp.eq[nodes[a] * dim + c];
        we[a * dim + c] = w ? w[mp.indep[nodes[a]] * dim + c] : 0.0;
      }
    const double* pm = &mat[mstride * phase[e]];
    for (int q = 0; q < nq; ++q) {
      double xi[3], N[MAXNEN], dNdx[MAXNEN][3], G[MAXM][MAXNEN * 3];
      gauss_point(dim, q, xi);
      double wq = element_derivs(dim, x, xi, N, dNdx);
      strain_operator(dim, 1, dNdx, G);
      double F[4];
      for (int i = 0; i < 4; ++i) {
        F[i] = Fbar[i];
        for (int j = 0; j < nd; ++j) F[i] += G[i][j] * we[j]; /* eq:microGrad */
      }
      double P[4], A[16];
      if (orc_mr_material(F, pm[0], mstride == 3 ? pm[1] : 0.0, pm[mstride - 1], NULL, P, A)) {
        rc = ORC_ERR_JACOBIAN;
        goto done;
      }
      vol += wq;
      for (int i = 0; i < 16; ++i) Aavg[i] += wq * A[i];
      for (int i = 0; i < 4; ++i) Pavg[i] += wq * P[i];
      for (int i = 0; i < nd; ++i) {
        if (eqs[i] < 0) continue;
        double gp = 0;
        for (int k = 0; k < 4; ++k) gp += G[k][i] * P[k];
        rf[eqs[i]] += wq * gp;
        for (int j = 0; j < nd; ++j) {
          if (eqs[j] < 0 || eqs[j] > eqs[i]) continue;
          double v = 0;
          for (int k = 0; k < 4; ++k)
            for (int l = 0; l < 4; ++l) v += G[k][i] * A[k * 4 + l] * G[l][j];
          *sky_at(&K, eqs[i], eqs[j]) += wq * v;
        }
        for (int j = 0; j < 4; ++j) {
          double v = 0;
          for (int k = 0; k < 4; ++k) v += G[k][i] * A[k * 4 + j];
          KfF[(size_t)eqs[i] * m + j] += wq * v;
        }
      }
    }
  }
  if (rf_norm) {
    double s = 0;
    for (int i = 0; i < ne; ++i) s += rf[i] * rf[i];
    *rf_norm = sqrt(s);
  }
  if (sky_cholesky(&K)) { rc = ORC_ERR_NOT_SPD; goto done; }
  for (int j = 0; j < m; ++j) {
    double* v = &sol[(size_t)j * ne];
    for (int i = 0; i < ne; ++i) v[i] = -KfF[(size_t)i * m + j];
    sky_solve(&K, v);
  }
  {
    double* v = &sol[(size_t)m * ne];
    for (int i = 0; i < ne; ++i) v[i] = -rf[i];
    sky_solve(&K, v);
  }
  /* averages of the linearised response (A_eff, P_eff) */
  double Ae[16] = {0}, Pe[4] = {0};
  for (int e = 0; e < g.nelem; ++e) {
    int nodes[MAXNEN]; double x[MAXNEN][3];
    grid_elem(&g, e, nodes, x);
    double we[MAXNEN * 3];
    for (int a = 0; a < g.nen; ++a)
      for (int c = 0; c < dim; ++c) we[a * dim + c] = w ? w[mp.indep[nodes[a]] * dim + c] : 0.0;
    const double* pm = &mat[mstride * phase[e]];
    for (int q = 0; q < nq; ++q) {
      double xi[3], N[MAXNEN], dNdx[MAXNEN][3], G[MAXM][MAXNEN * 3];
      gauss_point(dim, q, xi);
      double wq = element_derivs(dim, x, xi, N, dNdx);
      strain_operator(dim, 1, dNdx, G);
      double F[4];
      for (int i = 0; i < 4; ++i) {
        F[i] = Fbar[i];
        for (int j = 0; j < nd; ++j) F[i] += G[i][j] * we[j];
      }
      double P[4], A[16];
      orc_mr_material(F, pm[0], mstride == 3 ? pm[1] : 0.0, pm[mstride - 1], NULL, P, A);
      for (int j = 0; j <= m; ++j) { /* j < m: unit gradient e_j; j == m: z */
        const double* v = &sol[(size_t)j * ne];
        double d[4];
        for (int k = 0; k < 4; ++k) d[k] = (j < m && k == j) ? 1.0 : 0.0;
        for (int a = 0; a < g.nen; ++a)
          for (int c = 0; c < dim; ++c) {
            int qe = mp.eq[nodes[a] * dim + c];
            if (qe < 0) continue;
            for (int k = 0; k < 4; ++k) d[k] += G[k][a * dim + c] * v[qe];
          }
        for (int i = 0; i < 4; ++i) {
          double s = 0;
          for (int k = 0; k < 4; ++k) s += A[i * 4 + k] * d[k];
          if (j < m) Ae[i * 4 + j] += wq * s / vol;
          else Pe[i] += wq * (P[i] + s) / vol;
        }
      }
    }
  }
  for (int i = 0; i < 16; ++i) A_eff[i] = Ae[i];
  if (P_eff) for (int i = 0; i < 4; ++i) P_eff[i] = Pe[i];
  if (P_avg) for (int i = 0; i < 4; ++i) P_avg[i] = Pavg[i] / vol;
  (void)Aavg;
  for (int j = 0; j <= m; ++j) {
    double* out = (j < m) ? (Wout ? &Wout[(size_t)j * npad] : NULL) : z;
    if (!out) continue;
    const double* v = &sol[(size_t)j * ne];
    for (int i = 0; i < npad; ++i) out[i] = 0.0;
    for (int n = 0; n < g.nnode; ++n)
      for (int c = 0; c < dim; ++c) {
        int qe = mp.eq[n * dim + c];
        out[mp.indep[n] * dim + c] = qe < 0 ? 0.0 : v[qe];
      }
  }
done:
  free(KfF); free(rf); free(sol); sky_free(&K); rvemap_free(&mp);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* Batched drivers (pthreads over RVEs).                                     */
/* ------------------------------------------------------------------------ */

typedef struct {
  int kind; /* 0 linear, 1 nh */
  int dim, r, n_rve, phase_per_rve, mat_per_rve, n_phase, mstride;
  double L;
  const double* axes; /* linear: tensor-product RVE grid coordinates or NULL */
  const uint8_t* phase;
  const double* mat;
  const double* Fbar; const double* w;
  double *C_eff, *P_eff, *P_avg, *Z, *W, *rf_norm;
  int next, status, bad_rve;
  pthread_mutex_t mu;
} batch_t;

static void* batch_worker(void* arg) {
  batch_t* b = (batch_t*)arg;
  int dim = b->dim, r = b->r, nel = 1, nq = 1 << dim;
  for (int k = 0; k < dim; ++k) nel *= r;
  int m = b->kind == 1 ? 4 : m_of(dim, 0), npad = nel * dim;
  double* Cq = b->kind == 0 ? (double*)malloc(sizeof(double) * (size_t)nel * nq * m * m) : NULL;
  for (;;) {
    pthread_mutex_lock(&b->mu);
    int i = b->next++;
    pthread_mutex_unlock(&b->mu);
    if (i >= b->n_rve) break;
    const uint8_t* ph = b->phase + (b->phase_per_rve ? (size_t)i * nel : 0);
    const double* mt = b->mat + (b->mat_per_rve ? (size_t)i * b->n_phase * b->mstride : 0);
    int rc;
    if (b->kind == 0) {
      for (int e = 0; e < nel; ++e) {
        double C[MAXM * MAXM];
        orc_linear_C(dim, mt[2 * ph[e]], mt[2 * ph[e] + 1], C);
        for (int q = 0; q < nq; ++q) memcpy(&Cq[((size_t)e * nq + q) * m * m], C, sizeof(double) * m * m);
      }
      rc = rve_condense_linear_ax(dim, r, 1.0, b->axes, 0, Cq, &b->C_eff[(size_t)i * m * m],
                                  b->W ? &b->W[(size_t)i * m * npad] : NULL);
    } else {
      rc = orc_rve_condense_nh(r, b->L, b->mstride, ph, mt, &b->Fbar[(size_t)i * 4],
                               b->w ? &b->w[(size_t)i * npad] : NULL,
                               &b->C_eff[(size_t)i * 16], b->P_eff ? &b->P_eff[(size_t)i * 4] : NULL,
                               b->P_avg ? &b->P_avg[(size_t)i * 4] : NULL,
                               b->Z ? &b->Z[(size_t)i * npad] : NULL,
                               b->W ? &b->W[(size_t)i * 4 * npad] : NULL,
                               b->rf_norm ? &b->rf_norm[i] : NULL);
    }
    if (rc) {
      pthread_mutex_lock(&b->mu);
      if (!b->status) { b->status = rc; b->bad_rve = i; }
      pthread_mutex_unlock(&b->mu);
    }
  }
  free(Cq);
  return NULL;
}

static int run_batch(batch_t* b, int nthreads, int* bad_rve) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  b->next = 0; b->status = 0; b->bad_rve = -1;
  pthread_mutex_init(&b->mu, NULL);
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, batch_worker, b);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  pthread_mutex_destroy(&b->mu);
  if (bad_rve) *bad_rve = b->bad_rve;
  return b->status;
}

/* Linear batch: phase [n_rve or 1][r^dim] u8; mat [n_rve or 1][n_phase][2] = (E, nu).
 * C_eff [n_rve][m][m]; W (nullable) [n_rve][m][dim r^dim]. */
int orc_condense_batch_linear(int dim, int r, int n_rve, int phase_per_rve, const uint8_t* phase,
                              int mat_per_rve, int n_phase, const double* mat, double* C_eff,
                              double* W, int nthreads, int* bad_rve) {
  batch_t b;
  memset(&b, 0, sizeof(b));
  b.kind = 0; b.dim = dim; b.r = r; b.n_rve = n_rve; b.phase_per_rve = phase_per_rve; b.mstride = 2; b.L = 1.0;
  b.mat_per_rve = mat_per_rve; b.n_phase = n_phase; b.phase = phase; b.mat = mat;
  b.C_eff = C_eff; b.W = W;
  return run_batch(&b, nthreads, bad_rve);
}

/* Linear batch on a tensor-product (graded) RVE grid: axes [dim][r+1]; otherwise as above. */
int orc_condense_batch_linear_axes(int dim, int r, const double* axes, int n_rve, int phase_per_rve,
                                   const uint8_t* phase, int mat_per_rve, int n_phase, const double* mat,
                                   double* C_eff, double* W, int nthreads, int* bad_rve) {
  batch_t b;
  memset(&b, 0, sizeof(b));
  b.kind = 0; b.dim = dim; b.r = r; b.n_rve = n_rve; b.phase_per_rve = phase_per_rve; b.mstride = 2; b.L = 1.0;
  b.axes = axes;
  b.mat_per_rve = mat_per_rve; b.n_phase = n_phase; b.phase = phase; b.mat = mat;
  b.C_eff = C_eff; b.W = W;
  return run_batch(&b, nthreads, bad_rve);
}

/* Finite-strain batch (2-D, RVE [0,L]^2): mat [.. ][n_phase][mstride] = (alpha, kappa) or
 * (alpha, beta, kappa); Fbar [n_rve][4]; w [n_rve][2 r^2] or NULL; outputs A_eff [n_rve][16],
 * P_eff/P_avg [n_rve][4], Z [n_rve][2r^2], W [n_rve][4][2r^2], rf_norm [n_rve] (nullable
 * except A_eff). */
int orc_condense_batch_nh(int r, double L, int mstride, int n_rve, int phase_per_rve, const uint8_t* phase,
                          int mat_per_rve, int n_phase, const double* mat, const double* Fbar, const double* w,
                          double* A_eff, double* P_eff, double* P_avg, double* Z, double* W,
                          double* rf_norm, int nthreads, int* bad_rve) {
  batch_t b;
  memset(&b, 0, sizeof(b));
  b.kind = 1; b.dim = 2; b.r = r; b.n_rve = n_rve; b.phase_per_rve = phase_per_rve;
  b.mstride = mstride; b.L = L;
  b.mat_per_rve = mat_per_rve; b.n_phase = n_phase; b.phase = phase; b.mat = mat;
  b.Fbar = Fbar; b.w = w; b.C_eff = A_eff; b.P_eff = P_eff; b.P_avg = P_avg; b.Z = Z; b.W = W;
  b.rf_norm = rf_norm;
  return run_batch(&b, nthreads, bad_rve);
}

/* ------------------------------------------------------------------------ */
/* Macro problem on the structured grid [0,Lm]^dim (eq:linSys).    */
/* RVE b = e * 2^dim + q (Dirac basis, one RVE per macro qp).      */
/* ------------------------------------------------------------------------ */

/* kinematics at every macro qp: kind 0 -> Voigt strain, kind 1 -> grad u */
static int macro_kin_g(const grid_t* gp, int kind, const double* u, double* out) {
  const grid_t g = *gp;
  const int dim = g.dim;
  int m = m_of(dim, kind), nq = 1 << dim, nd = g.nen * dim;
  for (int e = 0; e < g.nelem; ++e) {
    int nodes[MAXNEN]; double x[MAXNEN][3];
    grid_elem(&g, e, nodes, x);
    for (int q = 0; q < nq; ++q) {
      double xi[3], N[MAXNEN], dNdx[MAXNEN][3], Bm[MAXM][MAXNEN * 3];
      gauss_point(dim, q, xi);
      element_derivs(dim, x, xi, N, dNdx);
      strain_operator(dim, kind, dNdx, Bm);
      for (int i = 0; i < m; ++i) {
        double s = 0;
        for (int j = 0; j < nd; ++j) s += Bm[i][j] * u[nodes[j / dim] * dim + (j % dim)];
        out[((size_t)e * nq + q) * m + i] = s;
      }
    }
  }
  return ORC_OK;
}

/* R = sum_qp eta B^T S - f_body - f_ext  (all DOFs; S [B][m] stress, nullable; body [dim]
 * nullable; fext [ndof] external nodal forces, nullable) */
static int macro_residual_g(const grid_t* gp, int kind, const double* S, const double* body,
                            const double* fext, double* R) {
  const grid_t g = *gp;
  const int dim = g.dim;
  int m = m_of(dim, kind), nq = 1 << dim, nd = g.nen * dim;
  for (int i = 0; i < g.nnode * dim; ++i) R[i] = 0.0;
  for (int e = 0; e < g.nelem; ++e) {
    int nodes[MAXNEN]; double x[MAXNEN][3];
    grid_elem(&g, e, nodes, x);
    for (int q = 0; q < nq; ++q) {
      double xi[3], N[MAXNEN], dNdx[MAXNEN][3], Bm[MAXM][MAXNEN * 3];
      gauss_point(dim, q, xi);
      double w = element_derivs(dim, x, xi, N, dNdx);
      strain_operator(dim, kind, dNdx, Bm);
      for (int j = 0; j < nd; ++j) {
        int dof = nodes[j / dim] * dim + (j % dim);
        double v = 0;
        if (S)
          for (int i = 0; i < m; ++i) v += Bm[i][j] * S[((size_t)e * nq + q) * m + i];
        if (body) v -= N[j / dim] * body[j % dim];
        R[dof] += w * v;
      }
    }
  }
  if (fext)
    for (int i = 0; i < g.nnode * dim; ++i) R[i] -= fext[i];
  return ORC_OK;
}

/*
 * orc_macro_solve: direct solve of the condensed macro system
 *   K_FF x_F = -(R_F) - K_FD x_D,  K = sum eta B^T D B,  R = sum eta B^T S - f_body
 * D [B][m][m] (C_eff or A_eff), S [B][m] or NULL, body [dim] or NULL,
 * dir_dof [n_dir]; x [n_dof]: in = values at Dirichlet DOFs, out = full vector.
 * Linear: S = NULL, x_D = prescribed u. Newton: S = P_eff, x_D = 0, x = du.
 */
static int macro_solve_g(const grid_t* gp, int kind, const double* D, const double* S,
                         const double* body, const double* fext, int n_dir, const int* dir_dof, double* x) {
  const grid_t g = *gp;
  const int dim = g.dim;
  int m = m_of(dim, kind), nq = 1 << dim, nd = g.nen * dim, ndof = g.nnode * dim;
  int* eq = (int*)malloc(sizeof(int) * ndof);
  double* rhs = (double*)malloc(sizeof(double) * ndof);
  double* R = (double*)malloc(sizeof(double) * ndof);
  sky_t K = {0};
  int rc = ORC_OK;
  if (!eq || !rhs || !R) { rc = ORC_ERR_OOM; goto done; }
  for (int i = 0; i < ndof; ++i) eq[i] = 0;
  for (int i = 0; i < n_dir; ++i) {
    if (dir_dof[i] < 0 || dir_dof[i] >= ndof) { rc = ORC_ERR_ARG; goto done; }
    eq[dir_dof[i]] = -1;
  }
  int neq = 0;
  for (int i = 0; i < ndof; ++i) eq[i] = eq[i] < 0 ? -1 : neq++;
  rc = sky_profile_from_grid(&g, eq, neq, &K);
  if (rc) goto done;
  macro_residual_g(&g, kind, S, body, fext, R);
  for (int i = 0; i < neq; ++i) rhs[i] = 0.0;
  for (int i = 0; i < ndof; ++i)
    if (eq[i] >= 0) rhs[eq[i]] = -R[i];
  for (int e = 0; e < g.nelem; ++e) {
    int nodes[MAXNEN]; double xx[MAXNEN][3];
    grid_elem(&g, e, nodes, xx);
    int dofs[MAXNEN * 3];
    for (int j = 0; j < nd; ++j) dofs[j] = nodes[j / dim] * dim + (j % dim);
    for (int q = 0; q < nq; ++q) {
      double xi[3], N[MAXNEN], dNdx[MAXNEN][3], Bm[MAXM][MAXNEN * 3];
      gauss_point(dim, q, xi);
      double w = element_derivs(dim, xx, xi, N, dNdx);
      strain_operator(dim, kind, dNdx, Bm);
      const double* Dq = &D[((size_t)e * nq + q) * m * m];
      for (int i = 0; i < nd; ++i) {
        int ei = eq[dofs[i]];
        if (ei < 0) continue;
        for (int j = 0; j < nd; ++j) {
          double v = 0;
          for (int k = 0; k < m; ++k)
            for (int l = 0; l < m; ++l) v += Bm[k][i] * Dq[k * m + l] * Bm[l][j];
          v *= w;
          int ej = eq[dofs[j]];
          if (ej < 0) rhs[ei] -= v * x[dofs[j]]; /* Dirichlet lifting */
          else if (ej <= ei) *sky_at(&K, ei, ej) += v;
        }
      }
    }
  }
  if (neq > 0) {
    if (sky_cholesky(&K)) { rc = ORC_ERR_NOT_SPD; goto done; }
    sky_solve(&K, rhs);
  }
  for (int i = 0; i < ndof; ++i)
    if (eq[i] >= 0) x[i] = rhs[eq[i]];
done:
  free(eq); free(rhs); free(R); sky_free(&K);
  return rc;
}

/* structured grid [0,Lm]^dim with nel cells per direction */
int orc_macro_kin(int dim, int nel, double Lm, int kind, const double* u, double* out) {
  grid_t g; grid_init(&g, dim, nel, Lm);
  return macro_kin_g(&g, kind, u, out);
}
int orc_macro_residual(int dim, int nel, double Lm, int kind, const double* S, const double* body,
                       double* R) {
  grid_t g; grid_init(&g, dim, nel, Lm);
  return macro_residual_g(&g, kind, S, body, NULL, R);
}
int orc_macro_solve(int dim, int nel, double Lm, int kind, const double* D, const double* S,
                    const double* body, int n_dir, const int* dir_dof, double* x) {
  grid_t g; grid_init(&g, dim, nel, Lm);
  return macro_solve_g(&g, kind, D, S, body, NULL, n_dir, dir_dof, x);
}
/* explicit macro mesh: coords [nnode][dim], conn [nelem][2^dim] (grid local order), external
 * nodal forces fext [nnode*dim] (nullable) -- the Cook membrane of PAPER.md §4.2 */
int orc_mesh_macro_kin(int dim, int nnode, int nelem, const double* xc, const int* conn, int kind,
                       const double* u, double* out) {
  grid_t g; mesh_init(&g, dim, nnode, nelem, xc, conn);
  return macro_kin_g(&g, kind, u, out);
}
int orc_mesh_macro_residual(int dim, int nnode, int nelem, const double* xc, const int* conn, int kind,
                            const double* S, const double* body, const double* fext, double* R) {
  grid_t g; mesh_init(&g, dim, nnode, nelem, xc, conn);
  return macro_residual_g(&g, kind, S, body, fext, R);
}
int orc_mesh_macro_solve(int dim, int nnode, int nelem, const double* xc, const int* conn, int kind,
                         const double* D, const double* S, const double* body, const double* fext, int n_dir,
                         const int* dir_dof, double* x) {
  grid_t g; mesh_init(&g, dim, nnode, nelem, xc, conn);
  return macro_solve_g(&g, kind, D, S, body, fext, n_dir, dir_dof, x);
}

/* ------------------------------------------------------------------------ */
/* Piecewise-constant macro fluctuation basis (eq:constSolution1/2), */
/* small strain.  One fluctuation field per macro element e; its micro         */
/* equilibrium integrated over the element gives w_e = -K_ff^-1 K_fe eps_bar_e */
/* with the element-average strain eps_bar_e = |B_e|^-1 int_e eps dV; inserted */
/* in the macro equation the element stiffness becomes                         */
/*   K_e = int_e B^T <C>_e B dV - |B_e|^-1 (int_e B dV)^T (<C>_e - C_eff,e) (int_e B dV). */
/* ------------------------------------------------------------------------ */
int orc_macro_kin_const(int dim, int nel, double Lm, const double* u, double* out) {
  grid_t g; grid_init(&g, dim, nel, Lm);
  int m = m_of(dim, 0), nq = 1 << dim, nd = g.nen * dim;
  for (int e = 0; e < g.nelem; ++e) {
    int nodes[MAXNEN]; double x[MAXNEN][3];
    grid_elem(&g, e, nodes, x);
    double acc[MAXM] = {0}, vol = 0.0;
    for (int q = 0; q < nq; ++q) {
      double xi[3], N[MAXNEN], dNdx[MAXNEN][3], Bm[MAXM][MAXNEN * 3];
      gauss_point(dim, q, xi);
      double w = element_derivs(dim, x, xi, N, dNdx);
      strain_operator(dim, 0, dNdx, Bm);
      vol += w;
      for (int i = 0; i < m; ++i)
        for (int j = 0; j < nd; ++j) acc[i] += w * Bm[i][j] * u[nodes[j / dim] * dim + (j % dim)];
    }
    for (int i = 0; i < m; ++i) out[(size_t)e * m + i] = acc[i] / vol;
  }
  return ORC_OK;
}

int orc_macro_solve_const(int dim, int nel, double Lm, const double* Cavg, const double* Ceff,
                          const double* body, int n_dir, const int* dir_dof, double* x) {
  grid_t g; grid_init(&g, dim, nel, Lm);
  int m = m_of(dim, 0), nq = 1 << dim, nd = g.nen * dim, ndof = g.nnode * dim;
  int* eq = (int*)malloc(sizeof(int) * ndof);
  double* rhs = (double*)malloc(sizeof(double) * ndof);
  double* R = (double*)malloc(sizeof(double) * ndof);
  sky_t K = {0};
  int rc = ORC_OK;
  if (!eq || !rhs || !R) { rc = ORC_ERR_OOM; goto done; }
  for (int i = 0; i < ndof; ++i) eq[i] = 0;
  for (int i = 0; i < n_dir; ++i) {
    if (dir_dof[i] < 0 || dir_dof[i] >= ndof) { rc = ORC_ERR_ARG; goto done; }
    eq[dir_dof[i]] = -1;
  }
  int neq = 0;
  for (int i = 0; i < ndof; ++i) eq[i] = eq[i] < 0 ? -1 : neq++;
  rc = sky_profile_from_grid(&g, eq, neq, &K);
  if (rc) goto done;
  macro_residual_g(&g, 0, NULL, body, NULL, R);
  for (int i = 0; i < neq; ++i) rhs[i] = 0.0;
  for (int i = 0; i < ndof; ++i)
    if (eq[i] >= 0) rhs[eq[i]] = -R[i];
  for (int e = 0; e < g.nelem; ++e) {
    int nodes[MAXNEN]; double xx[MAXNEN][3];
    grid_elem(&g, e, nodes, xx);
    int dofs[MAXNEN * 3];
    for (int j = 0; j < nd; ++j) dofs[j] = nodes[j / dim] * dim + (j % dim);
    const double* Ca = &Cavg[(size_t)e * m * m];
    const double* Ce = &Ceff[(size_t)e * m * m];
    double Ke[MAXNEN * 3][MAXNEN * 3], Bbar[MAXM][MAXNEN * 3], vol = 0.0;
    memset(Ke, 0, sizeof(Ke));
    memset(Bbar, 0, sizeof(Bbar));
    for (int q = 0; q < nq; ++q) {
      double xi[3], N[MAXNEN], dNdx[MAXNEN][3], Bm[MAXM][MAXNEN * 3];
      gauss_point(dim, q, xi);
      double w = element_derivs(dim, xx, xi, N, dNdx);
      strain_operator(dim, 0, dNdx, Bm);
      vol += w;
      for (int k = 0; k < m; ++k)
        for (int i = 0; i < nd; ++i) Bbar[k][i] += w * Bm[k][i];
      for (int i = 0; i < nd; ++i)
        for (int j = 0; j < nd; ++j) {
          double v = 0;
          for (int k = 0; k < m; ++k)
            for (int l = 0; l < m; ++l) v += Bm[k][i] * Ca[k * m + l] * Bm[l][j];
          Ke[i][j] += w * v;
        }
    }
    for (int i = 0; i < nd; ++i)
      for (int j = 0; j < nd; ++j) {
        double v = 0;
        for (int k = 0; k < m; ++k)
          for (int l = 0; l < m; ++l) v += Bbar[k][i] * (Ca[k * m + l] - Ce[k * m + l]) * Bbar[l][j];
        Ke[i][j] -= v / vol;
      }
    for (int i = 0; i < nd; ++i) {
      int ei = eq[dofs[i]];
      if (ei < 0) continue;
      for (int j = 0; j < nd; ++j) {
        int ej = eq[dofs[j]];
        if (ej < 0) rhs[ei] -= Ke[i][j] * x[dofs[j]];
        else if (ej <= ei) *sky_at(&K, ei, ej) += Ke[i][j];
      }
    }
  }
  if (neq > 0) {
    if (sky_cholesky(&K)) { rc = ORC_ERR_NOT_SPD; goto done; }
    sky_solve(&K, rhs);
  }
  for (int i = 0; i < ndof; ++i)
    if (eq[i] >= 0) x[i] = rhs[eq[i]];
done:
  free(eq); free(rhs); free(R); sky_free(&K);
  return rc;
}

/* Dense symmetric check helper for tests: skyline solve of a small SPD dense matrix
 * (row-major n x n) -- used to pin the skyline routine against a textbook solve. */
int orc_dense_spd_solve(int n, const double* A, double* x) {
  sky_t s = {0};
  s.n = n;
  s.first = (int*)malloc(sizeof(int) * n);
  if (!s.first) return ORC_ERR_OOM;
  for (int j = 0; j < n; ++j) {
    s.first[j] = j;
    for (int i = 0; i < j; ++i)
      if (A[(size_t)j * n + i] != 0.0) { s.first[j] = i; break; }
  }
  if (sky_alloc(&s)) { sky_free(&s); return ORC_ERR_OOM; }
  for (int j = 0; j < n; ++j)
    for (int i = s.first[j]; i <= j; ++i) *sky_at(&s, j, i) = A[(size_t)j * n + i];
  int rc = sky_cholesky(&s) ? ORC_ERR_NOT_SPD : ORC_OK;
  if (!rc) sky_solve(&s, x);
  sky_free(&s);
  return rc;
}
