/*
 * fem_oracle.c -- plain, slow, obviously-correct CPU oracle for the hot path of
 * arXiv 2308.09839 ("low-order matrix-free FE operators in CG").
 *
 * THIS IS TEST INFRASTRUCTURE, NOT THE PRODUCT.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  It shares no code,
 * header, table or constant generator with the CUDA path (paper_2308_09839_b200/csrc).
 *
 * Citations: "P:n" = line n of the paper text (reference PAPER.md), "S:n" = SPEC.md line n.
 * Every function names the passage it follows.  Arithmetic is IEEE fp64; build with
 * -O2 -ffp-contract=off so that no FMA contraction changes rounding (reading R10).
 *
 * What is computed (readings R1-R7):
 *   A^e by 2x2x2 Gauss-Legendre quadrature of Eq. 4 / 5 / 6 with the
 *   isoparametric map J = sum_j x_j (x) grad^phi_j  (Alg. 1 line "Calculate Jacobian"),
 *   v^e = A^e u^e, assembled by the three-step gather/multiply/scatter of P:188-196,
 *   Dirichlet as y = P A P x + (I - P) x, all 6 box faces, all components.
 *   CG: Hestenes-Stiefel with the recurrences of Table 4.
 *
 * Element node ordering (reading R2): VTK hexahedron
 *   a : 0       1       2       3       4       5       6       7
 *   d : (0,0,0) (1,0,0) (1,1,0) (0,1,0) (0,0,1) (1,0,1) (1,1,1) (0,1,1)
 * Global numbering: node n = i + (nx+1)(j + (ny+1)k), DOF = c*n + comp.
 *
 * Parity status: every function here is pinned by tests/test_oracle_pins.py (closed forms,
 * exact rational integration, Kronecker identities, null spaces, dense solves); see DESIGN.md.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_SCALAR 0
#define ORC_VECTOR 1
#define ORC_ELASTIC 2

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_EGEOM 2
#define ORC_EBREAKDOWN 3
#define ORC_ENOMEM 4

/* Corner offsets of the VTK ordering (reading R2). */
static const int CORNER[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                                 {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};

/* ---------------------------------------------------------------------------------------
 * Reference element ("lowest-order nodal basis", "Gaussian quadrature")
 * phi^_a(xi) = prod_d (1 + s_ad xi_d) / 2, s_ad = 2*CORNER[a][d] - 1.
 * ------------------------------------------------------------------------------------- */
void orc_basis_values(const double xi[3], double phi[8]) {
  for (int a = 0; a < 8; ++a) {
    double v = 1.0;
    for (int d = 0; d < 3; ++d) {
      double s = 2.0 * CORNER[a][d] - 1.0;
      v *= 0.5 * (1.0 + s * xi[d]);
    }
    phi[a] = v;
  }
}

/* grad^ phi^_a(xi): d/dxi_d of the product above. dphi[a][d]. */
void orc_basis_gradients(const double xi[3], double dphi[8][3]) {
  for (int a = 0; a < 8; ++a) {
    for (int d = 0; d < 3; ++d) {
      double g = 1.0;
      for (int e = 0; e < 3; ++e) {
        double s = 2.0 * CORNER[a][e] - 1.0;
        if (e == d)
          g *= 0.5 * s;
        else
          g *= 0.5 * (1.0 + s * xi[e]);
      }
      dphi[a][d] = g;
    }
  }
}

/* Quadrature rule of every element matrix below (reading R1):
 *   ORC_GAUSS (default): 2-point Gauss-Legendre per direction, +-1/sqrt(3), weight 1;
 *   ORC_GLL: 2-point Gauss-Lobatto-Legendre, +-1 (the nodes), weight 1 -- the quadrature of the
 *            CEED benchmark problems BP5/BP6 the paper names (SURVEY
 *            §8(c) item 1), collocated with the Q1 nodes.
 * A process-wide setting (the oracle is single-threaded at this level); orc_set_quadrature
 * returns the previous rule. */
#define ORC_GAUSS 0
#define ORC_GLL 1
static int g_rule = ORC_GAUSS;
int orc_set_quadrature(int rule) {
  const int old = g_rule;
  g_rule = (rule == ORC_GLL) ? ORC_GLL : ORC_GAUSS;
  return old;
}

/* Quadrature point q uses the same corner pattern as node q. */
void orc_reference_element(double xq[8][3], double wq[8], double dphi[8][8][3], double phi[8][8]) {
  const double g = (g_rule == ORC_GLL) ? 1.0 : 1.0 / sqrt(3.0);
  for (int q = 0; q < 8; ++q) {
    for (int d = 0; d < 3; ++d) xq[q][d] = (2.0 * CORNER[q][d] - 1.0) * g;
    wq[q] = 1.0;
    orc_basis_gradients(xq[q], dphi[q]);
    orc_basis_values(xq[q], phi[q]);
  }
}

/* ---------------------------------------------------------------------------------------
 * 3x3 helpers for J, det J, J^{-1} (Alg. 1 lines P:335-337).
 * ------------------------------------------------------------------------------------- */
static double det3(const double J[3][3]) {
  return J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
         J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
         J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
}

static void inv3(const double J[3][3], double det, double Ji[3][3]) {
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

/* Isotropic linear elastic law (reading R4; "appropriate constitutive law", P:12
 * "isotropic"): sigma = lambda tr(eps) I + 2 mu eps, eps = sym(grad u). */
static void constitutive(const double gradu[3][3], double lam, double mu, double sig[3][3]) {
  double eps[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) eps[i][j] = 0.5 * (gradu[i][j] + gradu[j][i]);
  double tr = eps[0][0] + eps[1][1] + eps[2][2];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) sig[i][j] = 2.0 * mu * eps[i][j] + (i == j ? lam * tr : 0.0);
}

/* ---------------------------------------------------------------------------------------
 * Local element matrix by quadrature, Eq. 4 / 5 / 6, row/col index 3(i-1)+k
 * (0-based: c*a + k).  X[a][d] are the 8 nodal coordinates.  Ae is (8c)x(8c) row-major.
 * Returns ORC_EGEOM if det J <= 0 at any point.
 * ------------------------------------------------------------------------------------- */
int orc_element_matrix(int kind, const double X[8][3], double lam, double mu, double* Ae) {
  double xq[8][3], wq[8], dphi[8][8][3], phi[8][8];
  orc_reference_element(xq, wq, dphi, phi);
  const int c = (kind == ORC_SCALAR) ? 1 : 3;
  const int n = 8 * c;
  memset(Ae, 0, sizeof(double) * n * n);
  for (int q = 0; q < 8; ++q) {
    /* J = sum_j x_j (x) grad^phi_j : J[d][e] = sum_j X[j][d] dphi[q][j][e] */
    double J[3][3] = {{0}};
    for (int j = 0; j < 8; ++j)
      for (int d = 0; d < 3; ++d)
        for (int e = 0; e < 3; ++e) J[d][e] += X[j][d] * dphi[q][j][e];
    double detJ = det3(J);
    if (!(detJ > 0.0)) return ORC_EGEOM;
    double Ji[3][3];
    inv3(J, detJ, Ji);
    /* physical gradients G_a = J^{-T} grad^phi_a : G[a][d] = sum_e Ji[e][d] dphi[q][a][e] */
    double G[8][3];
    for (int a = 0; a < 8; ++a)
      for (int d = 0; d < 3; ++d) {
        double s = 0.0;
        for (int e = 0; e < 3; ++e) s += Ji[e][d] * dphi[q][a][e];
        G[a][d] = s;
      }
    const double wdet = wq[q] * detJ;
    for (int a = 0; a < 8; ++a) {
      for (int b = 0; b < 8; ++b) {
        double GaGb = G[a][0] * G[b][0] + G[a][1] * G[b][1] + G[a][2] * G[b][2];
        if (kind == ORC_SCALAR) {
          /* Eq. 4 */
          Ae[a * n + b] += GaGb * wdet;
        } else if (kind == ORC_VECTOR) {
          /* Eq. 5 (l->j typo at P:121 read as j, reading R8):
           * (e_k (x) G_a) : (e_l (x) G_b) = delta_kl G_a . G_b */
          for (int k = 0; k < 3; ++k)
            for (int l = 0; l < 3; ++l) {
              double t = 0.0;
              for (int i = 0; i < 3; ++i)
                for (int jj = 0; jj < 3; ++jj) {
                  double A_ij = (i == k) ? G[a][jj] : 0.0; /* (e_k (x) G_a)_ij */
                  double B_ij = (i == l) ? G[b][jj] : 0.0; /* (e_l (x) G_b)_ij */
                  t += A_ij * B_ij;
                }
              Ae[(3 * a + k) * n + 3 * b + l] += t * wdet;
            }
        } else {
          /* Eq. 6: (e_k (x) G_a) : sigma(e_l (x) G_b) */
          for (int l = 0; l < 3; ++l) {
            double gradu[3][3] = {{0}};
            for (int jj = 0; jj < 3; ++jj) gradu[l][jj] = G[b][jj]; /* e_l (x) G_b */
            double sig[3][3];
            constitutive(gradu, lam, mu, sig);
            for (int k = 0; k < 3; ++k) {
              double t = 0.0;
              for (int jj = 0; jj < 3; ++jj) t += G[a][jj] * sig[k][jj]; /* (e_k (x) G_a):sig */
              Ae[(3 * a + k) * n + 3 * b + l] += t * wdet;
            }
          }
        }
      }
    }
  }
  return ORC_OK;
}

/* ---------------------------------------------------------------------------------------
 * Mesh: box of nx*ny*nz cubes of side h, node (i h, j h, k h).
 * ------------------------------------------------------------------------------------- */
static int64_t node_id(int64_t i, int64_t j, int64_t k, int64_t nx, int64_t ny) {
  return i + (nx + 1) * (j + (ny + 1) * k);
}

int orc_is_boundary_node(int64_t n, int64_t nx, int64_t ny, int64_t nz) {
  int64_t i = n % (nx + 1);
  int64_t j = (n / (nx + 1)) % (ny + 1);
  int64_t k = n / ((nx + 1) * (ny + 1));
  return i == 0 || j == 0 || k == 0 || i == nx || j == ny || k == nz;
}

/* ---------------------------------------------------------------------------------------
 * Operator apply y = A_c x  (three steps of P:188-196 with A^e from Eq. 4-6).
 * kind: 0 scalar Laplace, 1 vector Laplace, 2 elasticity (lam/mu per cell, lexicographic).
 * bc:   0 none, 1 homogeneous Dirichlet on the 6 box faces: y = P A P x + (I-P) x.
 * Deterministic: cells are visited in 8 colours (i%2 + 2(j%2) + 4(k%2)); within a colour no
 * two cells share a node, so the OpenMP loop over one colour has no write conflicts.
 * ------------------------------------------------------------------------------------- */
int orc_apply(int kind, int bc, int64_t nx, int64_t ny, int64_t nz, double h, const double* lam,
              const double* mu, const double* x, double* y, int nthreads) {
  if (nx < 1 || ny < 1 || nz < 1 || !(h > 0.0) || kind < 0 || kind > 2 || bc < 0 || bc > 1)
    return ORC_EINVAL;
  if (kind == ORC_ELASTIC && (!lam || !mu)) return ORC_EINVAL;
  const int c = (kind == ORC_SCALAR) ? 1 : 3;
  const int64_t nnodes = (nx + 1) * (ny + 1) * (nz + 1);
  memset(y, 0, sizeof(double) * nnodes * c);
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  int err = ORC_OK;
  for (int colour = 0; colour < 8; ++colour) {
    const int ci = colour & 1, cj = (colour >> 1) & 1, ck = (colour >> 2) & 1;
    const int64_t mx = (nx - ci + 1) / 2, my = (ny - cj + 1) / 2, mz = (nz - ck + 1) / 2;
    const int64_t ncol = mx * my * mz;
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < ncol; ++t) {
      const int64_t i = ci + 2 * (t % mx);
      const int64_t j = cj + 2 * ((t / mx) % my);
      const int64_t k = ck + 2 * (t / (mx * my));
      /* step 1: gather coordinates (Alg. 1 line 1) and u^e */
      double X[8][3], ue[24], ve[24], Ae[24 * 24];
      int64_t nid[8];
      for (int a = 0; a < 8; ++a) {
        int64_t ii = i + CORNER[a][0], jj = j + CORNER[a][1], kk = k + CORNER[a][2];
        X[a][0] = (double)ii * h;
        X[a][1] = (double)jj * h;
        X[a][2] = (double)kk * h;
        nid[a] = node_id(ii, jj, kk, nx, ny);
        int masked = bc && orc_is_boundary_node(nid[a], nx, ny, nz);
        for (int comp = 0; comp < c; ++comp) ue[c * a + comp] = masked ? 0.0 : x[c * nid[a] + comp];
      }
      const int64_t e = i + nx * (j + ny * k);
      double le = (kind == ORC_ELASTIC) ? lam[e] : 0.0, me = (kind == ORC_ELASTIC) ? mu[e] : 0.0;
      /* step 2: local multiply v^e = A^e u^e */
      if (orc_element_matrix(kind, X, le, me, Ae) != ORC_OK) {
#pragma omp atomic write
        err = ORC_EGEOM;
        continue;
      }
      const int n = 8 * c;
      for (int r = 0; r < n; ++r) {
        double s = 0.0;
        for (int q = 0; q < n; ++q) s += Ae[r * n + q] * ue[q];
        ve[r] = s;
      }
      /* step 3: assemble into v */
      for (int a = 0; a < 8; ++a)
        for (int comp = 0; comp < c; ++comp) y[c * nid[a] + comp] += ve[c * a + comp];
    }
  }
  if (err) return err;
  if (bc) {
#pragma omp parallel for schedule(static)
    for (int64_t nn = 0; nn < nnodes; ++nn)
      if (orc_is_boundary_node(nn, nx, ny, nz))
        for (int comp = 0; comp < c; ++comp) y[c * nn + comp] = x[c * nn + comp];
  }
  return ORC_OK;
}

/* y_n = (A_c x)_n for a list of nodes only (same three steps of P:188-196 restricted to the
 * <= 8 cells around each requested node), for sampled parity at sizes where the full oracle
 * apply is too slow.  out[c*t + comp] for t-th requested node. */
int orc_apply_nodes(int kind, int bc, int64_t nx, int64_t ny, int64_t nz, double h,
                    const double* lam, const double* mu, const double* x, const int64_t* nodes,
                    int64_t nreq, double* out, int nthreads) {
  if (nx < 1 || ny < 1 || nz < 1 || !(h > 0.0) || kind < 0 || kind > 2) return ORC_EINVAL;
  const int c = (kind == ORC_SCALAR) ? 1 : 3;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  int err = ORC_OK;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t t = 0; t < nreq; ++t) {
    const int64_t n = nodes[t];
    const int64_t ni = n % (nx + 1), nj = (n / (nx + 1)) % (ny + 1), nk = n / ((nx + 1) * (ny + 1));
    double acc[3] = {0.0, 0.0, 0.0};
    if (bc && orc_is_boundary_node(n, nx, ny, nz)) {
      for (int comp = 0; comp < c; ++comp) out[c * t + comp] = x[c * n + comp];
      continue;
    }
    for (int64_t k = nk - 1; k <= nk; ++k)
      for (int64_t j = nj - 1; j <= nj; ++j)
        for (int64_t i = ni - 1; i <= ni; ++i) {
          if (i < 0 || j < 0 || k < 0 || i >= nx || j >= ny || k >= nz) continue;
          double X[8][3], ue[24], Ae[24 * 24];
          int arow = -1;
          for (int a = 0; a < 8; ++a) {
            int64_t ii = i + CORNER[a][0], jj = j + CORNER[a][1], kk = k + CORNER[a][2];
            X[a][0] = (double)ii * h;
            X[a][1] = (double)jj * h;
            X[a][2] = (double)kk * h;
            int64_t id = node_id(ii, jj, kk, nx, ny);
            if (id == n) arow = a;
            int masked = bc && orc_is_boundary_node(id, nx, ny, nz);
            for (int comp = 0; comp < c; ++comp) ue[c * a + comp] = masked ? 0.0 : x[c * id + comp];
          }
          const int64_t e = i + nx * (j + ny * k);
          if (orc_element_matrix(kind, X, kind == ORC_ELASTIC ? lam[e] : 0.0,
                                 kind == ORC_ELASTIC ? mu[e] : 0.0, Ae) != ORC_OK) {
#pragma omp atomic write
            err = ORC_EGEOM;
            continue;
          }
          const int nn = 8 * c;
          for (int comp = 0; comp < c; ++comp) {
            double s = 0.0;
            for (int q = 0; q < nn; ++q) s += Ae[(c * arow + comp) * nn + q] * ue[q];
            acc[comp] += s;
          }
        }
    for (int comp = 0; comp < c; ++comp) out[c * t + comp] = acc[comp];
  }
  return err;
}

/* Dense assembly of A_c for tiny meshes: A[r*ndof + s] (same element matrices, scatter). */
int orc_assemble_dense(int kind, int bc, int64_t nx, int64_t ny, int64_t nz, double h,
                       const double* lam, const double* mu, double* A) {
  const int c = (kind == ORC_SCALAR) ? 1 : 3;
  const int64_t nnodes = (nx + 1) * (ny + 1) * (nz + 1);
  const int64_t ndof = nnodes * c;
  if (ndof > 20000) return ORC_EINVAL;
  memset(A, 0, sizeof(double) * ndof * ndof);
  for (int64_t k = 0; k < nz; ++k)
    for (int64_t j = 0; j < ny; ++j)
      for (int64_t i = 0; i < nx; ++i) {
        double X[8][3], Ae[24 * 24];
        int64_t nid[8];
        for (int a = 0; a < 8; ++a) {
          int64_t ii = i + CORNER[a][0], jj = j + CORNER[a][1], kk = k + CORNER[a][2];
          X[a][0] = ii * h;
          X[a][1] = jj * h;
          X[a][2] = kk * h;
          nid[a] = node_id(ii, jj, kk, nx, ny);
        }
        const int64_t e = i + nx * (j + ny * k);
        int rc = orc_element_matrix(kind, X, kind == ORC_ELASTIC ? lam[e] : 0.0,
                                    kind == ORC_ELASTIC ? mu[e] : 0.0, Ae);
        if (rc) return rc;
        const int n = 8 * c;
        for (int a = 0; a < 8; ++a)
          for (int ca = 0; ca < c; ++ca)
            for (int b = 0; b < 8; ++b)
              for (int cb = 0; cb < c; ++cb)
                A[(c * nid[a] + ca) * ndof + c * nid[b] + cb] += Ae[(c * a + ca) * n + c * b + cb];
      }
  if (bc) {
    for (int64_t nn = 0; nn < nnodes; ++nn) {
      if (!orc_is_boundary_node(nn, nx, ny, nz)) continue;
      for (int comp = 0; comp < c; ++comp) {
        int64_t r = c * nn + comp;
        for (int64_t s = 0; s < ndof; ++s) {
          A[r * ndof + s] = 0.0;
          A[s * ndof + r] = 0.0;
        }
        A[r * ndof + r] = 1.0;
      }
    }
  }
  return ORC_OK;
}

/* ---------------------------------------------------------------------------------------
 * dot (Table 4 "ddot" rows): sequential accumulation in long double.
 * ------------------------------------------------------------------------------------- */
double orc_dot(int64_t n, const double* a, const double* b) {
  long double s = 0.0L;
  for (int64_t i = 0; i < n; ++i) s += (long double)a[i] * (long double)b[i];
  return (double)s;
}

typedef struct {
  int iterations, converged, breakdown_iter, status;
  double r0_norm, r_norm, true_r_norm;
} orc_cg_info;

/* Apply callback of the CG core: y = A_c x for one of the two mesh descriptions below. */
typedef int (*orc_apply_fn)(const void* ctx, const double* x, double* y);

/* CG core (P:185 Krylov method; recurrences of Table 4; stopping per reading R12):
 *   r = b - A x0; p = r; rr = r.r; rho0 = sqrt(rr)
 *   for k < maxit: stop if sqrt(rr) <= tol*rho0 or rr == 0
 *     q = A p; pq = p.q; (pq <= 0 or non-finite -> breakdown)
 *     alpha = rr/pq; x += alpha p; r -= alpha q; rr' = r.r; beta = rr'/rr; p = r + beta p
 * res_hist (optional, length maxit+1) receives sqrt(rr) per iteration. */
static int cg_core(orc_apply_fn apply, const void* ctx, int64_t n, const double* b, double* x,
                   double tol, int maxit, orc_cg_info* info, double* res_hist) {
  double* r = (double*)malloc(sizeof(double) * n);
  double* p = (double*)malloc(sizeof(double) * n);
  double* q = (double*)malloc(sizeof(double) * n);
  if (!r || !p || !q) {
    free(r); free(p); free(q);
    return ORC_ENOMEM;
  }
  int rc = apply(ctx, x, q);
  if (rc) goto done;
  for (int64_t i = 0; i < n; ++i) {
    r[i] = b[i] - q[i];
    p[i] = r[i];
  }
  double rr = orc_dot(n, r, r);
  const double rho0 = sqrt(rr);
  info->r0_norm = rho0;
  info->converged = 0;
  info->breakdown_iter = -1;
  info->status = ORC_OK;
  int it = 0;
  if (res_hist) res_hist[0] = rho0;
  for (; it < maxit; ++it) {
    if (rr == 0.0 || sqrt(rr) <= tol * rho0) {
      info->converged = 1;
      break;
    }
    rc = apply(ctx, p, q);
    if (rc) goto done;
    double pq = orc_dot(n, p, q);
    if (!(pq > 0.0) || !isfinite(pq)) {
      info->breakdown_iter = it;
      info->status = ORC_EBREAKDOWN;
      rc = ORC_EBREAKDOWN;
      break;
    }
    double alpha = rr / pq;
    for (int64_t i = 0; i < n; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * q[i];
    }
    double rr_new = orc_dot(n, r, r);
    double beta = rr_new / rr;
    for (int64_t i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
    rr = rr_new;
    if (res_hist) res_hist[it + 1] = sqrt(rr);
  }
  if (it == maxit && (rr == 0.0 || sqrt(rr) <= tol * rho0)) info->converged = 1;
  info->iterations = it;
  info->r_norm = sqrt(rr);
  /* true residual ||b - A x|| */
  if (apply(ctx, x, q) == ORC_OK) {
    for (int64_t i = 0; i < n; ++i) q[i] = b[i] - q[i];
    info->true_r_norm = sqrt(orc_dot(n, q, q));
  }
done:
  free(r);
  free(p);
  free(q);
  return rc;
}

typedef struct {
  int kind, bc;
  int64_t nx, ny, nz;
  double h;
  const double *lam, *mu;
  int nthreads;
} box_ctx;

static int box_apply(const void* c, const double* x, double* y) {
  const box_ctx* b = (const box_ctx*)c;
  return orc_apply(b->kind, b->bc, b->nx, b->ny, b->nz, b->h, b->lam, b->mu, x, y, b->nthreads);
}

/* CG on the box mesh (orc_apply). */
int orc_cg(int kind, int bc, int64_t nx, int64_t ny, int64_t nz, double h, const double* lam,
           const double* mu, const double* b, double* x, double tol, int maxit, orc_cg_info* info,
           double* res_hist, int nthreads) {
  const int c = (kind == ORC_SCALAR) ? 1 : 3;
  const int64_t n = (nx + 1) * (ny + 1) * (nz + 1) * c;
  box_ctx ctx = {kind, bc, nx, ny, nz, h, lam, mu, nthreads};
  return cg_core(box_apply, &ctx, n, b, x, tol, maxit, info, res_hist);
}

/* ---------------------------------------------------------------------------------------
 * General hexahedral mesh: Algorithm 1 as written, i.e. an explicit node map
 * ("node map", Table 2) and nodal coordinates ("read nodal position", Table 2), the
 * Jacobian recomputed at every quadrature point from the gathered coordinates.
 *   coords[3 n + d]   node n, coordinate d
 *   cells[8 e + a]    global node of local node a of cell e, VTK order (reading R2)
 *   dirichlet[n]      != 0: node n constrained (all components); NULL: no constraint
 *   lam, mu           per cell e (elasticity)
 * y = P A P x + (I - P) x with P zeroing the constrained DOFs.  Cells are visited
 * in index order; element products are formed in parallel, the scatter is sequential
 * in cell order (deterministic).
 * ------------------------------------------------------------------------------------- */
int orc_apply_hex(int kind, int64_t n_nodes, int64_t n_cells, const double* coords,
                  const int32_t* cells, const uint8_t* dirichlet, const double* lam,
                  const double* mu, const double* x, double* y, int nthreads) {
  if (n_nodes < 1 || n_cells < 1 || kind < 0 || kind > 2 || !coords || !cells) return ORC_EINVAL;
  if (kind == ORC_ELASTIC && (!lam || !mu)) return ORC_EINVAL;
  for (int64_t e = 0; e < 8 * n_cells; ++e)
    if (cells[e] < 0 || cells[e] >= n_nodes) return ORC_EINVAL;
  const int c = (kind == ORC_SCALAR) ? 1 : 3;
  const int n = 8 * c;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  memset(y, 0, sizeof(double) * n_nodes * c);
  const int64_t CH = 4096; /* cells per chunk: products in parallel, scatter in order */
  double* ve = (double*)malloc(sizeof(double) * CH * n);
  if (!ve) return ORC_ENOMEM;
  int err = ORC_OK;
  for (int64_t e0 = 0; e0 < n_cells && !err; e0 += CH) {
    const int64_t e1 = (e0 + CH < n_cells) ? e0 + CH : n_cells;
#pragma omp parallel for schedule(static)
    for (int64_t e = e0; e < e1; ++e) {
      /* step 1: gather x^e and u^e (Alg. 1 line 1) */
      double X[8][3], ue[24], Ae[24 * 24];
      for (int a = 0; a < 8; ++a) {
        const int64_t id = cells[8 * e + a];
        for (int d = 0; d < 3; ++d) X[a][d] = coords[3 * id + d];
        const int masked = dirichlet && dirichlet[id];
        for (int comp = 0; comp < c; ++comp) ue[c * a + comp] = masked ? 0.0 : x[c * id + comp];
      }
      /* step 2: v^e = A^e u^e with A^e by quadrature at the gathered geometry */
      if (orc_element_matrix(kind, X, kind == ORC_ELASTIC ? lam[e] : 0.0,
                             kind == ORC_ELASTIC ? mu[e] : 0.0, Ae) != ORC_OK) {
#pragma omp atomic write
        err = ORC_EGEOM;
        continue;
      }
      for (int r = 0; r < n; ++r) {
        double s = 0.0;
        for (int q = 0; q < n; ++q) s += Ae[r * n + q] * ue[q];
        ve[(e - e0) * n + r] = s;
      }
    }
    /* step 3: assemble into v, in cell order */
    for (int64_t e = e0; e < e1 && !err; ++e)
      for (int a = 0; a < 8; ++a) {
        const int64_t id = cells[8 * e + a];
        for (int comp = 0; comp < c; ++comp) y[c * id + comp] += ve[(e - e0) * n + c * a + comp];
      }
  }
  free(ve);
  if (err) return err;
  if (dirichlet)
    for (int64_t nn = 0; nn < n_nodes; ++nn)
      if (dirichlet[nn])
        for (int comp = 0; comp < c; ++comp) y[c * nn + comp] = x[c * nn + comp];
  return ORC_OK;
}

typedef struct {
  int kind;
  int64_t n_nodes, n_cells;
  const double* coords;
  const int32_t* cells;
  const uint8_t* dirichlet;
  const double *lam, *mu;
  int nthreads;
} hex_ctx;

static int hex_apply(const void* c, const double* x, double* y) {
  const hex_ctx* m = (const hex_ctx*)c;
  return orc_apply_hex(m->kind, m->n_nodes, m->n_cells, m->coords, m->cells, m->dirichlet, m->lam,
                       m->mu, x, y, m->nthreads);
}

/* CG on a general hexahedral mesh (orc_apply_hex), same recurrences. */
int orc_cg_hex(int kind, int64_t n_nodes, int64_t n_cells, const double* coords,
               const int32_t* cells, const uint8_t* dirichlet, const double* lam, const double* mu,
               const double* b, double* x, double tol, int maxit, orc_cg_info* info,
               double* res_hist, int nthreads) {
  const int c = (kind == ORC_SCALAR) ? 1 : 3;
  hex_ctx ctx = {kind, n_nodes, n_cells, coords, cells, dirichlet, lam, mu, nthreads};
  return cg_core(hex_apply, &ctx, n_nodes * c, b, x, tol, maxit, info, res_hist);
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
