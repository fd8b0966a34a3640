/*
 * hom2d_oracle.c -- plain, slow, obviously-correct CPU oracle for the hot path of
 * Zimmerman, Regele & Wie, "A Comparative Study of 2D Numerical Methods with GPU
 * Computing" (arXiv 1709.01619).  Citations "P:<line>" are PAPER.md lines.
 *
 * *** TEST INFRASTRUCTURE ONLY. ***  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  It
 * shares no code, header, table or generator with the CUDA path
 * (paper_1709_01619_b200/csrc); it builds every operator at run time from the
 * textbook definitions (Newton iteration in long double).
 *
 * Arithmetic: fp64 throughout (the paper: "Double precision is used for all
 * computations"), compiled with -O2 -ffp-contract=off; one thread unless
 * orc_set_threads asks for more (OpenMP over independent elements / faces /
 * values, bitwise the single-thread result: a timing option for bench.py's
 * cpu_baseline, never a different arithmetic).
 *
 * Layout (ABI choice): Q[c*(Ne*np) + m*np + p], c in {rho, rho u,
 * rho v, e} (SoA), element m = j*nx + i (row-major), point p = b*n + a
 * (x fastest), n = k+1, np = n*n (FV: np = 1).
 *
 * Every residual is computed into a separate array R and then combined by the
 * SSP-RK3 driver (no fusion).  Readings of ambiguous passages follow SURVEY
 * section 8(c).2 (Q1..Q35) and are listed in DESIGN.md.
 *
 * Parity pins: see tests/test_oracle_*.py.  The shock-tube centreline profile
 * (Fig. 5; Toro's digitised curve is not available) is pinned by
 * convergence to a radially symmetric 1-D reference (oracle/radial1d.py, itself
 * pinned to the exact Riemann solution): tests/test_radial_reference.py.
 */
#include <math.h>
#include <stdint.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* configuration (mirrors the fields of the product's hom2d_config, but is its
 * own definition: the oracle includes no product header)                      */
/* ------------------------------------------------------------------------- */
enum { ORC_FV = 0, ORC_CPR = 1, ORC_DG = 2, ORC_NDG = 3, ORC_SD = 4 };
enum { ORC_PERIODIC = 0, ORC_TRANSMISSIVE = 1 };
enum { ORC_CASE_VORTEX = 0, ORC_CASE_SHOCK = 1 };
enum { ORC_OK = 0, ORC_ERR_ARG = 1, ORC_ERR_MESH = 2, ORC_ERR_ORDER = 3,
       ORC_ERR_NONPHYSICAL = 4, ORC_ERR_NOMEM = 7 };

typedef struct {
  int32_t nx, ny;
  double xmin, xmax, ymin, ymax;
  int32_t bc;
  int32_t method;
  int32_t k;              /* HO: polynomial degree 1..4; FV: 1 = MUSCL-2, 2 = MUSCL-3 */
  double gamma;           /* 1.4 (Q1) */
  double cfl;
  int32_t limiter;        /* HO: detect+limit after every stage (Q13) */
  double limiter_eps;     /* 1e-3 */
  int32_t cpr_chain_rule; /* 1 = chain rule; 0 = flux differentiation */
  int32_t physics;        /* test-only: 0 = Euler, 1 = linear advection */
  double adv_a, adv_b;    /* test-only: advection velocity for physics == 1 */
  double dt_fixed;        /* test-only: > 0 replaces the CFL dt of Eq. (36) */
  /* method variants (the defaults 0 are the readings Q10, Q12, Q13) */
  int32_t limiter_per_step;  /* HO: 1 = limit once per step (after stage 3) instead of every stage (Q13) */
  int32_t limiter_all_vars;  /* HO: 1 = detect on all four conserved components, not rho only (Q12) */
  int32_t fv_unlimited;      /* FV: 1 = unlimited kappa-scheme (kappa = 0 / 1/3), no minmod (Q10) */
  int32_t limiter_characteristic; /* HO: 1 = Eq. (35) slopes limited in the characteristic fields of
                                     the element average (Cockburn-Shu), not componentwise (Q12) */
  int32_t fv_error_recon;    /* FV: 1 = error of the reconstructed solution (f4; DESIGN R22),
                                0 = cell value vs exact cell average */
  int32_t dg_overintegrate;  /* DG: 1 = volume and surface integrals of Eq. (19) by (k+2)-point
                                Gauss-Legendre over-integration (SPEC's alternative, f3), 0 = the
                                n-point collocation of Eq. (20) (Q8) */
} orc_config;

/* decision counters (parity of branch decisions); a minmod whose
 * arguments or their difference lie within DEC_TIE of the switch point is a tie */
enum { DEC_MARKED = 0, DEC_MM_ZERO = 1, DEC_MM_FIRST = 2, DEC_MM_SECOND = 3, DEC_MM_TIE = 4 };
#define DEC_TIE 1e-12

#define MAXN 9   /* up to 8-point rules (error quadrature) */

/* Threads (timing only: OpenMP over element rows / faces / values; every value is
 * computed by exactly the same operations whatever the thread count, so results
 * are bitwise those of one thread -- tests/test_oracle_threads.py).  Default 1. */
void orc_set_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n < 1 ? 1 : n);
#else
  (void)n;
#endif
}
int orc_get_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------------- */
/* Legendre polynomials, Gauss / Gauss-Lobatto points (Fig. 1) */
/* ------------------------------------------------------------------------- */
/* P_m(x) and P'_m(x) by the three-term recurrence. */
static void legendre(int m, long double x, long double *P, long double *dP) {
  long double p0 = 1.0L, p1 = x, d0 = 0.0L, d1 = 1.0L;
  if (m == 0) { *P = 1.0L; *dP = 0.0L; return; }
  for (int j = 1; j < m; ++j) {
    long double p2 = ((2 * j + 1) * x * p1 - j * p0) / (j + 1);
    long double d2 = d0 + (2 * j + 1) * p1;   /* P'_{j+1} = P'_{j-1} + (2j+1) P_j */
    p0 = p1; p1 = p2; d0 = d1; d1 = d2;
  }
  *P = p1; *dP = d1;
}

static void sort_ld(long double *v, int n) {
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j)
      if (v[j] < v[i]) { long double t = v[i]; v[i] = v[j]; v[j] = t; }
}

/* kind 0: Gauss-Legendre (roots of P_n); kind 1: Gauss-Lobatto ({-1, roots of
 * P'_{n-1}, +1}).  Ascending, exactly symmetrised (middle node exactly 0). */
int orc_nodes(int kind, int n, double *xi, double *w) {
  if (n < 1 || n > MAXN || (kind == 1 && n < 2)) return ORC_ERR_ARG;
  long double x[MAXN], ww[MAXN];
  if (kind == 0) {
    for (int i = 0; i < n; ++i) {
      long double z = cosl(3.14159265358979323846264338327950288L * (4 * i + 3) / (4 * n + 2));
      for (int it = 0; it < 100; ++it) {
        long double P, dP;
        legendre(n, z, &P, &dP);
        long double dz = P / dP;
        z -= dz;
        if (fabsl(dz) < 1e-30L) break;
      }
      x[i] = z;
    }
    sort_ld(x, n);
    for (int i = 0; i < n; ++i) {
      long double P, dP;
      legendre(n, x[i], &P, &dP);
      ww[i] = 2.0L / ((1.0L - x[i] * x[i]) * dP * dP);
    }
  } else {
    int m = n - 1;               /* interior nodes: roots of P'_m */
    x[0] = -1.0L; x[n - 1] = 1.0L;
    for (int i = 1; i < n - 1; ++i) {
      long double z = cosl(3.14159265358979323846264338327950288L * i / (n - 1));
      for (int it = 0; it < 100; ++it) {
        long double P, dP;
        legendre(m, z, &P, &dP);
        long double d2P = (2.0L * z * dP - m * (m + 1) * P) / (1.0L - z * z);
        long double dz = dP / d2P;
        z -= dz;
        if (fabsl(dz) < 1e-30L) break;
      }
      x[i] = z;
    }
    sort_ld(x, n);
    for (int i = 0; i < n; ++i) {
      long double P, dP;
      legendre(m, x[i], &P, &dP);
      ww[i] = 2.0L / ((long double)n * (n - 1) * P * P);
    }
  }
  for (int i = 0; i < n; ++i) {   /* symmetrise */
    int j = n - 1 - i;
    long double xs = 0.5L * (x[i] - x[j]);
    long double ws = 0.5L * (ww[i] + ww[j]);
    xi[i] = (double)xs;
    w[i] = (double)ws;
  }
  if (n % 2 == 1) xi[n / 2] = 0.0;
  return ORC_OK;
}

/* Lagrange basis l_l(x) on nodes xi[0..n-1] (long double evaluation). */
void orc_lagrange(int n, const double *xi, double x, double *l) {
  for (int j = 0; j < n; ++j) {
    long double v = 1.0L;
    for (int m = 0; m < n; ++m)
      if (m != j) v *= ((long double)x - xi[m]) / ((long double)xi[j] - xi[m]);
    l[j] = (double)v;
  }
}

/* derivative l'_l(x) = sum_{m != l} 1/(xi_l - xi_m) prod_{r != l,m} (x - xi_r)/(xi_l - xi_r) */
void orc_lagrange_deriv(int n, const double *xi, double x, double *dl) {
  for (int j = 0; j < n; ++j) {
    long double s = 0.0L;
    for (int m = 0; m < n; ++m) {
      if (m == j) continue;
      long double t = 1.0L / ((long double)xi[j] - xi[m]);
      for (int r = 0; r < n; ++r)
        if (r != j && r != m) t *= ((long double)x - xi[r]) / ((long double)xi[j] - xi[r]);
      s += t;
    }
    dl[j] = (double)s;
  }
}

/* Right Radau correction derivative g'_R(x) = (P'_{k+1}(x) + P'_k(x)) / 2
 * ("Radau polynomials ... casts delta into the DG framework";
 * g_R = (P_k + P_{k+1})/2, g_R(1) = 1, g_R(-1) = 0; g_L(x) = g_R(-x)). */
double orc_radau_dgR(int k, double x) {
  long double P1, dP1, P0, dP0;
  legendre(k + 1, x, &P1, &dP1);
  legendre(k, x, &P0, &dP0);
  return (double)(0.5L * (dP1 + dP0));
}

/* ------------------------------------------------------------------------- */
/* element operators                                                          */
/* ------------------------------------------------------------------------- */
typedef struct {
  int n;
  double xi[MAXN], w[MAXN];
  double D[MAXN][MAXN];      /* D[a][l] = l'_l(xi_a) */
  double gLp[MAXN], gRp[MAXN];
  double eL[MAXN], eR[MAXN]; /* l_l(-1), l_l(+1) */
  int nf;                    /* SD flux points */
  double xf[MAXN];
  double If[MAXN][MAXN];     /* If[r][a] = l_a(xf_r) */
  double Df[MAXN][MAXN];     /* Df[a][r] = lambda'_r(xi_a) */
} ops_t;

static int is_gll(int method) { return method == ORC_CPR || method == ORC_NDG; }

static void build_ops(int method, int k, ops_t *o) {
  memset(o, 0, sizeof(*o));
  int n = k + 1;
  o->n = n;
  orc_nodes(is_gll(method) ? 1 : 0, n, o->xi, o->w);
  for (int a = 0; a < n; ++a) orc_lagrange_deriv(n, o->xi, o->xi[a], o->D[a]);
  for (int a = 0; a < n; ++a) {
    o->gRp[a] = orc_radau_dgR(k, o->xi[a]);
    o->gLp[a] = -orc_radau_dgR(k, -o->xi[a]);
  }
  orc_lagrange(n, o->xi, -1.0, o->eL);
  orc_lagrange(n, o->xi, 1.0, o->eR);
  if (method == ORC_SD) {
    /* flux points: Chebyshev-Gauss-Lobatto x_r = -cos(pi r/(k+1)), r = 0..k+1
     * ("Gauss-Lobatto flux points", Fig. 1(c); the Chebyshev reading is
     * the one that reproduces Table 3's SD column, R9) */
    o->nf = n + 1;
    for (int r = 0; r <= n; ++r) o->xf[r] = -cos(3.14159265358979323846 * r / n);
    for (int r = 0; r <= n; ++r) {   /* exact symmetry, exact endpoints / middle */
      if (2 * r < n) { o->xf[n - r] = -o->xf[r]; }
    }
    o->xf[0] = -1.0; o->xf[n] = 1.0;
    if (n % 2 == 0) o->xf[n / 2] = 0.0;
    for (int r = 0; r < n + 1; ++r) orc_lagrange(n, o->xi, o->xf[r], o->If[r]);
    for (int a = 0; a < n; ++a) orc_lagrange_deriv(n + 1, o->xf, o->xi[a], o->Df[a]);
  }
}

/* ------------------------------------------------------------------------- */
/* physics (Eqs. (3)-(5); Rusanov P:869-870)                       */
/* ------------------------------------------------------------------------- */
typedef struct { int phys; double g, a, b; } phys_t;

static phys_t mkphys(const orc_config *c) {
  phys_t p; p.phys = c->physics; p.g = c->gamma; p.a = c->adv_a; p.b = c->adv_b; return p;
}

static double pressure(const phys_t *P, const double *q) {
  double u = q[1] / q[0], v = q[2] / q[0];
  return (P->g - 1.0) * (q[3] - 0.5 * q[0] * (u * u + v * v));
}

/* dir 0: f(q) (x), dir 1: g(q) (y) -- Eq. (4) */
static void flux(const phys_t *P, int dir, const double *q, double *f) {
  if (P->phys == 1) {
    double s = dir == 0 ? P->a : P->b;
    for (int c = 0; c < 4; ++c) f[c] = s * q[c];
    return;
  }
  double u = q[1] / q[0], v = q[2] / q[0];
  double p = pressure(P, q);
  if (dir == 0) {
    f[0] = q[1]; f[1] = p + q[0] * u * u; f[2] = q[0] * u * v; f[3] = u * (q[3] + p);
  } else {
    f[0] = q[2]; f[1] = q[0] * u * v; f[2] = p + q[0] * v * v; f[3] = v * (q[3] + p);
  }
}

/* |u.n| + c along axis dir */
static double normal_speed(const phys_t *P, int dir, const double *q) {
  if (P->phys == 1) return fabs(dir == 0 ? P->a : P->b);
  double un = (dir == 0 ? q[1] : q[2]) / q[0];
  double c = sqrt(P->g * pressure(P, q) / q[0]);
  return fabs(un) + c;
}

/* max(|u|,|v|) + c  (2-D reading of Eq. (36), Q4) */
static double wave_speed(const phys_t *P, const double *q) {
  if (P->phys == 1) return fmax(fabs(P->a), fabs(P->b));
  double u = q[1] / q[0], v = q[2] / q[0];
  double c = sqrt(P->g * pressure(P, q) / q[0]);
  return fmax(fabs(u), fabs(v)) + c;
}

/* Rusanov flux, always called as (west/south, east/north) */
static void rusanov(const phys_t *P, int dir, const double *qL, const double *qR, double *F) {
  double fL[4], fR[4];
  flux(P, dir, qL, fL);
  flux(P, dir, qR, fR);
  double lam = fmax(normal_speed(P, dir, qL), normal_speed(P, dir, qR));
  for (int c = 0; c < 4; ++c) F[c] = 0.5 * (fL[c] + fR[c]) - 0.5 * lam * (qR[c] - qL[c]);
}

/* flux Jacobian action A(q).d (dir 0) or B(q).d (dir 1) */
static void jac_apply(const phys_t *P, int dir, const double *q, const double *d, double *out) {
  if (P->phys == 1) {
    double s = dir == 0 ? P->a : P->b;
    for (int c = 0; c < 4; ++c) out[c] = s * d[c];
    return;
  }
  double g = P->g;
  double u = q[1] / q[0], v = q[2] / q[0];
  double p = pressure(P, q);
  double phi = 0.5 * (g - 1.0) * (u * u + v * v);
  double H = (q[3] + p) / q[0];
  if (dir == 0) {
    out[0] = d[1];
    out[1] = (phi - u * u) * d[0] + (3.0 - g) * u * d[1] - (g - 1.0) * v * d[2] + (g - 1.0) * d[3];
    out[2] = -u * v * d[0] + v * d[1] + u * d[2];
    out[3] = u * (phi - H) * d[0] + (H - (g - 1.0) * u * u) * d[1] - (g - 1.0) * u * v * d[2] + g * u * d[3];
  } else {
    out[0] = d[2];
    out[1] = -u * v * d[0] + v * d[1] + u * d[2];
    out[2] = (phi - v * v) * d[0] - (g - 1.0) * u * d[1] + (3.0 - g) * v * d[2] + (g - 1.0) * d[3];
    out[3] = v * (phi - H) * d[0] - (g - 1.0) * u * v * d[1] + (H - (g - 1.0) * v * v) * d[2] + g * v * d[3];
  }
}

/* exported physics for the pins (P1) */
void orc_flux(const orc_config *c, int dir, const double *q, double *f) { phys_t P = mkphys(c); flux(&P, dir, q, f); }
void orc_rusanov(const orc_config *c, int dir, const double *qL, const double *qR, double *F) { phys_t P = mkphys(c); rusanov(&P, dir, qL, qR, F); }
void orc_jacobian_apply(const orc_config *c, int dir, const double *q, const double *d, double *o) { phys_t P = mkphys(c); jac_apply(&P, dir, q, d, o); }
double orc_wave_speed(const orc_config *c, const double *q) { phys_t P = mkphys(c); return wave_speed(&P, q); }
double orc_pressure(const orc_config *c, const double *q) { phys_t P = mkphys(c); return pressure(&P, q); }

/* Right / left eigenvectors of the Euler flux Jacobian along axis dir (dir 0:
 * A(q), dir 1: B(q)) at the state q: A = R diag(un-c, un, un, un+c) L,
 * columns of R = (1, u - c nx, v - c ny, H - c un), (1, u, v, |u|^2/2),
 * (0, ny..., tangential), (1, u + c nx, v + c ny, H + c un); L = R^-1 in closed
 * form with b1 = (gamma-1)/c^2, b2 = b1 |u|^2/2 (textbook, e.g. Toro ch. 3 /
 * Hesthaven-Warburton).  Pinned: L R = I and L A R diagonal (tests). */
static void char_vectors(const phys_t *P, int dir, const double *q, double R[4][4], double L[4][4]) {
  double g = P->g, u = q[1] / q[0], v = q[2] / q[0];
  double p = pressure(P, q), H = (q[3] + p) / q[0], c = sqrt(g * p / q[0]);
  double nx = dir == 0 ? 1.0 : 0.0, ny = 1.0 - nx;
  double un = u * nx + v * ny, ut = -u * ny + v * nx;   /* normal / tangential velocity */
  double q2 = 0.5 * (u * u + v * v), b1 = (g - 1.0) / (c * c), b2 = b1 * q2;
  /* columns: acoustic -, entropy, shear, acoustic + */
  double r[4][4] = {{1.0, u - c * nx, v - c * ny, H - c * un},
                    {1.0, u, v, q2},
                    {0.0, -ny, nx, ut},
                    {1.0, u + c * nx, v + c * ny, H + c * un}};
  for (int i = 0; i < 4; ++i)
    for (int k = 0; k < 4; ++k) R[i][k] = r[k][i];
  double l[4][4] = {{0.5 * (b2 + un / c), -0.5 * (b1 * u + nx / c), -0.5 * (b1 * v + ny / c), 0.5 * b1},
                    {1.0 - b2, b1 * u, b1 * v, -b1},
                    {-ut, -ny, nx, 0.0},
                    {0.5 * (b2 - un / c), -0.5 * (b1 * u - nx / c), -0.5 * (b1 * v - ny / c), 0.5 * b1}};
  for (int i = 0; i < 4; ++i)
    for (int k = 0; k < 4; ++k) L[i][k] = l[i][k];
}
void orc_char_vectors(const orc_config *cf, int dir, const double *q, double *R16, double *L16) {
  phys_t P = mkphys(cf);
  double R[4][4], L[4][4];
  char_vectors(&P, dir, q, R, L);
  for (int i = 0; i < 16; ++i) { R16[i] = R[i / 4][i % 4]; L16[i] = L[i / 4][i % 4]; }
}

/* ------------------------------------------------------------------------- */
/* minmod (Q17)                                                         */
/* ------------------------------------------------------------------------- */
/* cell: optional per-cell decision map entry (SURVEY C12 dumps): the outcome is
 * added as 1 << (16 * slot), slot 0 -> 0, 1 -> first argument, 2 -> second, 3 tie */
static double mm2c(double a, double b, int64_t *cnt, int64_t *cell) {
  double r = 0.0; int which = 0;
  if (a > 0.0 && b > 0.0) { if (a <= b) { r = a; which = 1; } else { r = b; which = 2; } }
  else if (a < 0.0 && b < 0.0) { if (a >= b) { r = a; which = 1; } else { r = b; which = 2; } }
  if (cnt || cell) {
    int slot = (fabs(a) <= DEC_TIE || fabs(b) <= DEC_TIE || fabs(a - b) <= DEC_TIE) ? 3 : which;
    if (cnt) cnt[slot == 3 ? DEC_MM_TIE : (slot == 0 ? DEC_MM_ZERO : (slot == 1 ? DEC_MM_FIRST : DEC_MM_SECOND))]++;
    if (cell) *cell += (int64_t)1 << (16 * slot);
  }
  return r;
}
static double mm2(double a, double b, int64_t *cnt) { return mm2c(a, b, cnt, NULL); }
static double mm3(double a, double b, double c) {
  if (a > 0.0 && b > 0.0 && c > 0.0) return fmin(a, fmin(b, c));
  if (a < 0.0 && b < 0.0 && c < 0.0) return fmax(a, fmax(b, c));
  return 0.0;
}
double orc_minmod2(double a, double b) { return mm2(a, b, NULL); }
double orc_minmod3(double a, double b, double c) { return mm3(a, b, c); }

/* ------------------------------------------------------------------------- */
/* mesh helpers                                                   */
/* ------------------------------------------------------------------------- */
static int points_per_elem(const orc_config *c) {
  return c->method == ORC_FV ? 1 : (c->k + 1) * (c->k + 1);
}

/* neighbour column/row index; -1 = physical (transmissive) boundary */
static int nb_index(int i, int d, int n, int bc) {
  int j = i + d;
  if (j >= 0 && j < n) return j;
  if (bc == ORC_PERIODIC) return (j + n) % n;
  return -1;
}

static int check_cfg(const orc_config *c) {
  if (!c) return ORC_ERR_ARG;
  if (c->nx < 2 || c->ny < 2 || !(c->xmax > c->xmin) || !(c->ymax > c->ymin)) return ORC_ERR_MESH;
  if (c->method < 0 || c->method > 4) return ORC_ERR_ARG;
  if (c->method == ORC_FV) { if (c->k < 1 || c->k > 2) return ORC_ERR_ORDER; }
  else if (c->k < 1 || c->k > 4) return ORC_ERR_ORDER;
  if (c->bc != ORC_PERIODIC && c->bc != ORC_TRANSMISSIVE) return ORC_ERR_ARG;
  return ORC_OK;
}

/* gather the 4 conserved values of point p of element m */
static void getq(const double *Q, int64_t N, int64_t m, int np, int p, double *q) {
  for (int c = 0; c < 4; ++c) q[c] = Q[c * N + m * np + p];
}

/* Element trace on side s (0 W, 1 E, 2 S, 3 N) at line index t. GLL:
 * the edge node; GL: interpolation along the solution line (Alg. 2). */
static void trace(const ops_t *o, int gll, const double *Q, int64_t N, int64_t m, int s, int t, double *q) {
  int n = o->n, np = n * n;
  if (gll) {
    int p = s == 0 ? t * n : s == 1 ? t * n + n - 1 : s == 2 ? t : (n - 1) * n + t;
    getq(Q, N, m, np, p, q);
    return;
  }
  const double *e = (s == 0 || s == 2) ? o->eL : o->eR;
  for (int c = 0; c < 4; ++c) {
    double acc = 0.0;
    for (int l = 0; l < n; ++l) {
      int p = (s <= 1) ? t * n + l : l * n + t;
      acc += e[l] * Q[c * N + m * np + p];
    }
    q[c] = acc;
  }
}

/* Common face fluxes of element (i,j) on its 4 sides, n points each.
 * FW[b][c], FE[b][c] along x; FS[a][c], FN[a][c] along y. */
static void face_fluxes(const orc_config *cf, const phys_t *P, const ops_t *o, const double *Q,
                        int i, int j, double FW[][4], double FE[][4], double FS[][4], double FN[][4]) {
  int n = o->n, gll = is_gll(cf->method);
  int64_t N = (int64_t)cf->nx * cf->ny * n * n;
  int64_t m = (int64_t)j * cf->nx + i;
  int iw = nb_index(i, -1, cf->nx, cf->bc), ie = nb_index(i, 1, cf->nx, cf->bc);
  int js = nb_index(j, -1, cf->ny, cf->bc), jn = nb_index(j, 1, cf->ny, cf->bc);
  double qo[4], qn[4];
  for (int t = 0; t < n; ++t) {
    trace(o, gll, Q, N, m, 0, t, qo);
    if (iw >= 0) trace(o, gll, Q, N, (int64_t)j * cf->nx + iw, 1, t, qn); else memcpy(qn, qo, sizeof qn);
    rusanov(P, 0, qn, qo, FW[t]);
    trace(o, gll, Q, N, m, 1, t, qo);
    if (ie >= 0) trace(o, gll, Q, N, (int64_t)j * cf->nx + ie, 0, t, qn); else memcpy(qn, qo, sizeof qn);
    rusanov(P, 0, qo, qn, FE[t]);
    trace(o, gll, Q, N, m, 2, t, qo);
    if (js >= 0) trace(o, gll, Q, N, (int64_t)js * cf->nx + i, 3, t, qn); else memcpy(qn, qo, sizeof qn);
    rusanov(P, 1, qn, qo, FS[t]);
    trace(o, gll, Q, N, m, 3, t, qo);
    if (jn >= 0) trace(o, gll, Q, N, (int64_t)jn * cf->nx + i, 2, t, qn); else memcpy(qn, qo, sizeof qn);
    rusanov(P, 1, qo, qn, FN[t]);
  }
}

/* ------------------------------------------------------------------------- */
/* CPR / NDG residual (Eqs. (13)-(17), (24)-(29); Algs. 7-8)      */
/* ------------------------------------------------------------------------- */
static void residual_cpr_ndg(const orc_config *cf, const ops_t *o, const double *Q, double *R) {
  phys_t P = mkphys(cf);
  int n = o->n, np = n * n;
  int64_t N = (int64_t)cf->nx * cf->ny * np;
  double dx = (cf->xmax - cf->xmin) / cf->nx, dy = (cf->ymax - cf->ymin) / cf->ny;
  int chain = (cf->method == ORC_CPR) && cf->cpr_chain_rule;
  double FW[MAXN][4], FE[MAXN][4], FS[MAXN][4], FN[MAXN][4];
#pragma omp parallel for private(FW, FE, FS, FN) schedule(static)
  for (int j = 0; j < cf->ny; ++j)
    for (int i = 0; i < cf->nx; ++i) {
      int64_t m = (int64_t)j * cf->nx + i;
      face_fluxes(cf, &P, o, Q, i, j, FW, FE, FS, FN);
      for (int b = 0; b < n; ++b)
        for (int a = 0; a < n; ++a) {
          double q[4], qx[4] = {0, 0, 0, 0}, qy[4] = {0, 0, 0, 0};
          double Fx[4], Gy[4];
          getq(Q, N, m, np, b * n + a, q);
          if (chain) {
            /* Pi[div F] by the chain rule: A(q) dq/dxi + B(q) dq/deta */
            for (int l = 0; l < n; ++l)
              for (int c = 0; c < 4; ++c) {
                qx[c] += o->D[a][l] * Q[c * N + m * np + b * n + l];
                qy[c] += o->D[b][l] * Q[c * N + m * np + l * n + a];
              }
            jac_apply(&P, 0, q, qx, Fx);
            jac_apply(&P, 1, q, qy, Gy);
          } else {
            /* NDG: D[F] (Eq. (28)); also CPR with cpr_chain_rule = 0 */
            double f[4];
            for (int c = 0; c < 4; ++c) Fx[c] = Gy[c] = 0.0;
            for (int l = 0; l < n; ++l) {
              double ql[4];
              getq(Q, N, m, np, b * n + l, ql);
              flux(&P, 0, ql, f);
              for (int c = 0; c < 4; ++c) Fx[c] += o->D[a][l] * f[c];
              getq(Q, N, m, np, l * n + a, ql);
              flux(&P, 1, ql, f);
              for (int c = 0; c < 4; ++c) Gy[c] += o->D[b][l] * f[c];
            }
          }
          /* correction (CPR, Radau g_DG) == lift (NDG, exact mass): both
           * directions, 2 updates each (Alg. 8: n_upd; Q6, Q7, Q34) */
          double q0[4], q1[4], f0[4], f1[4];
          getq(Q, N, m, np, b * n + 0, q0);
          getq(Q, N, m, np, b * n + n - 1, q1);
          flux(&P, 0, q0, f0);
          flux(&P, 0, q1, f1);
          for (int c = 0; c < 4; ++c)
            Fx[c] += o->gLp[a] * (FW[b][c] - f0[c]) + o->gRp[a] * (FE[b][c] - f1[c]);
          getq(Q, N, m, np, 0 * n + a, q0);
          getq(Q, N, m, np, (n - 1) * n + a, q1);
          flux(&P, 1, q0, f0);
          flux(&P, 1, q1, f1);
          for (int c = 0; c < 4; ++c)
            Gy[c] += o->gLp[b] * (FS[a][c] - f0[c]) + o->gRp[b] * (FN[a][c] - f1[c]);
          for (int c = 0; c < 4; ++c)
            R[c * N + m * np + b * n + a] = -(2.0 / dx) * Fx[c] - (2.0 / dy) * Gy[c];
        }
    }
}

/* ------------------------------------------------------------------------- */
/* DG residual, weak form on Gauss-Legendre points (Eqs. (18)-(21),  */
/* Algs. 2-4)                                             */
/* ------------------------------------------------------------------------- */
static void residual_dg(const orc_config *cf, const ops_t *o, const double *Q, double *R) {
  phys_t P = mkphys(cf);
  int n = o->n, np = n * n;
  int64_t N = (int64_t)cf->nx * cf->ny * np;
  double dx = (cf->xmax - cf->xmin) / cf->nx, dy = (cf->ymax - cf->ymin) / cf->ny;
  double FW[MAXN][4], FE[MAXN][4], FS[MAXN][4], FN[MAXN][4];
#pragma omp parallel for private(FW, FE, FS, FN) schedule(static)
  for (int j = 0; j < cf->ny; ++j)
    for (int i = 0; i < cf->nx; ++i) {
      int64_t m = (int64_t)j * cf->nx + i;
      face_fluxes(cf, &P, o, Q, i, j, FW, FE, FS, FN);
      for (int b = 0; b < n; ++b)
        for (int a = 0; a < n; ++a) {
          double volx[4] = {0, 0, 0, 0}, voly[4] = {0, 0, 0, 0}, f[4], ql[4];
          /* volume integral: sum_l w_l l'_a(xi_l) f_{l,b} */
          for (int l = 0; l < n; ++l) {
            getq(Q, N, m, np, b * n + l, ql);
            flux(&P, 0, ql, f);
            for (int c = 0; c < 4; ++c) volx[c] += o->w[l] * o->D[l][a] * f[c];
            getq(Q, N, m, np, l * n + a, ql);
            flux(&P, 1, ql, f);
            for (int c = 0; c < 4; ++c) voly[c] += o->w[l] * o->D[l][b] * f[c];
          }
          for (int c = 0; c < 4; ++c) {
            /* surface integral: l_a(1) F^E - l_a(-1) F^W */
            double surx = o->eR[a] * FE[b][c] - o->eL[a] * FW[b][c];
            double sury = o->eR[b] * FN[a][c] - o->eL[b] * FS[a][c];
            /* M^{-1}: diagonal (Delta/2) w_a */
            R[c * N + m * np + b * n + a] = (2.0 / dx) * (volx[c] - surx) / o->w[a]
                                          + (2.0 / dy) * (voly[c] - sury) / o->w[b];
          }
        }
    }
}

/* DG residual of Eq. (19) with the integrals by an nq-point Gauss-Legendre rule
 * (f3 variant: nq = k+2 over-integration; nq = n is residual_dg's collocation).
 * The solution polynomial q_h is interpolated to the nq x nq quadrature points
 * (zeta_r, zeta_s) and to nq points along every edge; the fluxes are evaluated
 * there:
 *   Vol^x_ab = sum_rs W_r W_s f(q_h(zeta_r, zeta_s)) l'_a(zeta_r) l_b(zeta_s)
 *   Sur^x_ab = sum_s W_s [l_a(1) F^E(zeta_s) - l_a(-1) F^W(zeta_s)] l_b(zeta_s)
 * (F^E/W: Rusanov between the two traces q_h(+-1, zeta_s), transmissive ghost =
 * own trace), y likewise, and with the exact (diagonal) GL mass matrix
 *   R_ab = (2/dx)(Vol^x - Sur^x)_ab / (w_a w_b) + (2/dy)(Vol^y - Sur^y)_ab / (w_a w_b). */
static void residual_dg_quad(const orc_config *cf, const ops_t *o, int nq, const double *Q, double *R) {
  phys_t P = mkphys(cf);
  int n = o->n, np = n * n;
  int64_t N = (int64_t)cf->nx * cf->ny * np;
  double dx = (cf->xmax - cf->xmin) / cf->nx, dy = (cf->ymax - cf->ymin) / cf->ny;
  double z[MAXN], W[MAXN], Lz[MAXN][MAXN], dLz[MAXN][MAXN];
  orc_nodes(0, nq, z, W);
  for (int r = 0; r < nq; ++r) {
    orc_lagrange(n, o->xi, z[r], Lz[r]);
    orc_lagrange_deriv(n, o->xi, z[r], dLz[r]);
  }
  /* q_h of element m at (x-coordinate weights ex[a], y-coordinate weights ey[b]) */
#define QH(m_, ex, ey, out)                                                              \
  for (int c = 0; c < 4; ++c) {                                                         \
    double acc = 0.0;                                                                   \
    for (int b = 0; b < n; ++b)                                                         \
      for (int a = 0; a < n; ++a) acc += (ex)[a] * (ey)[b] * Q[c * N + (m_) * np + b * n + a]; \
    (out)[c] = acc;                                                                     \
  }
#pragma omp parallel for schedule(static)
  for (int j = 0; j < cf->ny; ++j)
    for (int i = 0; i < cf->nx; ++i) {
      int64_t m = (int64_t)j * cf->nx + i;
      int iw = nb_index(i, -1, cf->nx, cf->bc), ie = nb_index(i, 1, cf->nx, cf->bc);
      int js = nb_index(j, -1, cf->ny, cf->bc), jn = nb_index(j, 1, cf->ny, cf->bc);
      int64_t mw = (int64_t)j * cf->nx + iw, me = (int64_t)j * cf->nx + ie;
      int64_t ms = (int64_t)js * cf->nx + i, mn = (int64_t)jn * cf->nx + i;
      double f[MAXN][MAXN][4], g[MAXN][MAXN][4];
      for (int s2 = 0; s2 < nq; ++s2)
        for (int r = 0; r < nq; ++r) {
          double q[4];
          QH(m, Lz[r], Lz[s2], q);
          flux(&P, 0, q, f[s2][r]);
          flux(&P, 1, q, g[s2][r]);
        }
      double FW[MAXN][4], FE[MAXN][4], FS[MAXN][4], FN[MAXN][4];
      for (int t = 0; t < nq; ++t) {
        double qo[4], qn[4];
        QH(m, o->eL, Lz[t], qo);                       /* own west trace at eta = zeta_t */
        if (iw >= 0) { QH(mw, o->eR, Lz[t], qn); } else memcpy(qn, qo, sizeof qn);
        rusanov(&P, 0, qn, qo, FW[t]);
        QH(m, o->eR, Lz[t], qo);
        if (ie >= 0) { QH(me, o->eL, Lz[t], qn); } else memcpy(qn, qo, sizeof qn);
        rusanov(&P, 0, qo, qn, FE[t]);
        QH(m, Lz[t], o->eL, qo);                       /* own south trace at xi = zeta_t */
        if (js >= 0) { QH(ms, Lz[t], o->eR, qn); } else memcpy(qn, qo, sizeof qn);
        rusanov(&P, 1, qn, qo, FS[t]);
        QH(m, Lz[t], o->eR, qo);
        if (jn >= 0) { QH(mn, Lz[t], o->eL, qn); } else memcpy(qn, qo, sizeof qn);
        rusanov(&P, 1, qo, qn, FN[t]);
      }
      for (int b = 0; b < n; ++b)
        for (int a = 0; a < n; ++a)
          for (int c = 0; c < 4; ++c) {
            double vx = 0.0, vy = 0.0, sx = 0.0, sy = 0.0;
            for (int s2 = 0; s2 < nq; ++s2)
              for (int r = 0; r < nq; ++r) {
                vx += W[r] * W[s2] * f[s2][r][c] * dLz[r][a] * Lz[s2][b];
                vy += W[r] * W[s2] * g[s2][r][c] * Lz[r][a] * dLz[s2][b];
              }
            for (int t = 0; t < nq; ++t) {
              sx += W[t] * (o->eR[a] * FE[t][c] - o->eL[a] * FW[t][c]) * Lz[t][b];
              sy += W[t] * (o->eR[b] * FN[t][c] - o->eL[b] * FS[t][c]) * Lz[t][a];
            }
            R[c * N + m * np + b * n + a] = (2.0 / dx) * (vx - sx) / (o->w[a] * o->w[b])
                                          + (2.0 / dy) * (vy - sy) / (o->w[a] * o->w[b]);
          }
    }
#undef QH
}

/* the quadrature DG residual with an explicit rule size (tests: nq = n equals
 * residual_dg up to rounding, nq = k+2 is the over-integrated variant) */
int orc_residual_dg_quad(const orc_config *cf, int nq, const double *Q, double *R) {
  int st = check_cfg(cf);
  if (st) return st;
  if (cf->method != ORC_DG || nq < cf->k + 1 || nq > 8) return ORC_ERR_ARG;
  ops_t o;
  build_ops(cf->method, cf->k, &o);
  residual_dg_quad(cf, &o, nq, Q, R);
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* SD residual: GL solution points, GLL(k+2) flux points (SURVEY C7;            */
/* Eqs. (30)-(34), with the Eq. (34) typo f -> g; Algs. 5-6)          */
/* ------------------------------------------------------------------------- */
/* q at flux point r of line t of element m; dir 0: x-line (row t), 1: y-line (column t) */
static void sd_qf(const ops_t *o, const double *Q, int64_t N, int64_t m, int dir, int t, int r, double *q) {
  int n = o->n, np = n * n;
  for (int c = 0; c < 4; ++c) {
    double acc = 0.0;
    for (int a = 0; a < n; ++a) {
      int p = dir == 0 ? t * n + a : a * n + t;
      acc += o->If[r][a] * Q[c * N + m * np + p];
    }
    q[c] = acc;
  }
}

static void residual_sd(const orc_config *cf, const ops_t *o, const double *Q, double *R) {
  phys_t P = mkphys(cf);
  int n = o->n, np = n * n, nf = o->nf;
  int64_t N = (int64_t)cf->nx * cf->ny * np;
  double dx = (cf->xmax - cf->xmin) / cf->nx, dy = (cf->ymax - cf->ymin) / cf->ny;
  double phi[2][MAXN][MAXN][4];   /* [dir][line][flux point][c] */
#pragma omp parallel for private(phi) schedule(static)
  for (int j = 0; j < cf->ny; ++j)
    for (int i = 0; i < cf->nx; ++i) {
      int64_t m = (int64_t)j * cf->nx + i;
      int iw = nb_index(i, -1, cf->nx, cf->bc), ie = nb_index(i, 1, cf->nx, cf->bc);
      int js = nb_index(j, -1, cf->ny, cf->bc), jn = nb_index(j, 1, cf->ny, cf->bc);
      for (int dir = 0; dir < 2; ++dir)
        for (int t = 0; t < n; ++t) {
          double q[4], qn[4];
          for (int r = 1; r < nf - 1; ++r) {
            sd_qf(o, Q, N, m, dir, t, r, q);
            flux(&P, dir, q, phi[dir][t][r]);
          }
          /* left/bottom end: Riemann with the W/S neighbour's last flux point */
          int64_t mlo = dir == 0 ? (iw >= 0 ? (int64_t)j * cf->nx + iw : -1) : (js >= 0 ? (int64_t)js * cf->nx + i : -1);
          int64_t mhi = dir == 0 ? (ie >= 0 ? (int64_t)j * cf->nx + ie : -1) : (jn >= 0 ? (int64_t)jn * cf->nx + i : -1);
          sd_qf(o, Q, N, m, dir, t, 0, q);
          if (mlo >= 0) sd_qf(o, Q, N, mlo, dir, t, nf - 1, qn); else memcpy(qn, q, sizeof qn);
          rusanov(&P, dir, qn, q, phi[dir][t][0]);
          sd_qf(o, Q, N, m, dir, t, nf - 1, q);
          if (mhi >= 0) sd_qf(o, Q, N, mhi, dir, t, 0, qn); else memcpy(qn, q, sizeof qn);
          rusanov(&P, dir, q, qn, phi[dir][t][nf - 1]);
        }
      for (int b = 0; b < n; ++b)
        for (int a = 0; a < n; ++a)
          for (int c = 0; c < 4; ++c) {
            double Fx = 0.0, Gy = 0.0;
            for (int r = 0; r < nf; ++r) {
              Fx += o->Df[a][r] * phi[0][b][r][c];
              Gy += o->Df[b][r] * phi[1][a][r][c];
            }
            R[c * N + m * np + b * n + a] = -(2.0 / dx) * Fx - (2.0 / dy) * Gy;
          }
    }
}

/* ------------------------------------------------------------------------- */
/* FV residual with MUSCL reconstruction (Eqs. (6)-(8);   */
/* P:346-351; Alg. 1)                                                 */
/* ------------------------------------------------------------------------- */
/* cell index along a line with 2 ghost layers: periodic wrap, transmissive clamp */
static int fv_idx(int i, int n, int bc) {
  if (bc == ORC_PERIODIC) return ((i % n) + n) % n;
  return i < 0 ? 0 : (i >= n ? n - 1 : i);
}

/* face states at face between cells q0 (=i) and q1 (=i+1), stencil qm1, q0, q1, q2.
 * unlim = 1: the same kappa-schemes without the limiter (Q10 alternative, f3):
 * MUSCL-2 kappa = 0, q_W = q_i + (dm + dp)/4; MUSCL-3 kappa = 1/3 with the raw
 * differences in place of the two minmods (van Leer's kappa-scheme). */
/* emW / emE: optional decision-map entries of cells i and i+1 (the cell whose
 * slope each minmod limits) */
static void muscl_face(int order, const double *qm1, const double *q0, const double *q1, const double *q2,
                       double *qW, double *qE, int64_t *cnt, int unlim, int64_t *emW, int64_t *emE) {
  for (int c = 0; c < 4; ++c) {
    if (unlim) {
      const double kap = order == 1 ? 0.0 : 1.0 / 3.0;
      double dm0 = q0[c] - qm1[c], dp0 = q1[c] - q0[c];   /* cell i   */
      double dm1 = q1[c] - q0[c], dp1 = q2[c] - q1[c];    /* cell i+1 */
      qW[c] = q0[c] + 0.25 * ((1.0 - kap) * dm0 + (1.0 + kap) * dp0);
      qE[c] = q1[c] - 0.25 * ((1.0 - kap) * dp1 + (1.0 + kap) * dm1);
    } else if (order == 1) {
      double s0 = mm2c(q0[c] - qm1[c], q1[c] - q0[c], cnt, emW);
      double s1 = mm2c(q1[c] - q0[c], q2[c] - q1[c], cnt, emE);
      qW[c] = q0[c] + 0.5 * s0;
      qE[c] = q1[c] - 0.5 * s1;
    } else {
      const double kap = 1.0 / 3.0, beta = (3.0 - kap) / (1.0 - kap);
      double dm0 = q0[c] - qm1[c], dp0 = q1[c] - q0[c];   /* cell i   */
      double dm1 = q1[c] - q0[c], dp1 = q2[c] - q1[c];    /* cell i+1 */
      qW[c] = q0[c] + 0.25 * ((1.0 - kap) * mm2c(dm0, beta * dp0, cnt, emW) + (1.0 + kap) * mm2c(dp0, beta * dm0, cnt, emW));
      qE[c] = q1[c] - 0.25 * ((1.0 - kap) * mm2c(dp1, beta * dm1, cnt, emE) + (1.0 + kap) * mm2c(dm1, beta * dp1, cnt, emE));
    }
  }
}

void orc_muscl_face(int order, const double *qm1, const double *q0, const double *q1, const double *q2,
                    double *qW, double *qE) {
  muscl_face(order, qm1, q0, q1, q2, qW, qE, NULL, 0, NULL, NULL);
}

void orc_muscl_face_unlimited(int order, const double *qm1, const double *q0, const double *q1, const double *q2,
                              double *qW, double *qE) {
  muscl_face(order, qm1, q0, q1, q2, qW, qE, NULL, 1, NULL, NULL);
}

/* emap (nullable): per-cell decision map, the cell index after the periodic wrap
 * / transmissive clamp of fv_idx */
static void residual_fv(const orc_config *cf, const double *Q, double *R, int64_t *cnt, int64_t *emap) {
  phys_t P = mkphys(cf);
  int nx = cf->nx, ny = cf->ny;
  int64_t N = (int64_t)nx * ny;
  double dx = (cf->xmax - cf->xmin) / nx, dy = (cf->ymax - cf->ymin) / ny;
  /* face fluxes stored separately, then differenced (the paper's 2 kernels) */
  double *Fx = (double *)malloc(sizeof(double) * 4 * (size_t)(nx + 1) * ny);
  double *Gy = (double *)malloc(sizeof(double) * 4 * (size_t)nx * (ny + 1));
#pragma omp parallel for if (!cnt && !emap) schedule(static)
  for (int j = 0; j < ny; ++j)
    for (int f = 0; f <= nx; ++f) {   /* face f between cells f-1 and f */
      double s[4][4], qW[4], qE[4], F[4];
      for (int t = 0; t < 4; ++t) getq(Q, N, (int64_t)j * nx + fv_idx(f - 2 + t, nx, cf->bc), 1, 0, s[t]);
      muscl_face(cf->k, s[0], s[1], s[2], s[3], qW, qE, cnt, cf->fv_unlimited,
                 emap ? emap + (int64_t)j * nx + fv_idx(f - 1, nx, cf->bc) : NULL,
                 emap ? emap + (int64_t)j * nx + fv_idx(f, nx, cf->bc) : NULL);
      rusanov(&P, 0, qW, qE, F);
      for (int c = 0; c < 4; ++c) Fx[((size_t)j * (nx + 1) + f) * 4 + c] = F[c];
    }
#pragma omp parallel for if (!cnt && !emap) schedule(static)
  for (int f = 0; f <= ny; ++f)
    for (int i = 0; i < nx; ++i) {
      double s[4][4], qW[4], qE[4], F[4];
      for (int t = 0; t < 4; ++t) getq(Q, N, (int64_t)fv_idx(f - 2 + t, ny, cf->bc) * nx + i, 1, 0, s[t]);
      muscl_face(cf->k, s[0], s[1], s[2], s[3], qW, qE, cnt, cf->fv_unlimited,
                 emap ? emap + (int64_t)fv_idx(f - 1, ny, cf->bc) * nx + i : NULL,
                 emap ? emap + (int64_t)fv_idx(f, ny, cf->bc) * nx + i : NULL);
      rusanov(&P, 1, qW, qE, F);
      for (int c = 0; c < 4; ++c) Gy[((size_t)f * nx + i) * 4 + c] = F[c];
    }
#pragma omp parallel for schedule(static)
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i)
      for (int c = 0; c < 4; ++c)
        R[c * N + (int64_t)j * nx + i] =
            -(Fx[((size_t)j * (nx + 1) + i + 1) * 4 + c] - Fx[((size_t)j * (nx + 1) + i) * 4 + c]) / dx
            - (Gy[((size_t)(j + 1) * nx + i) * 4 + c] - Gy[((size_t)j * nx + i) * 4 + c]) / dy;
  free(Fx);
  free(Gy);
}

/* ------------------------------------------------------------------------- */
/* public: residual                                                            */
/* ------------------------------------------------------------------------- */
/* emap (nullable, FV only): per-cell minmod outcomes, see mm2c */
int orc_residual_map(const orc_config *cf, const double *Q, double *R, int64_t *cnt, int64_t *emap) {
  int st = check_cfg(cf);
  if (st) return st;
  if (cf->method == ORC_FV) { residual_fv(cf, Q, R, cnt, emap); return ORC_OK; }
  ops_t o;
  build_ops(cf->method, cf->k, &o);
  if (cf->method == ORC_CPR || cf->method == ORC_NDG) residual_cpr_ndg(cf, &o, Q, R);
  else if (cf->method == ORC_DG && cf->dg_overintegrate) residual_dg_quad(cf, &o, cf->k + 2, Q, R);
  else if (cf->method == ORC_DG) residual_dg(cf, &o, Q, R);
  else residual_sd(cf, &o, Q, R);
  return ORC_OK;
}

int orc_residual(const orc_config *cf, const double *Q, double *R, int64_t *cnt) {
  return orc_residual_map(cf, Q, R, cnt, NULL);
}

/* ------------------------------------------------------------------------- */
/* element averages (Alg. 9; G7: accumulate) and the HO limiter     */
/* (Eq. (35); Algs. 10-11)                     */
/* ------------------------------------------------------------------------- */
int orc_averages(const orc_config *cf, const double *Q, double *Qbar) {
  int st = check_cfg(cf);
  if (st) return st;
  int64_t Ne = (int64_t)cf->nx * cf->ny;
  if (cf->method == ORC_FV) { memcpy(Qbar, Q, sizeof(double) * 4 * Ne); return ORC_OK; }
  ops_t o;
  build_ops(cf->method, cf->k, &o);
  int n = o.n, np = n * n;
  int64_t N = Ne * np;
  for (int c = 0; c < 4; ++c)
    for (int64_t m = 0; m < Ne; ++m) {
      double s = 0.0;
      for (int b = 0; b < n; ++b)
        for (int a = 0; a < n; ++a) s += o.w[a] * o.w[b] * Q[c * N + m * np + b * n + a];
      Qbar[c * Ne + m] = 0.25 * s;
    }
  return ORC_OK;
}

/* applies the limiter in place; marks[m] = 1 if element m was limited (nullable) */
int orc_limit(const orc_config *cf, double *Q, int32_t *marks, int64_t *cnt) {
  int st = check_cfg(cf);
  if (st) return st;
  if (cf->method == ORC_FV) return ORC_ERR_ARG;
  ops_t o;
  build_ops(cf->method, cf->k, &o);
  int n = o.n, np = n * n, gll = is_gll(cf->method);
  int nx = cf->nx, ny = cf->ny;
  int64_t Ne = (int64_t)nx * ny, N = Ne * np;
  double dx = (cf->xmax - cf->xmin) / nx, dy = (cf->ymax - cf->ymin) / ny;
  double eps = cf->limiter_eps;
  /* step 1: all averages before any element is limited (Jacobi) */
  double *Qbar = (double *)malloc(sizeof(double) * 4 * Ne);
  int32_t *mk = (int32_t *)calloc((size_t)Ne, sizeof(int32_t));
  orc_averages(cf, Q, Qbar);
  /* step 2: detect on density (limiter_all_vars: on every conserved component)
   * at every edge point */
  const int nvar = cf->limiter_all_vars ? 4 : 1;
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      int64_t m = (int64_t)j * nx + i;
      int iw = nb_index(i, -1, nx, cf->bc), ie = nb_index(i, 1, nx, cf->bc);
      int js = nb_index(j, -1, ny, cf->bc), jn = nb_index(j, 1, ny, cf->bc);
      int trip = 0;
      for (int c = 0; c < nvar; ++c) {
        double qb = Qbar[c * Ne + m];
        double qW = iw >= 0 ? Qbar[c * Ne + (int64_t)j * nx + iw] : qb;
        double qE = ie >= 0 ? Qbar[c * Ne + (int64_t)j * nx + ie] : qb;
        double qS = js >= 0 ? Qbar[c * Ne + (int64_t)js * nx + i] : qb;
        double qN = jn >= 0 ? Qbar[c * Ne + (int64_t)jn * nx + i] : qb;
        for (int s = 0; s < 4; ++s)
          for (int t = 0; t < n; ++t) {
            double qt[4];
            trace(&o, gll, Q, N, m, s, t, qt);
            double ql = qt[c], qe;
            double qp = (s <= 1) ? qE : qN, qm = (s <= 1) ? qW : qS;
            if (s == 1 || s == 3) {           /* right / top side */
              qe = qb + mm3(ql - qb, qp - qb, qb - qm);
            } else {                          /* left / bottom side */
              qe = qb - mm3(qb - ql, qp - qb, qb - qm);
            }
            if (fabs(ql - qe) > eps) trip = 1;
          }
      }
      mk[m] = trip;
    }
  /* step 3: rebuild marked elements from neighbour averages (Eq. (35), Q14) */
  int64_t nmarked = 0;
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      int64_t m = (int64_t)j * nx + i;
      if (marks) marks[m] = mk[m];
      if (!mk[m]) continue;
      ++nmarked;
      int iw = nb_index(i, -1, nx, cf->bc), ie = nb_index(i, 1, nx, cf->bc);
      int js = nb_index(j, -1, ny, cf->bc), jn = nb_index(j, 1, ny, cf->bc);
      double qb[4], dE[4], dW[4], dN[4], dS[4], sx[4], sy[4];
      for (int c = 0; c < 4; ++c) {
        qb[c] = Qbar[c * Ne + m];
        double qW = iw >= 0 ? Qbar[c * Ne + (int64_t)j * nx + iw] : qb[c];
        double qE = ie >= 0 ? Qbar[c * Ne + (int64_t)j * nx + ie] : qb[c];
        double qS = js >= 0 ? Qbar[c * Ne + (int64_t)js * nx + i] : qb[c];
        double qN = jn >= 0 ? Qbar[c * Ne + (int64_t)jn * nx + i] : qb[c];
        dE[c] = (qE - qb[c]) / dx; dW[c] = (qb[c] - qW) / dx;
        dN[c] = (qN - qb[c]) / dy; dS[c] = (qb[c] - qS) / dy;
      }
      if (!cf->limiter_characteristic) {   /* componentwise (Q12 reading) */
        for (int c = 0; c < 4; ++c) { sx[c] = mm2(dE[c], dW[c], NULL); sy[c] = mm2(dN[c], dS[c], NULL); }
      } else {                             /* minmod of the characteristic fields at qbar, mapped back */
        phys_t P = mkphys(cf);
        for (int dir = 0; dir < 2; ++dir) {
          double R[4][4], L[4][4], wp[4], wm[4], sw[4];
          char_vectors(&P, dir, qb, R, L);
          const double *dp = dir == 0 ? dE : dN, *dm = dir == 0 ? dW : dS;
          for (int k = 0; k < 4; ++k) {
            wp[k] = 0.0; wm[k] = 0.0;
            for (int c = 0; c < 4; ++c) { wp[k] += L[k][c] * dp[c]; wm[k] += L[k][c] * dm[c]; }
            sw[k] = mm2(wp[k], wm[k], NULL);
          }
          double *so = dir == 0 ? sx : sy;
          for (int c = 0; c < 4; ++c) {
            so[c] = 0.0;
            for (int k = 0; k < 4; ++k) so[c] += R[c][k] * sw[k];
          }
        }
      }
      for (int c = 0; c < 4; ++c)
        for (int b = 0; b < n; ++b)
          for (int a = 0; a < n; ++a)
            Q[c * N + m * np + b * n + a] = qb[c] + (0.5 * dx) * o.xi[a] * sx[c] + (0.5 * dy) * o.xi[b] * sy[c];
    }
  if (cnt) cnt[DEC_MARKED] += nmarked;
  free(Qbar);
  free(mk);
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* time step (Eq. (36); Q4) and SSP-RK3 (Q2)              */
/* ------------------------------------------------------------------------- */
double orc_max_wave_speed(const orc_config *cf, const double *Q) {
  phys_t P = mkphys(cf);
  int64_t NP = (int64_t)cf->nx * cf->ny * points_per_elem(cf);
  double lam = 0.0;
  for (int64_t p = 0; p < NP; ++p) {
    double q[4];
    for (int c = 0; c < 4; ++c) q[c] = Q[c * NP + p];
    double s = wave_speed(&P, q);
    if (!(s <= lam)) lam = s;   /* NaN propagates */
  }
  return lam;
}

double orc_dt(const orc_config *cf, const double *Q) {
  if (cf->dt_fixed > 0.0) return cf->dt_fixed;
  double dx = (cf->xmax - cf->xmin) / cf->nx, dy = (cf->ymax - cf->ymin) / cf->ny;
  return cf->cfl * fmin(dx, dy) / orc_max_wave_speed(cf, Q);
}

typedef void (*orc_rhs_fn)(const double *q, double *r, void *ctx);
typedef void (*orc_post_fn)(double *q, void *ctx);

/* One SSP-RK3 (Shu-Osher) step of q' = L(q), with the stage operator Lambda
 * (limiter, or identity when post == NULL) after every stage; with post_last
 * only (limiter_per_step, f3) after the last stage. */
static void ssprk3_post(double *q, int64_t n, double dt, orc_rhs_fn rhs, orc_post_fn post, orc_post_fn post_last,
                        void *ctx);
void orc_ssprk3(double *q, int64_t n, double dt, orc_rhs_fn rhs, orc_post_fn post, void *ctx) {
  ssprk3_post(q, n, dt, rhs, post, post, ctx);
}
static void ssprk3_post(double *q, int64_t n, double dt, orc_rhs_fn rhs, orc_post_fn post, orc_post_fn post_last,
                        void *ctx) {
  double *q0 = (double *)malloc(sizeof(double) * n);
  double *r = (double *)malloc(sizeof(double) * n);
  memcpy(q0, q, sizeof(double) * n);
  rhs(q, r, ctx);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) q[i] = q0[i] + dt * r[i];                          /* q1 */
  if (post) post(q, ctx);
  rhs(q, r, ctx);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) q[i] = 0.75 * q0[i] + 0.25 * (q[i] + dt * r[i]);   /* q2 */
  if (post) post(q, ctx);
  rhs(q, r, ctx);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) q[i] = q0[i] / 3.0 + (2.0 / 3.0) * (q[i] + dt * r[i]); /* q^{n+1} */
  if (post_last) post_last(q, ctx);
  free(q0);
  free(r);
}

/* emap: per-element decision map (HO: stages in which the element was marked;
 * FV: per-cell minmod outcomes, mm2c), accumulated over the run */
typedef struct { const orc_config *cf; int64_t *cnt; int64_t *emap; int32_t *marks; } run_ctx;
static void run_rhs(const double *q, double *r, void *ctx) {
  run_ctx *c = (run_ctx *)ctx;
  orc_residual_map(c->cf, q, r, c->cnt, c->cf->method == ORC_FV ? c->emap : NULL);
}
static void run_post(double *q, void *ctx) {
  run_ctx *c = (run_ctx *)ctx;
  orc_limit(c->cf, q, c->emap ? c->marks : NULL, c->cnt);
  if (c->emap)
    for (int64_t m = 0; m < (int64_t)c->cf->nx * c->cf->ny; ++m) c->emap[m] += c->marks[m];
}

/* first non-physical point (rho <= 0, p <= 0 or non-finite), or -1 */
static int64_t first_nonphysical(const orc_config *cf, const double *Q) {
  phys_t P = mkphys(cf);
  int64_t NP = (int64_t)cf->nx * cf->ny * points_per_elem(cf);
  for (int64_t p = 0; p < NP; ++p) {
    double q[4];
    for (int c = 0; c < 4; ++c) q[c] = Q[c * NP + p];
    if (!(isfinite(q[0]) && isfinite(q[1]) && isfinite(q[2]) && isfinite(q[3]))) return p;
    if (cf->physics == 0 && (!(q[0] > 0.0) || !(pressure(&P, q) > 0.0))) return p;
  }
  return -1;
}

/* March until steps == max_steps or t == t_end; dt recomputed from q^n each step
 * and clipped to t_end - t.  *t is the start time on entry, the end time on exit. */
int orc_run_map(const orc_config *cf, double *Q, int32_t max_steps, double t_end, double *t,
                int64_t *steps, int64_t *cnt, int64_t *emap) {
  int st = check_cfg(cf);
  if (st) return st;
  int64_t n = (int64_t)4 * cf->nx * cf->ny * points_per_elem(cf);
  int32_t *marks = emap ? (int32_t *)calloc((size_t)cf->nx * cf->ny, sizeof(int32_t)) : NULL;
  run_ctx ctx = { cf, cnt, emap, marks };
  int use_lim = cf->limiter && cf->method != ORC_FV;
  int64_t s = 0;
  while (s < max_steps && *t < t_end) {
    double dt = orc_dt(cf, Q);
    if (dt > t_end - *t) dt = t_end - *t;
    ssprk3_post(Q, n, dt, run_rhs, use_lim && !cf->limiter_per_step ? run_post : NULL, use_lim ? run_post : NULL,
                &ctx);
    *t += dt;
    ++s;
    if (first_nonphysical(cf, Q) >= 0) { if (steps) *steps = s; free(marks); return ORC_ERR_NONPHYSICAL; }
  }
  if (steps) *steps = s;
  free(marks);
  return ORC_OK;
}

int orc_run(const orc_config *cf, double *Q, int32_t max_steps, double t_end, double *t,
            int64_t *steps, int64_t *cnt) {
  return orc_run_map(cf, Q, max_steps, t_end, t, steps, cnt, NULL);
}

/* ------------------------------------------------------------------------- */
/* test cases (P:897-913 vortex; P:1043-1047 radial shock tube)    */
/* ------------------------------------------------------------------------- */
static double wrapc(double s, double lo, double hi) {
  double L = hi - lo;
  return s - L * floor((s - lo) / L);
}

/* conserved isentropic-vortex state at (x,y,t): mean (1,1,0,1), eps = 5;
 * exact solution = initial field advected by (t, 0), single periodic image (Q19) */
void orc_vortex_state(const orc_config *cf, double x, double y, double t, double *q) {
  const double eps = 5.0, PI = 3.14159265358979323846;
  double g = cf->gamma;
  double xs = wrapc(x - t, cf->xmin, cf->xmax), ys = wrapc(y, cf->ymin, cf->ymax);
  double r2 = xs * xs + ys * ys;
  double du = -(eps / (2.0 * PI)) * exp(0.5 * (1.0 - r2)) * ys;
  double dv = (eps / (2.0 * PI)) * exp(0.5 * (1.0 - r2)) * xs;
  double T = 1.0 - (g - 1.0) * eps * eps / (8.0 * g * PI * PI) * exp(1.0 - r2);
  double rho = pow(T, 1.0 / (g - 1.0));
  double p = rho * T;
  double u = 1.0 + du, v = dv;
  q[0] = rho; q[1] = rho * u; q[2] = rho * v; q[3] = p / (g - 1.0) + 0.5 * rho * (u * u + v * v);
}

/* radial shock tube: (rho,p) = (1,1) inside r < 0.4 (strict), else (0.125,0.1) */
void orc_shock_state(const orc_config *cf, double x, double y, double *q) {
  double g = cf->gamma;
  int in = x * x + y * y < 0.16;
  double rho = in ? 1.0 : 0.125, p = in ? 1.0 : 0.1;
  q[0] = rho; q[1] = 0.0; q[2] = 0.0; q[3] = p / (g - 1.0);
}

static void case_state(const orc_config *cf, int case_id, double x, double y, double t, double *q) {
  if (case_id == ORC_CASE_VORTEX) orc_vortex_state(cf, x, y, t, q);
  else orc_shock_state(cf, x, y, q);
}

/* exact element average by 8x8 Gauss-Legendre quadrature */
static void exact_average(const orc_config *cf, int case_id, int i, int j, double t, double *qa) {
  double xg[8], wg[8];
  orc_nodes(0, 8, xg, wg);
  double dx = (cf->xmax - cf->xmin) / cf->nx, dy = (cf->ymax - cf->ymin) / cf->ny;
  double xc = cf->xmin + (i + 0.5) * dx, yc = cf->ymin + (j + 0.5) * dy;
  for (int c = 0; c < 4; ++c) qa[c] = 0.0;
  for (int b = 0; b < 8; ++b)
    for (int a = 0; a < 8; ++a) {
      double q[4];
      case_state(cf, case_id, xc + 0.5 * dx * xg[a], yc + 0.5 * dy * xg[b], t, q);
      for (int c = 0; c < 4; ++c) qa[c] += 0.25 * wg[a] * wg[b] * q[c];
    }
}

/* HO: pointwise at the solution points (Q21); FV: 8x8-GL cell averages (Q22).
 * With the limiter on, Lambda is applied once to the initial data (Q13). */
int orc_init_case(const orc_config *cf, int case_id, double *Q) {
  int st = check_cfg(cf);
  if (st) return st;
  if (case_id != ORC_CASE_VORTEX && case_id != ORC_CASE_SHOCK) return ORC_ERR_ARG;
  int nx = cf->nx, ny = cf->ny;
  double dx = (cf->xmax - cf->xmin) / nx, dy = (cf->ymax - cf->ymin) / ny;
  if (cf->method == ORC_FV) {
    int64_t N = (int64_t)nx * ny;
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        double qa[4];
        exact_average(cf, case_id, i, j, 0.0, qa);
        for (int c = 0; c < 4; ++c) Q[c * N + (int64_t)j * nx + i] = qa[c];
      }
    return ORC_OK;
  }
  ops_t o;
  build_ops(cf->method, cf->k, &o);
  int n = o.n, np = n * n;
  int64_t N = (int64_t)nx * ny * np;
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i)
      for (int b = 0; b < n; ++b)
        for (int a = 0; a < n; ++a) {
          double x = cf->xmin + (i + 0.5) * dx + 0.5 * dx * o.xi[a];
          double y = cf->ymin + (j + 0.5) * dy + 0.5 * dy * o.xi[b];
          double q[4];
          case_state(cf, case_id, x, y, 0.0, q);
          for (int c = 0; c < 4; ++c) Q[c * N + ((int64_t)j * nx + i) * np + b * n + a] = q[c];
        }
  if (cf->limiter) orc_limit(cf, Q, NULL, NULL);
  return ORC_OK;
}

/* solution-point coordinates (for tests): x[m*np+p], y[m*np+p] */
int orc_point_coords(const orc_config *cf, double *X, double *Y) {
  int st = check_cfg(cf);
  if (st) return st;
  int nx = cf->nx, ny = cf->ny;
  double dx = (cf->xmax - cf->xmin) / nx, dy = (cf->ymax - cf->ymin) / ny;
  if (cf->method == ORC_FV) {
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        X[(int64_t)j * nx + i] = cf->xmin + (i + 0.5) * dx;
        Y[(int64_t)j * nx + i] = cf->ymin + (j + 0.5) * dy;
      }
    return ORC_OK;
  }
  ops_t o;
  build_ops(cf->method, cf->k, &o);
  int n = o.n, np = n * n;
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i)
      for (int b = 0; b < n; ++b)
        for (int a = 0; a < n; ++a) {
          int64_t idx = ((int64_t)j * nx + i) * np + b * n + a;
          X[idx] = cf->xmin + (i + 0.5) * dx + 0.5 * dx * o.xi[a];
          Y[idx] = cf->ymin + (j + 0.5) * dy + 0.5 * dy * o.xi[b];
        }
  return ORC_OK;
}

/* FV reconstructed solution ("For P^2 FV, the error was computed by
 * reconstructing the solution along element faces, and then using a quadrature
 * rule to compute an averaged solution"; reading R22 in DESIGN.md).  Per cell
 * and direction, the scheme's own MUSCL face states (muscl_face: lo = the state
 * at the cell's i-1/2 face, hi = at its i+1/2 face, limited as in the residual)
 * and the cell average qbar fix the quadratic on [-1,1]
 *   q_d(s) = qbar + (hi - lo)/2 s + (hi + lo - 2 qbar)/4 (3 s^2 - 1)
 * (q_d(-1) = lo, q_d(1) = hi, mean qbar; linear for MUSCL-2, where
 * hi + lo = 2 qbar).  The cell's solution is q(xi, eta) = q_x(xi) + q_y(eta) -
 * qbar, evaluated at the 3x3 Gauss-Legendre points (xi_a, eta_b) of the cell,
 * out[(m*3 + b)*3 + a] (component var). */
int orc_fv_recon_points(const orc_config *cf, const double *Q, int var, double *out) {
  int st = check_cfg(cf);
  if (st) return st;
  if (cf->method != ORC_FV || var < 0 || var > 3) return ORC_ERR_ARG;
  int nx = cf->nx, ny = cf->ny;
  int64_t N = (int64_t)nx * ny;
  double xg[3], wg[3];
  orc_nodes(0, 3, xg, wg);
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      double s[5][4], qW[4], qE[4], lo[2], hi[2];
      /* x: faces i-1/2 (cells i-2..i+1; qE is cell i's lo) and i+1/2 (cells i-1..i+2; qW is its hi) */
      for (int t = 0; t < 5; ++t) getq(Q, N, (int64_t)j * nx + fv_idx(i - 2 + t, nx, cf->bc), 1, 0, s[t]);
      muscl_face(cf->k, s[0], s[1], s[2], s[3], qW, qE, NULL, cf->fv_unlimited, NULL, NULL);
      lo[0] = qE[var];
      muscl_face(cf->k, s[1], s[2], s[3], s[4], qW, qE, NULL, cf->fv_unlimited, NULL, NULL);
      hi[0] = qW[var];
      const double qb = s[2][var];
      for (int t = 0; t < 5; ++t) getq(Q, N, (int64_t)fv_idx(j - 2 + t, ny, cf->bc) * nx + i, 1, 0, s[t]);
      muscl_face(cf->k, s[0], s[1], s[2], s[3], qW, qE, NULL, cf->fv_unlimited, NULL, NULL);
      lo[1] = qE[var];
      muscl_face(cf->k, s[1], s[2], s[3], s[4], qW, qE, NULL, cf->fv_unlimited, NULL, NULL);
      hi[1] = qW[var];
      for (int b = 0; b < 3; ++b)
        for (int a = 0; a < 3; ++a) {
          double sx = xg[a], sy = xg[b];
          double qx = qb + 0.5 * (hi[0] - lo[0]) * sx + 0.25 * (hi[0] + lo[0] - 2.0 * qb) * (3.0 * sx * sx - 1.0);
          double qy = qb + 0.5 * (hi[1] - lo[1]) * sy + 0.25 * (hi[1] + lo[1] - 2.0 * qb) * (3.0 * sy * sy - 1.0);
          out[((int64_t)j * nx + i) * 9 + b * 3 + a] = qx + qy - qb;
        }
    }
  return ORC_OK;
}

/* L1/L2/Linf of the error in component var at time t (vortex only).
 * HO methods: pointwise error at the solution points, weighted by the
 * solution-point quadrature, i.e. the RMS over the domain of q_h - q_exact:
 *   L2 = sqrt( sum_m sum_ab (w_a w_b / 4) d_ab^2 / N_e ),  L1 likewise with |d|,
 *   Linf = max |d_ab|.
 * This reading of "L2 error norm of rho" reproduces Tables
 * 2-3 to the printed 3 digits (tests/golden/paper_tables_2_3.txt).
 * FV: the cell value against the exact cell average (8x8 Gauss-Legendre); with
 * fv_error_recon (R22) the same pointwise convention as HO applied to
 * the reconstructed solution of orc_fv_recon_points at the 3x3 GL points. */
int orc_error(const orc_config *cf, const double *Q, int case_id, double t, int var,
              double *l1, double *l2, double *linf) {
  int st = check_cfg(cf);
  if (st) return st;
  if (case_id != ORC_CASE_VORTEX || var < 0 || var > 3) return ORC_ERR_ARG;
  int nx = cf->nx, ny = cf->ny;
  int64_t Ne = (int64_t)nx * ny;
  double dx = (cf->xmax - cf->xmin) / nx, dy = (cf->ymax - cf->ymin) / ny;
  double s1 = 0.0, s2 = 0.0, mx = 0.0;
  if (cf->method == ORC_FV && cf->fv_error_recon) {
    double *qr = (double *)malloc(sizeof(double) * 9 * (size_t)Ne);
    if (!qr) return ORC_ERR_NOMEM;
    orc_fv_recon_points(cf, Q, var, qr);
    double xg[3], wg[3];
    orc_nodes(0, 3, xg, wg);
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i)
        for (int b = 0; b < 3; ++b)
          for (int a = 0; a < 3; ++a) {
            double x = cf->xmin + (i + 0.5) * dx + 0.5 * dx * xg[a];
            double y = cf->ymin + (j + 0.5) * dy + 0.5 * dy * xg[b];
            double qe[4];
            case_state(cf, case_id, x, y, t, qe);
            double d = qr[((int64_t)j * nx + i) * 9 + b * 3 + a] - qe[var];
            double wq = 0.25 * wg[a] * wg[b];
            s1 += wq * fabs(d);
            s2 += wq * d * d;
            if (fabs(d) > mx) mx = fabs(d);
          }
    free(qr);
  } else if (cf->method == ORC_FV) {
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        double qa[4];
        exact_average(cf, case_id, i, j, t, qa);
        double d = Q[var * Ne + (int64_t)j * nx + i] - qa[var];
        s1 += fabs(d);
        s2 += d * d;
        if (fabs(d) > mx) mx = fabs(d);
      }
  } else {
    ops_t o;
    build_ops(cf->method, cf->k, &o);
    int n = o.n, np = n * n;
    int64_t N = Ne * np;
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i)
        for (int b = 0; b < n; ++b)
          for (int a = 0; a < n; ++a) {
            double x = cf->xmin + (i + 0.5) * dx + 0.5 * dx * o.xi[a];
            double y = cf->ymin + (j + 0.5) * dy + 0.5 * dy * o.xi[b];
            double qe[4];
            case_state(cf, case_id, x, y, t, qe);
            double d = Q[var * N + ((int64_t)j * nx + i) * np + b * n + a] - qe[var];
            double wq = 0.25 * o.w[a] * o.w[b];
            s1 += wq * fabs(d);
            s2 += wq * d * d;
            if (fabs(d) > mx) mx = fabs(d);
          }
  }
  *l1 = s1 / (double)Ne;
  *l2 = sqrt(s2 / (double)Ne);
  *linf = mx;
  return ORC_OK;
}
