/*
 * oracle.c — plain, slow, fp64 CPU oracle of the hot path of arXiv 2603.28907
 * ("Bayesian muon tomography of block caves"): exact ray tracing through the
 * bilinear muck-top / cave-back height fields, opacity, Poisson likelihood,
 * CAR-copula prior, log-posterior and its reverse-mode gradient.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_2603_28907_b200/csrc) and neither side includes the other.
 *
 * Citations: "P:a-b" = /root/reference/PAPER.md lines a-b; "R<k>" = reading k
 * of the ambiguity register in DESIGN.md (§ "Readings of the paper").
 * Every function is pinned by a `-m "not gpu"` test (tests/test_oracle_*.py);
 * see DESIGN.md "Oracle pins".
 *
 * Precision: everything in double.  Inputs are the canonical fp32 arrays,
 * promoted exactly.  Node coordinates and detector positions are multiples of
 * 2^-12 m with |v| < 2^11 (R3), so every difference X_k - o_x is exact and every
 * product (X_k - o_x)*|d_y| of two 24-bit numbers is exact in double: the
 * traversal predicates below are exact comparisons.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_PI 3.14159265358979323846
#define OR_TCLAMP 10.0 /* R18: |t| <= 10, derivative 0 beyond */

typedef struct {
  int nx, ny;
  double *X, *Y;           /* node coordinates [nx], [ny] (R3) */
  double z_top;            /* known flat top surface (R6) */
  double rho_m, rho_a, rho_r, rho_e; /* unit densities (R8); rho_e beyond the footprint (R7) */
  double Lambda;           /* attenuation length of I(O) = I0 exp(-O/Lambda) (R9) */
  double r[2];             /* CAR dependence r_l, fixed (R13) */
  int ndet;
  double *det;             /* [ndet][3] */
  long nray;
  int *rdet;               /* [nray] */
  double *dir;             /* [nray][3] unit, d_z > 0 */
  double *w;               /* [nray] Δt·I0·ΔΩ_p·ε_p  (R9, R10) */
  double *cnt;             /* [nray] observed counts C_p */
} or_problem;

/* ------------------------------------------------------------------ */
/* problem                                                             */
/* ------------------------------------------------------------------ */
or_problem *or_problem_new(int nx, int ny, const float *X, const float *Y, float z_top,
                           double rho_m, double rho_a, double rho_r, double rho_e, double Lambda,
                           double r0, double r1, int ndet, const float *det, long nray,
                           const int *rdet, const float *dir, const float *w, const int *cnt) {
  or_problem *p = (or_problem *)calloc(1, sizeof(or_problem));
  p->nx = nx; p->ny = ny;
  p->X = (double *)malloc(sizeof(double) * nx);
  p->Y = (double *)malloc(sizeof(double) * ny);
  for (int i = 0; i < nx; i++) p->X[i] = X[i];
  for (int j = 0; j < ny; j++) p->Y[j] = Y[j];
  p->z_top = z_top;
  p->rho_m = rho_m; p->rho_a = rho_a; p->rho_r = rho_r; p->rho_e = rho_e; p->Lambda = Lambda;
  p->r[0] = r0; p->r[1] = r1;
  p->ndet = ndet;
  p->det = (double *)malloc(sizeof(double) * 3 * ndet);
  for (int i = 0; i < 3 * ndet; i++) p->det[i] = det[i];
  p->nray = nray;
  p->rdet = (int *)malloc(sizeof(int) * nray);
  p->dir = (double *)malloc(sizeof(double) * 3 * nray);
  p->w = (double *)malloc(sizeof(double) * nray);
  p->cnt = (double *)malloc(sizeof(double) * nray);
  for (long q = 0; q < nray; q++) {
    p->rdet[q] = rdet[q];
    for (int k = 0; k < 3; k++) p->dir[3 * q + k] = dir[3 * q + k];
    p->w[q] = w[q];
    p->cnt[q] = cnt[q];
  }
  return p;
}

void or_problem_free(or_problem *p) {
  if (!p) return;
  free(p->X); free(p->Y); free(p->det); free(p->rdet); free(p->dir); free(p->w); free(p->cnt);
  free(p);
}

/* ------------------------------------------------------------------ */
/* CAR prior on the periodic 4-neighbour grid              */
/* ------------------------------------------------------------------ */

/* Q = diag(A1) - rA on the torus is block-circulant;
 * its eigenvalues are 4 - 2r(cos 2πa/nx + cos 2πb/ny).  Σ_ii = (Q^-1)_ii is the
 * same for every node and equals the mean of 1/eigenvalue.
 * sigma = sqrt(Σ_ii) is the scale of the c.d.f. transform (R14);
 * logdet = ln det Q = Σ ln eigenvalue. */
void or_torus_spectrum(int nx, int ny, double r, double *sigma, double *logdet) {
  double s = 0.0, ld = 0.0;
  for (int a = 0; a < nx; a++)
    for (int b = 0; b < ny; b++) {
      double lam = 4.0 - 2.0 * r * (cos(2.0 * OR_PI * a / nx) + cos(2.0 * OR_PI * b / ny));
      s += 1.0 / lam;
      ld += log(lam);
    }
  *sigma = sqrt(s / ((double)nx * ny));
  *logdet = ld;
}

/* log N(x_l; 0, Q_l^-1) = -1/2 x^T Q x + 1/2 ln det Q - (N/2) ln 2π and its
 * gradient -Q x, for one surface.  Q_ii = |{j ~ i}| = 4 and Q_ij = -r for the
 * four periodic neighbours. */
double or_prior_surface(int nx, int ny, double r, const double *x, double *grad_out) {
  double sigma, ld;
  or_torus_spectrum(nx, ny, r, &sigma, &ld);
  double quad = 0.0;
  for (int i = 0; i < nx; i++)
    for (int j = 0; j < ny; j++) {
      int ip = (i + 1) % nx, im = (i - 1 + nx) % nx, jp = (j + 1) % ny, jm = (j - 1 + ny) % ny;
      double nb = x[ip * ny + j] + x[im * ny + j] + x[i * ny + jp] + x[i * ny + jm];
      double Qx = 4.0 * x[i * ny + j] - r * nb;
      quad += x[i * ny + j] * Qx;
      if (grad_out) grad_out[i * ny + j] = -Qx;
    }
  double N = (double)nx * ny;
  return -0.5 * quad + 0.5 * ld - 0.5 * N * log(2.0 * OR_PI);
}

/* ------------------------------------------------------------------ */
/* latent -> heights: Gaussian copula + stick-breaking     */
/* ------------------------------------------------------------------ */

/* Per node: t = clamp(x/σ, ±10) (R18); ǔ = Φ(t); H_1 = ǔ_1 z_top,
 * H_2 = (1-ǔ_2) H_1 + ǔ_2 z_top (P:466-470 with H_{n_layers} = z_top).
 * Here index 0 = paper layer 1 (muck top), 1 = paper layer 2 (cave back) (R4).
 * x, H: [2][nx][ny].  dH (optional) [3][nx][ny]: dH0/dx0, dH1/dx0, dH1/dx1. */
void or_heights(const or_problem *p, const double *x, double *H, double *dH) {
  int N = p->nx * p->ny;
  double sig[2], ld;
  for (int l = 0; l < 2; l++) or_torus_spectrum(p->nx, p->ny, p->r[l], &sig[l], &ld);
  for (int k = 0; k < N; k++) {
    double u[2], dudx[2];
    for (int l = 0; l < 2; l++) {
      double tt = x[l * N + k] / sig[l];
      int clamped = 0;
      if (tt > OR_TCLAMP) { tt = OR_TCLAMP; clamped = 1; }
      if (tt < -OR_TCLAMP) { tt = -OR_TCLAMP; clamped = 1; }
      u[l] = 0.5 * erfc(-tt / sqrt(2.0));                       /* Φ(t) */
      dudx[l] = clamped ? 0.0 : exp(-0.5 * tt * tt) / sqrt(2.0 * OR_PI) / sig[l];
    }
    double H0 = u[0] * p->z_top;
    double H1 = (1.0 - u[1]) * H0 + u[1] * p->z_top;
    H[k] = H0;
    H[N + k] = H1;
    if (dH) {
      dH[k] = p->z_top * dudx[0];                  /* ∂H0/∂x0 */
      dH[N + k] = (1.0 - u[1]) * p->z_top * dudx[0]; /* ∂H1/∂x0 */
      dH[2 * N + k] = (p->z_top - H0) * dudx[1];     /* ∂H1/∂x1 */
    }
  }
}

/* ------------------------------------------------------------------ */
/* rays                                                                */
/* ------------------------------------------------------------------ */

/* In-box extent of the ray ϱ(n̂) that starts at the sensor:
 * s_exit = min(side exit, top exit z_top/d_z); L_ext = rock path beyond a side
 * exit up to z_top (R7). */
void or_ray_extent(const or_problem *p, long q, double *s_exit, double *L_ext) {
  const double *o = p->det + 3 * p->rdet[q], *d = p->dir + 3 * q;
  double s_top = (p->z_top - o[2]) / d[2];
  double s = s_top;
  if (d[0] > 0) s = fmin(s, (p->X[p->nx - 1] - o[0]) / d[0]);
  if (d[0] < 0) s = fmin(s, (p->X[0] - o[0]) / d[0]);
  if (d[1] > 0) s = fmin(s, (p->Y[p->ny - 1] - o[1]) / d[1]);
  if (d[1] < 0) s = fmin(s, (p->Y[0] - o[1]) / d[1]);
  *s_exit = s;
  *L_ext = s_top - s;
}

/* a/b < c/d for a,c >= 0, b,d > 0, exactly (products of 24-bit values) */
static int frac_lt(double a, double b, double c, double d) { return a * d < c * b; }
static int frac_eq(double a, double b, double c, double d) { return a * d == c * b; }

/* Cell index along one axis containing coordinate o, taking the cell in the
 * direction of travel when o lies on a line (R16). */
static int start_cell(const double *X, int n, double o, double d) {
  int i = 0;
  for (int k = 0; k < n - 1; k++)
    if (d < 0 ? (X[k] < o) : (X[k] <= o)) i = k;
  if (i > n - 2) i = n - 2;
  return i;
}

/* Ordered list of control-grid cells (i,j) with positive-length intersection
 * with the in-box segment [0, s_exit] of ray q, with their [s_in, s_out].
 * Events (next x-line, next y-line, top) are ordered by exact comparisons;
 * a vertex hit steps both indices (R16).  Returns the number of cells; writes
 * at most cap entries. */
int or_traverse(const or_problem *p, long q, int *ij, double *s_in, double *s_out, int cap) {
  const double *o = p->det + 3 * p->rdet[q], *d = p->dir + 3 * q;
  int nx = p->nx, ny = p->ny;
  int i = start_cell(p->X, nx, o[0], d[0]);
  int j = start_cell(p->Y, ny, o[1], d[1]);
  int sx = d[0] > 0 ? 1 : (d[0] < 0 ? -1 : 0);
  int sy = d[1] > 0 ? 1 : (d[1] < 0 ? -1 : 0);
  double adx = fabs(d[0]), ady = fabs(d[1]);
  double s = 0.0;
  int n = 0;
  for (;;) {
    /* candidate events as fractions num/den */
    double nx_num = 0, ny_num = 0;
    int hx = 0, hy = 0;
    if (sx) { int k = sx > 0 ? i + 1 : i; nx_num = fabs(p->X[k] - o[0]); hx = 1; }
    if (sy) { int k = sy > 0 ? j + 1 : j; ny_num = fabs(p->Y[k] - o[1]); hy = 1; }
    double top_num = p->z_top - o[2], top_den = d[2];
    /* earliest event: start with top */
    double en = top_num, ed = top_den;
    int ex = 0, ey = 0, et = 1;
    if (hx) {
      if (frac_lt(nx_num, adx, en, ed)) { en = nx_num; ed = adx; ex = 1; ey = 0; et = 0; }
      else if (frac_eq(nx_num, adx, en, ed)) { ex = 1; }
    }
    if (hy) {
      if (frac_lt(ny_num, ady, en, ed)) { en = ny_num; ed = ady; ey = 1; ex = 0; et = 0; }
      else if (frac_eq(ny_num, ady, en, ed)) { ey = 1; }
    }
    double s_ev = en / ed;
    if (n < cap) {
      ij[2 * n] = i; ij[2 * n + 1] = j;
      s_in[n] = s; s_out[n] = s_ev;
    }
    n++;
    if (et) break;                                     /* top exit */
    int wall = 0;
    if (ex) { if ((sx > 0 && i + 1 == nx - 1) || (sx < 0 && i == 0)) wall = 1; }
    if (ey) { if ((sy > 0 && j + 1 == ny - 1) || (sy < 0 && j == 0)) wall = 1; }
    if (wall) break;                                   /* side exit */
    if (ex) i += sx;
    if (ey) j += sy;
    s = s_ev;
  }
  return n;
}

/* ------------------------------------------------------------------ */
/* exact below-surface length inside one bilinear cell                 */
/* ------------------------------------------------------------------ */

typedef struct { int i, j; double u, v, absg1; } or_cross;

/* Ray segment s in [s0, s1] inside cell (i,j) of surface h (node heights
 * [nx][ny]).  The surface is bilinear in the cell (R2):
 *   h(u,v) = a + b u + c v + e u v, u=(x-X_i)/ΔX_i, v=(y-Y_j)/ΔY_j,
 * and the ray is below it where g(τ) = h(x(τ),y(τ)) - z(τ) > 0 (Heaviside
 * layer map P:319-334, R17), a quadratic in τ = s - s0.  Returns the length of
 * {τ in [0, Δs] : g(τ) > 0}; appends crossings (sign changes of g) to xs. */
static double cell_below_length(const or_problem *p, const double *h, int i, int j,
                                const double *o, const double *d, double s0, double s1,
                                or_cross *xs, int *nxs, int cap, long *n_unresolved) {
  int ny = p->ny;
  double h00 = h[i * ny + j], h10 = h[(i + 1) * ny + j];
  double h01 = h[i * ny + j + 1], h11 = h[(i + 1) * ny + j + 1];
  double dX = p->X[i + 1] - p->X[i], dY = p->Y[j + 1] - p->Y[j];
  double a = h00, b = h10 - h00, c = h01 - h00, e = h00 - h10 - h01 + h11;
  double u0 = (o[0] + s0 * d[0] - p->X[i]) / dX;
  double v0 = (o[1] + s0 * d[1] - p->Y[j]) / dY;
  double z0 = o[2] + s0 * d[2];
  double al = d[0] / dX, be = d[1] / dY;
  double g0 = a + b * u0 + c * v0 + e * u0 * v0 - z0;
  double g1 = b * al + c * be + e * (u0 * be + v0 * al) - d[2];
  double g2 = e * al * be;
  double L = s1 - s0;
  /* instrumentation: the corner-bound test a fast tracer would use */
  {
    double hmin = fmin(fmin(h00, h10), fmin(h01, h11));
    double hmax = fmax(fmax(h00, h10), fmax(h01, h11));
    double za = z0, zb = o[2] + s1 * d[2];
    if (!(zb <= hmin || za >= hmax)) (*n_unresolved)++;
  }
  /* real roots of g0 + g1 τ + g2 τ² in (0, L) */
  double rt[2];
  int nr = 0;
  if (g2 == 0.0) {
    if (g1 != 0.0) { double t = -g0 / g1; if (t > 0 && t < L) rt[nr++] = t; }
  } else {
    double disc = g1 * g1 - 4.0 * g2 * g0;
    if (disc > 0.0) {
      double sq = sqrt(disc);
      double qq = -0.5 * (g1 + (g1 >= 0 ? sq : -sq));   /* stable form */
      double t1 = qq / g2, t2 = (qq != 0.0) ? g0 / qq : t1;
      if (t1 > t2) { double tmp = t1; t1 = t2; t2 = tmp; }
      if (t1 > 0 && t1 < L) rt[nr++] = t1;
      if (t2 > 0 && t2 < L && t2 != t1) rt[nr++] = t2;
    }
  }
  /* split [0, L] at the roots; sign of g at piece midpoints (R17) */
  double edges[4];
  int ne = 0;
  edges[ne++] = 0.0;
  for (int k = 0; k < nr; k++) edges[ne++] = rt[k];
  edges[ne++] = L;
  double below = 0.0;
  int prev_sign = 0;
  for (int k = 0; k + 1 < ne; k++) {
    double tm = 0.5 * (edges[k] + edges[k + 1]);
    double gm = g0 + g1 * tm + g2 * tm * tm;
    int sg = gm > 0 ? 1 : -1;
    if (sg > 0) below += edges[k + 1] - edges[k];
    if (k > 0 && sg != prev_sign && *nxs < cap) {
      double tc = edges[k];
      or_cross *x = &xs[(*nxs)++];
      x->i = i; x->j = j;
      x->u = u0 + al * tc;
      x->v = v0 + be * tc;
      x->absg1 = fabs(g1 + 2.0 * g2 * tc);
    }
    prev_sign = sg;
  }
  return below;
}

/* Per-ray result for one chain: B_l (length below surface l inside the box),
 * in-box length, exterior length, crossing records. */
#define OR_MAXX 512
typedef struct {
  double B[2], s_exit, L_ext;
  int nx[2];
  or_cross x[2][OR_MAXX];
  long n_inbox, n_band, n_unres, n_cross;
} or_ray_result;

static void trace_ray(const or_problem *p, long q, const double *H, or_ray_result *res,
                      int *ij, double *si, double *so, int cap) {
  const double *o = p->det + 3 * p->rdet[q], *d = p->dir + 3 * q;
  int N = p->nx * p->ny;
  or_ray_extent(p, q, &res->s_exit, &res->L_ext);
  int nc = or_traverse(p, q, ij, si, so, cap);
  if (nc > cap) nc = cap;
  double hmin = H[0], hmax = H[N];
  for (int k = 0; k < N; k++) { hmin = fmin(hmin, H[k]); hmax = fmax(hmax, H[N + k]); }
  res->n_inbox = nc; res->n_band = 0; res->n_unres = 0;
  for (int l = 0; l < 2; l++) {
    res->B[l] = 0.0;
    res->nx[l] = 0;
    for (int c = 0; c < nc; c++)
      res->B[l] += cell_below_length(p, H + l * N, ij[2 * c], ij[2 * c + 1], o, d, si[c], so[c],
                                     res->x[l], &res->nx[l], OR_MAXX, &res->n_unres);
  }
  for (int c = 0; c < nc; c++) {
    double za = o[2] + si[c] * d[2], zb = o[2] + so[c] * d[2];
    if (zb > hmin && za < hmax) res->n_band++;
  }
  res->n_cross = res->nx[0] + res->nx[1];
}

/* Opacity O = ∫ ρ du along the ray with the Heaviside unit map
 * (P:319-334): muck below H0, air between H0 and H1, rock above H1 up to z_top,
 * rho_e beyond a side exit (R7). */
static double opacity(const or_problem *p, const or_ray_result *r) {
  double Lm = r->B[0], La = r->B[1] - r->B[0], Lr = r->s_exit - r->B[1];
  return p->rho_m * Lm + p->rho_a * La + p->rho_r * Lr + p->rho_e * r->L_ext;
}

/* ------------------------------------------------------------------ */
/* public: traversal, path lengths, likelihood + gradient from heights */
/* ------------------------------------------------------------------ */

int or_traversal(const or_problem *p, long q, int *ij, double *s_in, double *s_out, int cap) {
  return or_traverse(p, q, ij, s_in, s_out, cap);
}

/* Every ray's traversal in one call (the same or_traverse per ray), CSR by ray:
 * with ij == NULL only off[R+1] is filled (cell counts, prefix-summed); then
 * ij[2 off[R]] and s_out[off[R]] receive the cells in ray order. */
void or_traversal_all(const or_problem *p, long *off, int *ij, double *s_out) {
  const int cap = 2 * (p->nx + p->ny) + 8;
  if (!ij) {
    off[0] = 0;
#pragma omp parallel
    {
      int *tij = (int *)malloc(sizeof(int) * 2 * cap);
      double *ts = (double *)malloc(sizeof(double) * 2 * cap);
#pragma omp for schedule(static)
      for (long q = 0; q < p->nray; q++) off[q + 1] = or_traverse(p, q, tij, ts, ts + cap, cap);
      free(tij);
      free(ts);
    }
    for (long q = 0; q < p->nray; q++) off[q + 1] += off[q];
    return;
  }
#pragma omp parallel
  {
    double *ts = (double *)malloc(sizeof(double) * cap);
#pragma omp for schedule(static)
    for (long q = 0; q < p->nray; q++) or_traverse(p, q, ij + 2 * off[q], ts, s_out + off[q], cap);
    free(ts);
  }
}

/* Per (chain, ray): L[3] = (muck, air, rock) in-box lengths, O, s_exit.
 * H: [C][2][nx][ny] double. */
void or_path_lengths(const or_problem *p, int C, const double *H, double *L, double *O,
                     double *crossings_min_absg1) {
  int N = p->nx * p->ny;
  long R = p->nray;
  int cap = 2 * (p->nx + p->ny) + 8;
#pragma omp parallel
  {
    int *ij = (int *)malloc(sizeof(int) * 2 * cap);
    double *si = (double *)malloc(sizeof(double) * cap), *so = (double *)malloc(sizeof(double) * cap);
    or_ray_result *res = (or_ray_result *)malloc(sizeof(or_ray_result));
#pragma omp for schedule(static)
    for (long pr = 0; pr < (long)C * R; pr++) {
      int c = (int)(pr / R);
      long q = pr % R;
      trace_ray(p, q, H + (long)c * 2 * N, res, ij, si, so, cap);
      L[3 * pr + 0] = res->B[0];
      L[3 * pr + 1] = res->B[1] - res->B[0];
      L[3 * pr + 2] = res->s_exit - res->B[1];
      O[pr] = opacity(p, res);
      if (crossings_min_absg1) {
        double m = INFINITY;
        for (int l = 0; l < 2; l++)
          for (int k = 0; k < res->nx[l]; k++) m = fmin(m, res->x[l][k].absg1);
        crossings_min_absg1[pr] = m;
      }
    }
    free(ij); free(si); free(so); free(res);
  }
}

/* Poisson log-likelihood with λ_p = w_p exp(-O_p/Λ) (R9)
 * and its gradient with respect to the node heights, per chain.
 *   ll_std = Σ_p [C ln λ - λ - ln Γ(C+1)]
 *   ll_dev = Σ_p [C (ln λ - ln C) - λ + C]     (C ln(.) = 0 when C = 0; R15)
 *   dldH[c][l][node] = Σ_p (λ_p - C_p)/Λ · ∂O/∂B_l · Σ_crossings φ_node/|g'|
 * with ∂O/∂B0 = ρ_m - ρ_a, ∂O/∂B1 = ρ_a - ρ_r and ∂B/∂h_node = φ_node/|g'| at
 * each crossing (a crossing moves by -δφ/g' when a node moves by δ).
 * H: [C][2][nx][ny].  Parallel over (chain, ray-chunk) with private gradient
 * buffers summed in chunk order (deterministic).
 * sens (optional) [C]: Σ over crossings of (∂ℓ/∂B)²·Σφ²/|g'|^4 — the oracle's
 * own estimate of gradient conditioning. */
#define OR_CHUNK 4096
void or_loglik_grad_H(const or_problem *p, int C, const double *H, double *ll_dev, double *ll_std,
                      double *dldH, double *sens, long *counters) {
  int N = p->nx * p->ny;
  long R = p->nray;
  long nch = (R + OR_CHUNK - 1) / OR_CHUNK;
  long ntask = (long)C * nch;
  double *part = (double *)calloc((size_t)ntask * (2 * N + 3), sizeof(double));
  long cnt_tot[4] = {0, 0, 0, 0};
  int cap = 2 * (p->nx + p->ny) + 8;
  double k0 = p->rho_m - p->rho_a, k1 = p->rho_a - p->rho_r;
#pragma omp parallel
  {
    int *ij = (int *)malloc(sizeof(int) * 2 * cap);
    double *si = (double *)malloc(sizeof(double) * cap), *so = (double *)malloc(sizeof(double) * cap);
    or_ray_result *res = (or_ray_result *)malloc(sizeof(or_ray_result));
    long lc[4] = {0, 0, 0, 0};
#pragma omp for schedule(dynamic, 1)
    for (long t = 0; t < ntask; t++) {
      int c = (int)(t / nch);
      long q0 = (t % nch) * OR_CHUNK, q1 = q0 + OR_CHUNK < R ? q0 + OR_CHUNK : R;
      const double *Hc = H + (long)c * 2 * N;
      double *g = part + t * (2 * N + 3);
      double sdev = 0, sstd = 0, ssens = 0;
      for (long q = q0; q < q1; q++) {
        trace_ray(p, q, Hc, res, ij, si, so, cap);
        lc[0] += res->n_inbox; lc[1] += res->n_band; lc[2] += res->n_unres; lc[3] += res->n_cross;
        double O = opacity(p, res);
        double lam = p->w[q] * exp(-O / p->Lambda);
        double Cq = p->cnt[q];
        sstd += Cq * log(lam) - lam - lgamma(Cq + 1.0);
        sdev += (Cq > 0 ? Cq * (log(lam) - log(Cq)) : 0.0) - lam + Cq;
        double dldO = (lam - Cq) / p->Lambda;
        for (int l = 0; l < 2; l++) {
          double f = dldO * (l == 0 ? k0 : k1);
          for (int k = 0; k < res->nx[l]; k++) {
            const or_cross *x = &res->x[l][k];
            double u = x->u, v = x->v, ig = 1.0 / x->absg1;
            double ph[4] = {(1 - u) * (1 - v), u * (1 - v), (1 - u) * v, u * v};
            int nd[4] = {x->i * p->ny + x->j, (x->i + 1) * p->ny + x->j, x->i * p->ny + x->j + 1,
                         (x->i + 1) * p->ny + x->j + 1};
            for (int m = 0; m < 4; m++) g[l * N + nd[m]] += f * ph[m] * ig;
            ssens += f * f * (ph[0] * ph[0] + ph[1] * ph[1] + ph[2] * ph[2] + ph[3] * ph[3]) * ig * ig * ig * ig;
          }
        }
      }
      g[2 * N] = sdev; g[2 * N + 1] = sstd; g[2 * N + 2] = ssens;
    }
#pragma omp critical
    for (int k = 0; k < 4; k++) cnt_tot[k] += lc[k];
    free(ij); free(si); free(so); free(res);
  }
  for (int c = 0; c < C; c++) {
    double *gc = dldH + (long)c * 2 * N;
    memset(gc, 0, sizeof(double) * 2 * N);
    double sd = 0, ss = 0, se = 0;
    for (long k = 0; k < nch; k++) {
      const double *g = part + ((long)c * nch + k) * (2 * N + 3);
      for (int m = 0; m < 2 * N; m++) gc[m] += g[m];
      sd += g[2 * N]; ss += g[2 * N + 1]; se += g[2 * N + 2];
    }
    ll_dev[c] = sd;
    if (ll_std) ll_std[c] = ss;
    if (sens) sens[c] = se;
  }
  if (counters) for (int k = 0; k < 4; k++) counters[k] = cnt_tot[k];
  free(part);
}

/* ------------------------------------------------------------------ */
/* log-posterior and gradient over the latent x            */
/* ------------------------------------------------------------------ */

/* logp[c] = ll_dev + Σ_l log N(x_l; 0, Q_l^-1); grad = ∂/∂x by the chain rule
 * through the heights map.  x: [C][2][nx][ny] double.  prior_out, ll_out,
 * sens (optional) [C]. */
void or_logpost_grad(const or_problem *p, int C, const double *x, double *logp, double *grad,
                     double *ll_out, double *ll_std_out, double *prior_out, double *sens,
                     long *counters) {
  int N = p->nx * p->ny;
  double *H = (double *)malloc(sizeof(double) * (size_t)C * 2 * N);
  double *dH = (double *)malloc(sizeof(double) * (size_t)C * 3 * N);
  double *G = (double *)malloc(sizeof(double) * (size_t)C * 2 * N);
  double *ll = (double *)malloc(sizeof(double) * C);
  for (int c = 0; c < C; c++) or_heights(p, x + (long)c * 2 * N, H + (long)c * 2 * N, dH + (long)c * 3 * N);
  or_loglik_grad_H(p, C, H, ll, ll_std_out, G, sens, counters);
  for (int c = 0; c < C; c++) {
    const double *xc = x + (long)c * 2 * N, *Gc = G + (long)c * 2 * N, *dHc = dH + (long)c * 3 * N;
    double *gc = grad + (long)c * 2 * N;
    double pr = 0.0;
    for (int l = 0; l < 2; l++) pr += or_prior_surface(p->nx, p->ny, p->r[l], xc + l * N, gc + l * N);
    for (int k = 0; k < N; k++) {
      gc[k] += Gc[k] * dHc[k] + Gc[N + k] * dHc[N + k];
      gc[N + k] += Gc[N + k] * dHc[2 * N + k];
    }
    logp[c] = ll[c] + pr;
    if (ll_out) ll_out[c] = ll[c];
    if (prior_out) prior_out[c] = pr;
  }
  free(H); free(dH); free(G); free(ll);
}

/* ------------------------------------------------------------------ */
/* Hierarchical r_l (readings R13b/R13c)    */
/* ------------------------------------------------------------------ */

/* The torus spectrum of Q(r) = 4I - rA and its r-derivatives: eigenvalues
 * λ_ab = 4 - r c_ab with c_ab = 2(cos 2πa/n_x + cos 2πb/n_y), so
 *   σ² = N⁻¹ Σ 1/λ,  dσ²/dr = N⁻¹ Σ c/λ²,  ln det Q = Σ ln λ,  d ln det Q/dr = -Σ c/λ. */
void or_torus_spectrum_dr(int nx, int ny, double r, double *sigma, double *dsigma, double *logdet,
                          double *dlogdet) {
  double s = 0.0, ds = 0.0, ld = 0.0, dld = 0.0;
  for (int a = 0; a < nx; a++)
    for (int b = 0; b < ny; b++) {
      double c = 2.0 * (cos(2.0 * OR_PI * a / nx) + cos(2.0 * OR_PI * b / ny));
      double lam = 4.0 - r * c;
      s += 1.0 / lam;
      ds += c / (lam * lam);
      ld += log(lam);
      dld -= c / lam;
    }
  double N = (double)nx * ny;
  *sigma = sqrt(s / N);
  *dsigma = (ds / N) / (2.0 * *sigma);
  *logdet = ld;
  *dlogdet = dld;
}

/* Log-posterior and gradient with the CAR dependence parameters sampled:
 * v [C][2N + 2] = (x_0, x_1, ρ_0, ρ_1) with r_l = 1/(1 + e^{-ρ_l}) (R13b: the
 * unconstrained coordinate of r_l ~ Unif(0,1), prior density of ρ_l
 * = r_l (1 - r_l) by the change of variables), x_l | r_l ~ N(0, Q(r_l)^-1)
 * (R13c: centred), heights ǔ = Φ(x/σ(r)):
 *   logp = ll + Σ_l [-½ x_lᵀQ(r_l)x_l + ½ ln det Q(r_l) - (N/2) ln 2π + ln r_l + ln(1 - r_l)].
 * ∂logp/∂ρ_l = r_l(1 - r_l) [½ x_lᵀ A x_l + ½ d ln det Q/dr + (∂ll/∂σ_l) dσ_l/dr] + 1 - 2 r_l,
 * with ∂t/∂σ = -t/σ for t = x/σ inside the clamp (R18), so ∂ǔ/∂σ = -t φ(t)/σ. */
void or_logpost_grad_r(const or_problem *p, int C, const double *v, double *logp, double *grad,
                       double *ll_out, double *prior_out) {
  int N = p->nx * p->ny, P = 2 * N + 2;
  double *H = (double *)malloc(sizeof(double) * (size_t)C * 2 * N);
  double *aux = (double *)malloc(sizeof(double) * (size_t)C * 5 * N);   /* dH/dx (3N), dH/dσ (2N) */
  double *G = (double *)malloc(sizeof(double) * (size_t)C * 2 * N);
  double *ll = (double *)malloc(sizeof(double) * C);
  double *rr = (double *)malloc(sizeof(double) * C * 2), *sg = (double *)malloc(sizeof(double) * C * 2);
  double *dsg = (double *)malloc(sizeof(double) * C * 2), *ld = (double *)malloc(sizeof(double) * C * 2);
  double *dld = (double *)malloc(sizeof(double) * C * 2);
  for (int c = 0; c < C; c++) {
    const double *vc = v + (long)c * P;
    for (int l = 0; l < 2; l++) {
      double r = 1.0 / (1.0 + exp(-vc[2 * N + l]));
      rr[2 * c + l] = r;
      or_torus_spectrum_dr(p->nx, p->ny, r, &sg[2 * c + l], &dsg[2 * c + l], &ld[2 * c + l], &dld[2 * c + l]);
    }
    double *Hc = H + (long)c * 2 * N, *dx = aux + (long)c * 5 * N, *ds = dx + 3 * N;
    for (int k = 0; k < N; k++) {
      double t[2], u[2], dudx[2], duds[2];
      for (int l = 0; l < 2; l++) {
        double s = sg[2 * c + l];
        double tt = vc[l * N + k] / s;
        int clamped = 0;
        if (tt > OR_TCLAMP) { tt = OR_TCLAMP; clamped = 1; }
        if (tt < -OR_TCLAMP) { tt = -OR_TCLAMP; clamped = 1; }
        t[l] = tt;
        u[l] = 0.5 * erfc(-tt / sqrt(2.0));
        double phi = clamped ? 0.0 : exp(-0.5 * tt * tt) / sqrt(2.0 * OR_PI);
        dudx[l] = phi / s;
        duds[l] = -tt * phi / s;
      }
      double H0 = u[0] * p->z_top, H1 = (1.0 - u[1]) * H0 + u[1] * p->z_top;
      Hc[k] = H0;
      Hc[N + k] = H1;
      dx[k] = p->z_top * dudx[0];
      dx[N + k] = (1.0 - u[1]) * p->z_top * dudx[0];
      dx[2 * N + k] = (p->z_top - H0) * dudx[1];
      ds[k] = p->z_top * duds[0];                         /* ∂H0/∂σ0 (∂H1/∂σ0 = (1-ǔ1)·this) */
      ds[N + k] = (p->z_top - H0) * duds[1];              /* ∂H1/∂σ1 */
      (void)t;
    }
  }
  or_loglik_grad_H(p, C, H, ll, NULL, G, NULL, NULL);
  for (int c = 0; c < C; c++) {
    const double *vc = v + (long)c * P, *Gc = G + (long)c * 2 * N;
    const double *dx = aux + (long)c * 5 * N, *ds = dx + 3 * N, *Hc = H + (long)c * 2 * N;
    double *gc = grad + (long)c * P;
    double pr = 0.0;
    double dll_ds[2] = {0.0, 0.0};
    for (int k = 0; k < N; k++) {
      double u1 = (Hc[N + k] - Hc[k]) / (p->z_top - Hc[k]);   /* ǔ1 from H0, H1 */
      dll_ds[0] += Gc[k] * ds[k] + Gc[N + k] * (1.0 - u1) * ds[k];
      dll_ds[1] += Gc[N + k] * ds[N + k];
    }
    for (int l = 0; l < 2; l++) {
      double r = rr[2 * c + l];
      const double *x = vc + l * N;
      double quad = 0.0, xAx = 0.0;
      for (int i = 0; i < p->nx; i++)
        for (int j = 0; j < p->ny; j++) {
          int ip = (i + 1) % p->nx, im = (i - 1 + p->nx) % p->nx, jp = (j + 1) % p->ny, jm = (j - 1 + p->ny) % p->ny;
          double nb = x[ip * p->ny + j] + x[im * p->ny + j] + x[i * p->ny + jp] + x[i * p->ny + jm];
          double Qx = 4.0 * x[i * p->ny + j] - r * nb;
          quad += x[i * p->ny + j] * Qx;
          xAx += x[i * p->ny + j] * nb;
          gc[l * N + i * p->ny + j] = -Qx;
        }
      pr += -0.5 * quad + 0.5 * ld[2 * c + l] - 0.5 * N * log(2.0 * OR_PI) + log(r) + log(1.0 - r);
      gc[2 * N + l] = r * (1.0 - r) * (0.5 * xAx + 0.5 * dld[2 * c + l] + dll_ds[l] * dsg[2 * c + l])
                      + 1.0 - 2.0 * r;
    }
    for (int k = 0; k < N; k++) {
      gc[k] += Gc[k] * dx[k] + Gc[N + k] * dx[N + k];
      gc[N + k] += Gc[N + k] * dx[2 * N + k];
    }
    logp[c] = ll[c] + pr;
    if (ll_out) ll_out[c] = ll[c];
    if (prior_out) prior_out[c] = pr;
  }
  free(H); free(aux); free(G); free(ll); free(rr); free(sg); free(dsg); free(ld); free(dld);
}

/* ------------------------------------------------------------------ */
/* Non-centred CAR parameterisation x = U z (*/
/* reading R13d in DESIGN.md)                                          */
/* ------------------------------------------------------------------ */

/* The square root U = Q(r)^{-1/2} of the torus CAR covariance: Q is circulant,
 * Q = F* diag(λ) F with λ_ab = 4 - r c_ab, c_ab = 2(cos 2πa/n_x + cos 2πb/n_y), so
 * U is the circulant with kernel k[d] = N^{-1} Σ_ab λ_ab^{-1/2} cos 2π(a d_i/n_x + b d_j/n_y)
 * (x_i = Σ_j k[i - j] z_j; UUᵀ = U² = Q^{-1} = Σ, as P:576-582 require), and
 * dk/dr the kernel of dU/dr (eigenvalues ½ c λ^{-3/2}).  Direct sums. */
void or_ncp_kernel(int nx, int ny, double r, double *k, double *dk) {
  int N = nx * ny;
  for (int di = 0; di < nx; di++)
    for (int dj = 0; dj < ny; dj++) {
      double s = 0.0, ds = 0.0;
      for (int a = 0; a < nx; a++)
        for (int b = 0; b < ny; b++) {
          double c = 2.0 * (cos(2.0 * OR_PI * a / nx) + cos(2.0 * OR_PI * b / ny));
          double lam = 4.0 - r * c;
          double ph = cos(2.0 * OR_PI * ((double)a * di / nx + (double)b * dj / ny));
          s += ph / sqrt(lam);
          ds += ph * 0.5 * c / (lam * sqrt(lam));
        }
      k[di * ny + dj] = s / N;
      if (dk) dk[di * ny + dj] = ds / N;
    }
}

/* y = (circulant with kernel k) v on the torus: y_i = Σ_j k[i - j] v_j. */
static void circ_apply(int nx, int ny, const double *k, const double *v, double *y) {
  for (int i = 0; i < nx; i++)
    for (int j = 0; j < ny; j++) {
      double s = 0.0;
      for (int i2 = 0; i2 < nx; i2++)
        for (int j2 = 0; j2 < ny; j2++) {
          int di = (i - i2 + nx) % nx, dj = (j - j2 + ny) % ny;
          s += k[di * ny + dj] * v[i2 * ny + j2];
        }
      y[i * ny + j] = s;
    }
}

/* Log-posterior and gradient in the non-centred parameters v [C][2N + 2] =
 * (z_0, z_1, ρ_0, ρ_1): z_l ~ N(0, I), r_l = logistic(ρ_l) with r_l ~ Unif(0,1)
 * (R13b), x_l = U(r_l) z_l, heights ǔ = Φ(x/σ(r)):
 *   logp = ll(H(x)) - ½ Σ_l |z_l|² - N ln 2π + Σ_l [ln r_l + ln(1 - r_l)],
 *   ∂/∂z_l = -z_l + U ∂ll/∂x_l   (U symmetric),
 *   ∂/∂ρ_l = r(1-r) [(∂ll/∂x_l)ᵀ (dU/dr) z_l + (∂ll/∂σ_l) dσ_l/dr] + 1 - 2r,
 * with ∂ll/∂x the likelihood part only (the prior is the standard normal on z). */
void or_logpost_grad_ncp(const or_problem *p, int C, const double *v, double *logp, double *grad,
                         double *ll_out) {
  int N = p->nx * p->ny, P = 2 * N + 2;
  double *H = (double *)malloc(sizeof(double) * (size_t)C * 2 * N);
  double *aux = (double *)malloc(sizeof(double) * (size_t)C * 5 * N);   /* dH/dx (3N), dH/dσ (2N) */
  double *X = (double *)malloc(sizeof(double) * (size_t)C * 2 * N);
  double *G = (double *)malloc(sizeof(double) * (size_t)C * 2 * N);
  double *ll = (double *)malloc(sizeof(double) * C);
  double *kk = (double *)malloc(sizeof(double) * (size_t)C * 4 * N);    /* k, dk per surface */
  double *rr = (double *)malloc(sizeof(double) * C * 2), *dsg = (double *)malloc(sizeof(double) * C * 2);
  for (int c = 0; c < C; c++) {
    const double *vc = v + (long)c * P;
    double sg[2];
    for (int l = 0; l < 2; l++) {
      double r = 1.0 / (1.0 + exp(-vc[2 * N + l])), ld, dld;
      rr[2 * c + l] = r;
      or_torus_spectrum_dr(p->nx, p->ny, r, &sg[l], &dsg[2 * c + l], &ld, &dld);
      double *k = kk + (long)c * 4 * N + 2 * l * N;
      or_ncp_kernel(p->nx, p->ny, r, k, k + N);
      circ_apply(p->nx, p->ny, k, vc + l * N, X + (long)c * 2 * N + l * N);
    }
    const double *xc = X + (long)c * 2 * N;
    double *Hc = H + (long)c * 2 * N, *dx = aux + (long)c * 5 * N, *ds = dx + 3 * N;
    for (int q = 0; q < N; q++) {
      double u[2], dudx[2], duds[2];
      for (int l = 0; l < 2; l++) {
        double tt = xc[l * N + q] / sg[l];
        int clamped = 0;
        if (tt > OR_TCLAMP) { tt = OR_TCLAMP; clamped = 1; }
        if (tt < -OR_TCLAMP) { tt = -OR_TCLAMP; clamped = 1; }
        u[l] = 0.5 * erfc(-tt / sqrt(2.0));
        double phi = clamped ? 0.0 : exp(-0.5 * tt * tt) / sqrt(2.0 * OR_PI);
        dudx[l] = phi / sg[l];
        duds[l] = -tt * phi / sg[l];
      }
      double H0 = u[0] * p->z_top, H1 = (1.0 - u[1]) * H0 + u[1] * p->z_top;
      Hc[q] = H0;
      Hc[N + q] = H1;
      dx[q] = p->z_top * dudx[0];
      dx[N + q] = (1.0 - u[1]) * p->z_top * dudx[0];
      dx[2 * N + q] = (p->z_top - H0) * dudx[1];
      ds[q] = p->z_top * duds[0];
      ds[N + q] = (p->z_top - H0) * duds[1];
    }
  }
  or_loglik_grad_H(p, C, H, ll, NULL, G, NULL, NULL);
  double *gx = (double *)malloc(sizeof(double) * 2 * N), *tmp = (double *)malloc(sizeof(double) * N);
  for (int c = 0; c < C; c++) {
    const double *vc = v + (long)c * P, *Gc = G + (long)c * 2 * N, *Hc = H + (long)c * 2 * N;
    const double *dx = aux + (long)c * 5 * N, *ds = dx + 3 * N;
    double *gc = grad + (long)c * P;
    double dll_ds[2] = {0.0, 0.0}, zz = 0.0;
    for (int q = 0; q < N; q++) {
      gx[q] = Gc[q] * dx[q] + Gc[N + q] * dx[N + q];
      gx[N + q] = Gc[N + q] * dx[2 * N + q];
      double u1 = (Hc[N + q] - Hc[q]) / (p->z_top - Hc[q]);
      dll_ds[0] += Gc[q] * ds[q] + Gc[N + q] * (1.0 - u1) * ds[q];
      dll_ds[1] += Gc[N + q] * ds[N + q];
    }
    double lp = ll[c];
    for (int l = 0; l < 2; l++) {
      const double *k = kk + (long)c * 4 * N + 2 * l * N, *dk = k + N, *z = vc + l * N;
      circ_apply(p->nx, p->ny, k, gx + l * N, tmp);                  /* U ∂ll/∂x */
      for (int q = 0; q < N; q++) { gc[l * N + q] = -z[q] + tmp[q]; zz += z[q] * z[q]; }
      circ_apply(p->nx, p->ny, dk, z, tmp);                          /* (dU/dr) z */
      double s = 0.0;
      for (int q = 0; q < N; q++) s += gx[l * N + q] * tmp[q];
      double r = rr[2 * c + l];
      gc[2 * N + l] = r * (1.0 - r) * (s + dll_ds[l] * dsg[2 * c + l]) + 1.0 - 2.0 * r;
      lp += log(r) + log(1.0 - r);
    }
    lp += -0.5 * zz - N * log(2.0 * OR_PI);
    logp[c] = lp;
    if (ll_out) ll_out[c] = ll[c];
  }
  free(gx); free(tmp);
  free(H); free(aux); free(X); free(G); free(ll); free(kk); free(rr); free(dsg);
}

/* ------------------------------------------------------------------ */
/* The paper's voxel / sigmoid / linearised forward model (P:242-390,  */
/* SURVEY §8(f) f3; reading R28 in DESIGN.md)                          */
/* ------------------------------------------------------------------ */

/* Voxel grid (R28): column (i,j) belongs to layer-grid node (i,j) (the map
 * (i,j) -> (x(i),y(j)) of P:248-250 is the identity) and spans
 * [e_i, e_{i+1}] x [f_j, f_{j+1}] with e_0 = X_0, e_i = (X_{i-1}+X_i)/2,
 * e_nx = X_{nx-1} (likewise f for y); layer k spans [kΔz, (k+1)Δz) with
 * Δz = z_top/nz.  Linear index v = (i*ny + j)*nz + k, the right-most index
 * fastest. */
static double col_edge(const double *X, int n, int i) {
  if (i <= 0) return X[0];
  if (i >= n) return X[n - 1];
  return 0.5 * (X[i - 1] + X[i]);
}

static int cmp_double(const void *a, const void *b) {
  double x = *(const double *)a, y = *(const double *)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* Voxels met by the in-box segment [0, s_exit] of ray q and the length in each
 * (the L_pv of the piecewise-constant restriction λ_p(R)): every
 * x-edge, y-edge and z-plane crossing in (0, s_exit) is a breakpoint; after
 * sorting, each piece of positive length lies in one voxel, found from its
 * midpoint.  Returns the number of pieces (writes at most cap). */
int or_voxel_path(const or_problem *p, int nz, long q, int *vox, double *len, int cap) {
  const double *o = p->det + 3 * p->rdet[q], *d = p->dir + 3 * q;
  double s_exit, L_ext;
  or_ray_extent(p, q, &s_exit, &L_ext);
  int nb_max = (p->nx + 1) + (p->ny + 1) + (nz + 1) + 2;
  double *bp = (double *)malloc(sizeof(double) * nb_max);
  int nb = 0;
  bp[nb++] = 0.0;
  bp[nb++] = s_exit;
  for (int i = 0; i <= p->nx; i++)
    if (d[0] != 0.0) {
      double s = (col_edge(p->X, p->nx, i) - o[0]) / d[0];
      if (s > 0.0 && s < s_exit) bp[nb++] = s;
    }
  for (int j = 0; j <= p->ny; j++)
    if (d[1] != 0.0) {
      double s = (col_edge(p->Y, p->ny, j) - o[1]) / d[1];
      if (s > 0.0 && s < s_exit) bp[nb++] = s;
    }
  double dz = p->z_top / nz;
  for (int k = 1; k <= nz; k++) {
    double s = (k * dz - o[2]) / d[2];
    if (s > 0.0 && s < s_exit) bp[nb++] = s;
  }
  qsort(bp, nb, sizeof(double), cmp_double);
  int n = 0;
  for (int m = 0; m + 1 < nb; m++) {
    double l = bp[m + 1] - bp[m];
    if (!(l > 0.0)) continue;
    double sm = 0.5 * (bp[m] + bp[m + 1]);
    double xm = o[0] + sm * d[0], ym = o[1] + sm * d[1], zm = o[2] + sm * d[2];
    int i = 0, j = 0;
    while (i < p->nx - 1 && xm >= col_edge(p->X, p->nx, i + 1)) i++;
    while (j < p->ny - 1 && ym >= col_edge(p->Y, p->ny, j + 1)) j++;
    int k = (int)floor(zm / dz);
    if (k < 0) k = 0;
    if (k > nz - 1) k = nz - 1;
    if (n < cap) { vox[n] = (i * p->ny + j) * nz + k; len[n] = l; }
    n++;
  }
  free(bp);
  return n;
}

/* Smooth layer indicators D^(l) with ς_γ(u) = 1/(1+e^{-u/γ})
 * (P:349-352), three units muck / air / rock (H_{-1} = 0, H_0 muck top,
 * H_1 cave back, H_2 = z_top; R27/R28), partition-of-unity weights
 * W^(l) = D^(l)/Σ_l' D^(l') and R̂ = Σ_l W^(l) R^(l) with
 * R^(l) = (ρ_m, ρ_a, ρ_r).  H: [2][nx][ny]; W [3][n_grid]
 * (optional), Rhat [n_grid]. */
static double sigm(double u, double gamma) { return 1.0 / (1.0 + exp(-u / gamma)); }

void or_voxel_rhat(const or_problem *p, int nz, double gamma, const double *H, double *W, double *Rhat) {
  int N = p->nx * p->ny;
  double dz = p->z_top / nz, rho[3] = {p->rho_m, p->rho_a, p->rho_r};
  for (int node = 0; node < N; node++)
    for (int k = 0; k < nz; k++) {
      double z = k * dz;
      double b[4] = {0.0, H[node], H[N + node], p->z_top};
      double D[3], S = 0.0;
      for (int l = 0; l < 3; l++) { D[l] = sigm(b[l + 1] - z, gamma) - sigm(b[l] - z, gamma); S += D[l]; }
      long v = (long)node * nz + k;
      double R = 0.0;
      for (int l = 0; l < 3; l++) {
        double w = D[l] / S;
        if (W) W[(long)l * N * nz + v] = w;
        R += w * rho[l];
      }
      Rhat[v] = R;
    }
}

/* λ_p(R) = w_p exp(-(Σ_v L_pv R_v + ρ_e L_ext)/Λ) for every ray: the restriction
 * of eq:expected_counts to piecewise-constant fields, the rock
 * beyond a side exit as in the exact model (R7). */
void or_voxel_lambda(const or_problem *p, int nz, const double *R, double *lam) {
  int cap = (p->nx + p->ny + nz) + 8;
#pragma omp parallel
  {
    int *vox = (int *)malloc(sizeof(int) * cap);
    double *len = (double *)malloc(sizeof(double) * cap);
#pragma omp for schedule(dynamic, 256)
    for (long q = 0; q < p->nray; q++) {
      int n = or_voxel_path(p, nz, q, vox, len, cap);
      double s_exit, L_ext, O = 0.0;
      or_ray_extent(p, q, &s_exit, &L_ext);
      for (int m = 0; m < n; m++) O += len[m] * R[vox[m]];
      O += p->rho_e * L_ext;
      lam[q] = p->w[q] * exp(-O / p->Lambda);
    }
    free(vox); free(len);
  }
}

/* Row p of the sensitivity matrix G = ∂λ/∂R at R0:
 * G_pv = -λ_p(R0) L_pv / Λ for the voxels on the ray (0 elsewhere).
 * Writes the voxel ids / values of the row and returns their number; lam0_out
 * receives λ_p(R0). */
int or_voxel_G_row(const or_problem *p, int nz, const double *R0, long q, int *vox, double *G, int cap,
                   double *lam0_out) {
  int n = or_voxel_path(p, nz, q, vox, G, cap);
  if (n > cap) n = cap;
  double s_exit, L_ext, O = 0.0;
  or_ray_extent(p, q, &s_exit, &L_ext);
  for (int m = 0; m < n; m++) O += G[m] * R0[vox[m]];
  O += p->rho_e * L_ext;
  double lam0 = p->w[q] * exp(-O / p->Lambda);
  for (int m = 0; m < n; m++) G[m] = -lam0 * G[m] / p->Lambda;
  if (lam0_out) *lam0_out = lam0;
  return n;
}

/* Log-posterior and gradient under the linearised smooth model
 * λ̂(R̂(H)) = λ(R0) + G(R̂(H) - R0) with
 * R0 = R̂(H_ref) for a reference geometry H_ref [2][nx][ny] (R28), the Poisson
 * deviance likelihood of the exact model (R15) and the floor
 * λ̂ <- max(λ̂, τ λ_p(R0)) with zero derivative below it (R29):
 *   ℓ = Σ_p C(ln λ̂ - ln C) - λ̂ + C,   ∂ℓ/∂λ̂_p = C/λ̂ - 1,
 *   ∂ℓ/∂R̂_v = Σ_p G_pv ∂ℓ/∂λ̂_p,
 *   ∂R̂_v/∂H_0 = ς'(H_0 - z_k)(ρ_m - ρ_a)/S_k,  ∂R̂_v/∂H_1 = ς'(H_1 - z_k)(ρ_a - ρ_r)/S_k,
 * S_k = Σ_l D^(l) = ς(z_top - z_k) - ς(-z_k) (the indicators telescope), then the
 * heights chain rule and the CAR prior exactly as or_logpost_grad.
 * x: [C][2N]; outputs as or_logpost_grad. */
void or_voxel_logpost_grad(const or_problem *p, int nz, double gamma, double tau, const double *Href, int C,
                           const double *x, double *logp, double *grad, double *ll_out, double *prior_out) {
  int N = p->nx * p->ny;
  long ng = (long)N * nz;
  long R = p->nray;
  int cap = (p->nx + p->ny + nz) + 8;
  double dz = p->z_top / nz;
  double *R0 = (double *)malloc(sizeof(double) * ng);
  or_voxel_rhat(p, nz, gamma, Href, NULL, R0);
  /* G rows at R0, once */
  long *row = (long *)malloc(sizeof(long) * (R + 1));
  double *lam0 = (double *)malloc(sizeof(double) * R);
  row[0] = 0;
  {
    int *vox = (int *)malloc(sizeof(int) * cap);
    double *len = (double *)malloc(sizeof(double) * cap);
    for (long q = 0; q < R; q++) {
      int n = or_voxel_path(p, nz, q, vox, len, cap);
      row[q + 1] = row[q] + (n < cap ? n : cap);
    }
    free(vox); free(len);
  }
  int *gv = (int *)malloc(sizeof(int) * (row[R] > 0 ? row[R] : 1));
  double *gx = (double *)malloc(sizeof(double) * (row[R] > 0 ? row[R] : 1));
#pragma omp parallel for schedule(dynamic, 256)
  for (long q = 0; q < R; q++) or_voxel_G_row(p, nz, R0, q, gv + row[q], gx + row[q], cap, &lam0[q]);
#pragma omp parallel
  {
    double *H = (double *)malloc(sizeof(double) * 2 * N), *dH = (double *)malloc(sizeof(double) * 3 * N);
    double *Rh = (double *)malloc(sizeof(double) * ng), *gR = (double *)malloc(sizeof(double) * ng);
    double *GH = (double *)malloc(sizeof(double) * 2 * N);
#pragma omp for schedule(dynamic, 1)
    for (int c = 0; c < C; c++) {
      const double *xc = x + (long)c * 2 * N;
      or_heights(p, xc, H, dH);
      or_voxel_rhat(p, nz, gamma, H, NULL, Rh);
      memset(gR, 0, sizeof(double) * ng);
      double ll = 0.0;
      for (long q = 0; q < R; q++) {
        double lam = lam0[q];
        for (long m = row[q]; m < row[q + 1]; m++) lam += gx[m] * (Rh[gv[m]] - R0[gv[m]]);
        double dl = 0.0;
        if (lam < tau * lam0[q]) lam = tau * lam0[q];
        else dl = p->cnt[q] / lam - 1.0;
        double Cq = p->cnt[q];
        ll += (Cq > 0 ? Cq * (log(lam) - log(Cq)) : 0.0) - lam + Cq;
        for (long m = row[q]; m < row[q + 1]; m++) gR[gv[m]] += gx[m] * dl;
      }
      for (int node = 0; node < N; node++) {
        double g0 = 0.0, g1 = 0.0;
        for (int k = 0; k < nz; k++) {
          double z = k * dz, S = sigm(p->z_top - z, gamma) - sigm(-z, gamma);
          double s0 = sigm(H[node] - z, gamma), s1 = sigm(H[N + node] - z, gamma);
          double gv_ = gR[(long)node * nz + k];
          g0 += gv_ * s0 * (1.0 - s0) / gamma * (p->rho_m - p->rho_a) / S;
          g1 += gv_ * s1 * (1.0 - s1) / gamma * (p->rho_a - p->rho_r) / S;
        }
        GH[node] = g0;
        GH[N + node] = g1;
      }
      double *gc = grad + (long)c * 2 * N;
      double pr = 0.0;
      for (int l = 0; l < 2; l++) pr += or_prior_surface(p->nx, p->ny, p->r[l], xc + l * N, gc + l * N);
      for (int k = 0; k < N; k++) {
        gc[k] += GH[k] * dH[k] + GH[N + k] * dH[N + k];
        gc[N + k] += GH[N + k] * dH[2 * N + k];
      }
      logp[c] = ll + pr;
      if (ll_out) ll_out[c] = ll;
      if (prior_out) prior_out[c] = pr;
    }
    free(H); free(dH); free(Rh); free(gR); free(GH);
  }
  free(R0); free(row); free(lam0); free(gv); free(gx);
}

/* ------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al., SC'11) and momenta (R22, reading c.1.12) */
/* ------------------------------------------------------------------ */
void or_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; r++) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* p ~ N(0, I) for chain `chain` (global id) at iteration `iter`: counter
 * (q, chain, iter mod 2^32, stream 0), key (seed lo, seed hi); uniforms
 * u = (k + 1/2) 2^-32; Box-Muller on word pairs (0,1) and (2,3). */
void or_momenta(int P, uint64_t seed, uint64_t iter, uint64_t chain, double *pout) {
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  for (int q = 0; 4 * q < P; q++) {
    uint32_t ctr[4] = {(uint32_t)q, (uint32_t)chain, (uint32_t)iter, 0u}, w[4];
    or_philox4x32_10(ctr, key, w);
    double u[4];
    for (int k = 0; k < 4; k++) u[k] = ((double)w[k] + 0.5) * 2.3283064365386963e-10;
    for (int h = 0; h < 2; h++) {
      double rad = sqrt(-2.0 * log(u[2 * h])), ang = 2.0 * OR_PI * u[2 * h + 1];
      if (4 * q + 2 * h < P) pout[4 * q + 2 * h] = rad * cos(ang);
      if (4 * q + 2 * h + 1 < P) pout[4 * q + 2 * h + 1] = rad * sin(ang);
    }
  }
}

/* MH uniform for chain/iter: counter (0, chain, iter, 1), word 0. */
double or_mh_uniform(uint64_t seed, uint64_t iter, uint64_t chain) {
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t ctr[4] = {0u, (uint32_t)chain, (uint32_t)iter, 1u}, w[4];
  or_philox4x32_10(ctr, key, w);
  return ((double)w[0] + 0.5) * 2.3283064365386963e-10;
}

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
