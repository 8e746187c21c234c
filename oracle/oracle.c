/*
 * ORACLE — test infrastructure only.
 *
 * A plain, slow, obviously-correct fp64 CPU implementation of what the EXACT
 * hot path computes (arXiv 2503.19925, PAPER.md).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library.  It shares no code, header, table or constant with
 * the CUDA path (paper_2503_19925_b200/csrc) and never imports it.
 *
 * Every function cites the passage it follows.  Loops run in the order the
 * definition is written (rows i ascending, columns k ascending, bins j
 * ascending); the only parallelism is OpenMP over fixed 4096-row chunks whose
 * partial sums are combined in chunk order, so results do not depend on the
 * thread count.
 *
 * Pins: see tests/test_oracle_pins.py (P1..P13 of SURVEY.md §8(c)).  Parity
 * of the ℓ(x) value is pinned only through finite differences (reading R2).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_CHUNK 4096

enum { OR_SET_NONE = 0, OR_SET_BALL = 1, OR_SET_NONNEG = 2, OR_SET_NONNEG_BALL = 3,
       OR_SET_TV_NONNEG = 4, OR_SET_TV = 5 };

typedef struct {
  int64_t n, d;             /* rows held here, columns                        */
  int64_t n_norm;           /* the n of the 1/n in Eq.(operator)              */
  int csr;                  /* 0: dense row-major A, 1: CSR (row_ptr,col,val)  */
  const void *A;            /* dense values, float or double, row pitch lda    */
  int a_f32;                /* 1: values (A or val) are float, 0: double       */
  int64_t lda;
  const int64_t *row_ptr;   /* CSR [n+1]                                      */
  const int32_t *col;       /* CSR [nnz]                                      */
  const void *val;          /* CSR [nnz]                                      */
  const double *y;          /* [n] counts / measurements                      */
  int W;
  const double *s, *mu;     /* [W] spectrum, Eq.(model)       */
  double I_bar;
  const double *s_row;      /* optional [n*W] per-row spectrum (A.1)          */
  const double *I_row;      /* optional [n] per-row intensity (A.1)           */
  int relu;                 /* 1: h uses t_+ (Eq. function-h-plus)            */
  int set;                  /* constraint set X                               */
  double R;                 /* radius of the ball part of X                   */
  const double *center;     /* [d] or NULL (= 0)                              */
  /* TV sets (NEXT-2): s x s image, d = s*s; see oracle_project_tv* below   */
  int tv_side;
  double tv_tau, tv_tol, tv_rtol, tv_dtol;
  int tv_max_it, tv_max_outer;
  int tv_k;                 /* λ evaluations per search round (reading R22); <= 1: binary */
  int tv_warm;              /* 1: warm-started proxes within a projection (reading R23) */
} oracle_problem;

void oracle_set_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
#else
  (void)t;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* h(t) = Σ_j s_j exp(-μ_j t_+)  — Eq.(function-h-plus).
 * relu = 0 drops the (.)_+ (Eq. eq:model-orig). */
double oracle_h(int W, const double *s, const double *mu, double t, int relu) {
  double tc = (relu && t < 0.0) ? 0.0 : t;
  double h = 0.0;
  for (int j = 0; j < W; ++j) h += s[j] * exp(-mu[j] * tc);
  return h;
}

/* |h'(t)| = Σ_j s_j μ_j exp(-μ_j t) for t > 0 — PAPER.md:1490 (§4.2 proof of
 * Theorem 2).  Returns NaN for t <= 0. */
double oracle_hprime_abs(int W, const double *s, const double *mu, double t) {
  if (!(t > 0.0)) return NAN;
  double v = 0.0;
  for (int j = 0; j < W; ++j) v += s[j] * mu[j] * exp(-mu[j] * t);
  return v;
}

/* H(t) = ∫_0^t h(u) du, the primitive whose derivative is h (reading R2 of
 * ℓ(x) = (1/n) Σ_i [y_i z_i - Ī H(z_i)] has gradient F(x)).
 *   t >= 0 (or relu = 0):  Σ_j (s_j/μ_j) (1 - exp(-μ_j t))
 *   t <  0 and relu = 1:   t Σ_j s_j           (h ≡ Σ s_j on t < 0)        */
double oracle_H(int W, const double *s, const double *mu, double t, int relu) {
  double v = 0.0;
  if (relu && t < 0.0) {
    for (int j = 0; j < W; ++j) v += s[j];
    return t * v;
  }
  for (int j = 0; j < W; ++j) v += (s[j] / mu[j]) * (1.0 - exp(-mu[j] * t));
  return v;
}

static double a_at(const oracle_problem *p, int64_t i, int64_t k) {
  if (p->a_f32) return (double)((const float *)p->A)[i * p->lda + k];
  return ((const double *)p->A)[i * p->lda + k];
}

static double v_at(const oracle_problem *p, int64_t e) {
  if (p->a_f32) return (double)((const float *)p->val)[e];
  return ((const double *)p->val)[e];
}

/* z_i = <a_i, x>, k ascending (dense) or in stored order (CSR). */
static double row_dot(const oracle_problem *p, int64_t i, const double *x) {
  double z = 0.0;
  if (!p->csr) {
    for (int64_t k = 0; k < p->d; ++k) z += a_at(p, i, k) * x[k];
  } else {
    for (int64_t e = p->row_ptr[i]; e < p->row_ptr[i + 1]; ++e) z += v_at(p, e) * x[p->col[e]];
  }
  return z;
}

static const double *row_s(const oracle_problem *p, int64_t i) {
  return p->s_row ? p->s_row + i * p->W : p->s;
}
static double row_I(const oracle_problem *p, int64_t i) {
  return p->I_row ? p->I_row[i] : p->I_bar;
}

/* z_i = <a_i, x> for every row (forward projection A x). */
void oracle_forward(const oracle_problem *p, const double *x, double *z) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < p->n; ++i) z[i] = row_dot(p, i, x);
}

/* Expected counts E[y_i | a_i] = Ī_i h_i(<a_i, x>) — Eq.(model),
 * PAPER.md:867-869 (per-row Ī', s' of Appendix A.1 when given). */
void oracle_mean(const oracle_problem *p, const double *x, double *lam) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < p->n; ++i)
    lam[i] = row_I(p, i) * oracle_h(p->W, row_s(p, i), p->mu, row_dot(p, i, x), p->relu);
}

/* F(x) = (1/n) Σ_i [y_i - Ī h(<a_i,x>)] a_i — Eq.(operator), PAPER.md:893-896,
 * with n = p->n_norm (reading R4), and the scalar
 * ℓ(x) = (1/n) Σ_i [y_i z_i - Ī H(z_i)] (reading R2).  g or loss may be NULL. */
void oracle_F(const oracle_problem *p, const double *x, double *g, double *loss) {
  const int64_t n = p->n, d = p->d;
  const int64_t nch = (n + ORACLE_CHUNK - 1) / ORACLE_CHUNK;
  double *part = (double *)calloc((size_t)(nch > 0 ? nch : 1) * (size_t)d, sizeof(double));
  double *lpart = (double *)calloc((size_t)(nch > 0 ? nch : 1), sizeof(double));
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < nch; ++c) {
    double *gc = part + c * d;
    const int64_t i1 = (c + 1) * ORACLE_CHUNK < n ? (c + 1) * ORACLE_CHUNK : n;
    for (int64_t i = c * ORACLE_CHUNK; i < i1; ++i) {
      const double z = row_dot(p, i, x);
      const double *si = row_s(p, i);
      const double Ii = row_I(p, i);
      const double r = p->y[i] - Ii * oracle_h(p->W, si, p->mu, z, p->relu);
      lpart[c] += p->y[i] * z - Ii * oracle_H(p->W, si, p->mu, z, p->relu);
      if (!p->csr) {
        for (int64_t k = 0; k < d; ++k) gc[k] += r * a_at(p, i, k);
      } else {
        for (int64_t e = p->row_ptr[i]; e < p->row_ptr[i + 1]; ++e) gc[p->col[e]] += r * v_at(p, e);
      }
    }
  }
  if (g) {
    for (int64_t k = 0; k < d; ++k) g[k] = 0.0;
    for (int64_t c = 0; c < nch; ++c)
      for (int64_t k = 0; k < d; ++k) g[k] += part[c * d + k];
    for (int64_t k = 0; k < d; ++k) g[k] /= (double)p->n_norm;
  }
  if (loss) {
    double l = 0.0;
    for (int64_t c = 0; c < nch; ++c) l += lpart[c];
    *loss = l / (double)p->n_norm;
  }
  free(part);
  free(lpart);
}

/* P_X(v): ℓ2 projection onto X.
 *  BALL        B(R; c): c + (v - c) min(1, R / ||v - c||)  — PAPER.md:946,1025;
 *                        SPEC.md:249-257
 *  NONNEG      max(v, 0)                                   — PAPER.md:1252,1263;
 *                                                            SPEC.md:240-248
 *  NONNEG_BALL R_+^d ∩ B(R) centred at 0: P_B(P_+(v))      — reading R14
 *  out may alias v. */
void oracle_project(int set, int64_t d, double R, const double *c, const double *v, double *out) {
  if (set == OR_SET_NONE) {
    if (out != v) memcpy(out, v, (size_t)d * sizeof(double));
    return;
  }
  if (set == OR_SET_NONNEG || set == OR_SET_NONNEG_BALL) {
    for (int64_t k = 0; k < d; ++k) out[k] = v[k] > 0.0 ? v[k] : 0.0;
    if (set == OR_SET_NONNEG) return;
    double nrm2 = 0.0;
    for (int64_t k = 0; k < d; ++k) nrm2 += out[k] * out[k];
    const double nrm = sqrt(nrm2);
    if (nrm > R) for (int64_t k = 0; k < d; ++k) out[k] = out[k] * (R / nrm);
    return;
  }
  /* ball */
  double nrm2 = 0.0;
  for (int64_t k = 0; k < d; ++k) {
    const double df = v[k] - (c ? c[k] : 0.0);
    nrm2 += df * df;
  }
  const double nrm = sqrt(nrm2);
  if (nrm <= R) {
    if (out != v) memcpy(out, v, (size_t)d * sizeof(double));
    return;
  }
  for (int64_t k = 0; k < d; ++k) {
    const double ck = c ? c[k] : 0.0;
    out[k] = ck + (v[k] - ck) * (R / nrm);
  }
}

int oracle_project_tv(int side, const double *z, double tau, double tv_tol, double rtol,
                      int max_it, double *x);
int oracle_project_tv_k(int side, const double *z, double tau, double tv_tol, double rtol,
                        int max_it, int K, double *x);
int oracle_project_tv_nonneg_k(int side, const double *z, double tau, double tv_tol, double rtol,
                               int max_it, double tol, int max_outer, int K, double *out);
int oracle_project_tv_nonneg(int side, const double *z, double tau, double tv_tol, double rtol,
                             int max_it, double tol, int max_outer, double *out);
int oracle_project_tv_nonneg_kw(int side, const double *z, double tau, double tv_tol, double rtol,
                                int max_it, double tol, int max_outer, int K, int warm, double *out);
int oracle_project_tv_k_warm(int side, const double *z, double tau, double tv_tol, double rtol,
                             int max_it, int K, double *ustate, double *x);
int oracle_prox_tv_from(int side, const double *z, double lam, double rtol, int max_it, double *x,
                        double *u_out, const double *u_in);

/* P_X for the problem's set: the closed forms above, or the TV sets of
 * NEXT-2.  out may alias v. */
static void project_p(const oracle_problem *p, const double *v, double *out) {
  if (p->set == OR_SET_TV_NONNEG || p->set == OR_SET_TV) {
    const int64_t d = p->d;
    double *t = (double *)malloc((size_t)d * sizeof(double));
    if (p->set == OR_SET_TV_NONNEG) {
      oracle_project_tv_nonneg_kw(p->tv_side, v, p->tv_tau, p->tv_tol, p->tv_rtol, p->tv_max_it,
                                  p->tv_dtol, p->tv_max_outer, p->tv_k, p->tv_warm, t);
    } else {
      const int K = p->tv_k < 1 ? 1 : p->tv_k;
      double *ust = p->tv_warm ? (double *)calloc((size_t)K * 2 * p->tv_side * (p->tv_side - 1) + 1,
                                                  sizeof(double))
                               : NULL;
      oracle_project_tv_k_warm(p->tv_side, v, p->tv_tau, p->tv_tol, p->tv_rtol, p->tv_max_it, K, ust, t);
      free(ust);
    }
    memcpy(out, t, (size_t)d * sizeof(double));
    free(t);
    return;
  }
  oracle_project(p->set, p->d, p->R, p->center, v, out);
}

/* EXACT, Eq.(extragrad-method), constant step γ:
 *   x_1 = P_X(x_in)                       (x_1 ∈ X)
 *   x_{t+1/2} = P_X(x_t - γ F(x_t))
 *   x_{t+1}   = P_X(x_t - γ F(x_{t+1/2}))   (both steps anchored at x_t)
 * Returns x_{T+1} in x.  trace (may be NULL) gets [2T] losses ℓ at the points
 * where F was evaluated.  Returns 0, or t (1-based) of the first non-finite
 * iterate. */
int oracle_solve(const oracle_problem *p, int T, double gamma, double *x, double *trace) {
  const int64_t d = p->d;
  double *g = (double *)malloc((size_t)d * sizeof(double));
  double *xh = (double *)malloc((size_t)d * sizeof(double));
  double *v = (double *)malloc((size_t)d * sizeof(double));
  int bad = 0;
  project_p(p, x, x);
  for (int t = 1; t <= T && !bad; ++t) {
    double l;
    oracle_F(p, x, g, &l);
    if (trace) trace[2 * (t - 1)] = l;
    for (int64_t k = 0; k < d; ++k) v[k] = x[k] - gamma * g[k];
    project_p(p, v, xh);
    oracle_F(p, xh, g, &l);
    if (trace) trace[2 * (t - 1) + 1] = l;
    for (int64_t k = 0; k < d; ++k) v[k] = x[k] - gamma * g[k];
    project_p(p, v, x);
    for (int64_t k = 0; k < d; ++k)
      if (!isfinite(x[k]) || !isfinite(xh[k])) { bad = t; break; }
  }
  free(g);
  free(xh);
  free(v);
  return bad;
}

/* λ_max(Σ), Σ = (1/n_norm) A^T A, by power iteration
 * v <- Σ v / ||Σ v|| from v_0 = 1/sqrt(d), stopping when the Rayleigh
 * estimate changes by <= tol relatively or after max_it. */
double oracle_lambda_max(const oracle_problem *p, int max_it, double tol, int *iters) {
  const int64_t n = p->n, d = p->d;
  double *v = (double *)malloc((size_t)d * sizeof(double));
  double *w = (double *)malloc((size_t)d * sizeof(double));
  double *z = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
  for (int64_t k = 0; k < d; ++k) v[k] = 1.0 / sqrt((double)d);
  double lam = 0.0;
  int it = 0;
  for (it = 1; it <= max_it; ++it) {
    oracle_forward(p, v, z);
    for (int64_t k = 0; k < d; ++k) w[k] = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      if (!p->csr) {
        for (int64_t k = 0; k < d; ++k) w[k] += z[i] * a_at(p, i, k);
      } else {
        for (int64_t e = p->row_ptr[i]; e < p->row_ptr[i + 1]; ++e) w[p->col[e]] += z[i] * v_at(p, e);
      }
    }
    double nrm2 = 0.0;
    for (int64_t k = 0; k < d; ++k) {
      w[k] /= (double)p->n_norm;
      nrm2 += w[k] * w[k];
    }
    const double nrm = sqrt(nrm2);
    const double prev = lam;
    lam = nrm; /* ||Σ v|| with ||v|| = 1 */
    for (int64_t k = 0; k < d; ++k) v[k] = w[k] / nrm;
    if (it > 1 && fabs(lam - prev) <= tol * lam) break;
  }
  if (iters) *iters = it;
  free(v);
  free(w);
  free(z);
  return lam;
}

/* Known-materials reparameterisation, Appendix A.1:
 *   Ī'_i  = Ī Σ_j s_j exp(-μ_j b_i)
 *   s'_ij = s_j exp(-μ_j b_i) / Σ_k s_k exp(-μ_k b_i)
 * with b_i = <a_i^1, x^1> + <a_i^2, x^2> the known-material line integral,
 * clamped to b_i+ when clamp = 1 (reading R7; SPEC.md:88-90 requires e_j >= 0). */
void oracle_reparam(int W, const double *s, const double *mu, double I_bar, int64_t n,
                    const double *b, int clamp, double *s_row, double *I_row) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const double bi = (clamp && b[i] < 0.0) ? 0.0 : b[i];
    double tot = 0.0;
    for (int j = 0; j < W; ++j) tot += s[j] * exp(-mu[j] * bi);
    for (int j = 0; j < W; ++j) s_row[i * W + j] = s[j] * exp(-mu[j] * bi) / tot;
    I_row[i] = I_bar * tot;
  }
}

/* ------------------------------------------------------------------ NEXT-1
 * Stacked multi-window operator.  Footnote to Eq.(eq:model-orig)
 * ("we do include multiple (distinct but overlapping) detector windows"), the
 * window-indexed model Eq.(model:multi-material) PAPER.md:782-784 with M = 1
 * (Ī_ω and s_{ω,j} per window, μ_j per wavelength), and
 * SPEC.md:310 ("n is the total stacked ray count"):
 *   F(x) = (1/n_tot) Σ_ω Σ_i [y_{ω,i} - Ī_ω h_ω(<a_i,x>)] a_i,
 *   h_ω(t) = Σ_j s_{ω,j} exp(-μ_j t_+),   n_tot = Ω · n_norm,
 *   ℓ(x) = (1/n_tot) Σ_ω Σ_i [y_{ω,i} z_i - Ī_ω H_ω(z_i)]   (reading R2 per window).
 * s_win: [Ω*W] (window-major), I_win: [Ω], y_win: [Ω*n] (window-major).
 * p->s, p->I_bar, p->y, p->s_row, p->I_row are not used.  Written as the
 * double sum of the definition: windows outer, rows inner. */
void oracle_F_windows(const oracle_problem *p, int Omega, const double *s_win,
                      const double *I_win, const double *y_win, const double *x, double *g,
                      double *loss) {
  const int64_t n = p->n, d = p->d;
  double *acc = (double *)calloc((size_t)d, sizeof(double));
  double l = 0.0;
  for (int w = 0; w < Omega; ++w) {
    const double *sw = s_win + (size_t)w * p->W;
    for (int64_t i = 0; i < n; ++i) {
      const double z = row_dot(p, i, x);
      const double yv = y_win[(size_t)w * n + i];
      const double r = yv - I_win[w] * oracle_h(p->W, sw, p->mu, z, p->relu);
      l += yv * z - I_win[w] * oracle_H(p->W, sw, p->mu, z, p->relu);
      if (!p->csr) {
        for (int64_t k = 0; k < d; ++k) acc[k] += r * a_at(p, i, k);
      } else {
        for (int64_t e = p->row_ptr[i]; e < p->row_ptr[i + 1]; ++e) acc[p->col[e]] += r * v_at(p, e);
      }
    }
  }
  const double ntot = (double)Omega * (double)p->n_norm;
  if (g)
    for (int64_t k = 0; k < d; ++k) g[k] = acc[k] / ntot;
  if (loss) *loss = l / ntot;
  free(acc);
}

/* Averaged iterate, PAPER.md:1277-1278 ("the average x̄_t of the previous t/2
 * iterates"), window ⌈k/2⌉..k inclusive (reading R15):
 * hist holds iterates x_1..x_k row by row ([k*d]); out = mean of rows
 * ⌈k/2⌉..k (1-based). */
void oracle_average(const double *hist, int k, int64_t d, double *out) {
  const int lo = (k + 1) / 2;  /* ⌈k/2⌉ */
  for (int64_t c = 0; c < d; ++c) out[c] = 0.0;
  for (int j = lo; j <= k; ++j)
    for (int64_t c = 0; c < d; ++c) out[c] += hist[(size_t)(j - 1) * d + c];
  for (int64_t c = 0; c < d; ++c) out[c] /= (double)(k - lo + 1);
}

/* EXACT (Eq. extragrad-method) with the averaged-iterate stopping rule of
 * PAPER.md:1279 ("the first iteration at which ||x̄_t - x̄_{t-1}||_2 <= 1e-5"):
 * iterates x_1 = P_X(x_in), x_{k+1} from x_k by one EXACT iteration; after
 * producing x_k (k >= 2) stop if ||x̄_k - x̄_{k-1}|| <= tol, or when k = T_max+1.
 * Returns in xbar the x̄_k at the stop, in x the last iterate x_k, in *iters
 * the EXACT iterations run (k - 1) and in *move the last ||x̄_k - x̄_{k-1}||.
 * Return value: 0, or the iteration of a non-finite iterate. */
int oracle_solve_avg(const oracle_problem *p, int T_max, double gamma, double tol, double *x,
                     double *xbar, int *iters, double *move) {
  const int64_t d = p->d;
  double *hist = (double *)malloc((size_t)(T_max + 1) * (size_t)d * sizeof(double));
  double *prev = (double *)malloc((size_t)d * sizeof(double));
  int bad = 0, k = 1;
  double mv = 0.0;
  project_p(p, x, x);
  memcpy(hist, x, (size_t)d * sizeof(double));
  oracle_average(hist, 1, d, xbar);
  double *g = (double *)malloc((size_t)d * sizeof(double));
  double *xh = (double *)malloc((size_t)d * sizeof(double));
  double *v = (double *)malloc((size_t)d * sizeof(double));
  for (int t = 1; t <= T_max; ++t) {
    /* one EXACT iteration, both half-steps anchored at x_t */
    oracle_F(p, x, g, NULL);
    for (int64_t c = 0; c < d; ++c) v[c] = x[c] - gamma * g[c];
    project_p(p, v, xh);
    oracle_F(p, xh, g, NULL);
    for (int64_t c = 0; c < d; ++c) v[c] = x[c] - gamma * g[c];
    project_p(p, v, x);
    for (int64_t c = 0; c < d; ++c)
      if (!isfinite(x[c])) bad = t;
    if (bad) break;
    k = t + 1;
    memcpy(hist + (size_t)t * d, x, (size_t)d * sizeof(double));
    memcpy(prev, xbar, (size_t)d * sizeof(double));
    oracle_average(hist, k, d, xbar);
    double s = 0.0;
    for (int64_t c = 0; c < d; ++c) s += (xbar[c] - prev[c]) * (xbar[c] - prev[c]);
    mv = sqrt(s);
    if (mv <= tol) break;
  }
  if (iters) *iters = k - 1;
  if (move) *move = mv;
  free(hist);
  free(prev);
  free(g);
  free(xh);
  free(v);
  return bad;
}

/* ------------------------------------------------------------------ NEXT-3
 * The comparison objectives of §3.1, evaluated on the same data:
 *   mode 1  L2(x) = (1/n) Σ_i (Ī h(z_i) - y_i)^2
 *   mode 2  L1(x) = (1/n) Σ_i |Ī h(z_i) - y_i|
 *   mode 3  NLL(x) = (1/n) Σ_i [Ī h(z_i) - y_i log(Ī h(z_i))]
 *           (Loss(z) at z = A x, scaled by 1/n like the other two)
 * and their (sub)gradients by the chain rule, with h's a.e. derivative
 * h'(t) = -Σ_j s_j μ_j exp(-μ_j t) for t > 0 and h'(t) = 0 for t <= 0 under
 * relu ("taken as 0 ... at exactly 0"); relu = 0: the
 * formula for every t.  sign(0) = 0 for L1.
 *   ∇L2  = (1/n) Σ_i 2 (Ī h - y_i) Ī h'(z_i) a_i
 *   ∂L1  = (1/n) Σ_i sign(Ī h - y_i) Ī h'(z_i) a_i
 *   ∇NLL = (1/n) Σ_i (Ī - y_i / h(z_i)) h'(z_i) a_i
 * Ī, s are per row when s_row/I_row are given. */
static double hprime(int W, const double *s, const double *mu, double t, int relu) {
  if (relu && !(t > 0.0)) return 0.0;
  double v = 0.0;
  for (int j = 0; j < W; ++j) v += s[j] * mu[j] * exp(-mu[j] * t);
  return -v;
}

void oracle_objective(const oracle_problem *p, int mode, const double *x, double *g,
                      double *loss) {
  const int64_t n = p->n, d = p->d;
  double *acc = (double *)calloc((size_t)d, sizeof(double));
  double l = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double z = row_dot(p, i, x);
    const double *si = row_s(p, i);
    const double Ii = row_I(p, i);
    const double h = oracle_h(p->W, si, p->mu, z, p->relu);
    const double hp = hprime(p->W, si, p->mu, z, p->relu);
    const double m = Ii * h;
    double phi = 0.0;
    if (mode == 1) {
      l += (m - p->y[i]) * (m - p->y[i]);
      phi = 2.0 * (m - p->y[i]) * Ii * hp;
    } else if (mode == 2) {
      const double r = m - p->y[i];
      l += fabs(r);
      phi = (r > 0.0 ? 1.0 : (r < 0.0 ? -1.0 : 0.0)) * Ii * hp;
    } else {
      l += m - p->y[i] * log(m);
      phi = (Ii - p->y[i] / h) * hp;
    }
    if (!p->csr) {
      for (int64_t k = 0; k < d; ++k) acc[k] += phi * a_at(p, i, k);
    } else {
      for (int64_t e = p->row_ptr[i]; e < p->row_ptr[i + 1]; ++e) acc[p->col[e]] += phi * v_at(p, e);
    }
  }
  if (g)
    for (int64_t k = 0; k < d; ++k) g[k] = acc[k] / (double)p->n_norm;
  if (loss) *loss = l / (double)p->n_norm;
  free(acc);
}

/* Projected gradient descent, the MSE-GD baseline's iteration (§3.1,
 * PAPER.md:1225-1229): x_1 = P_X(x_in), x_{t+1} = P_X(x_t - γ ∇L(x_t)) for the
 * objective `mode` of oracle_objective.  Returns 0 or the non-finite iteration. */
int oracle_solve_gd(const oracle_problem *p, int mode, int T, double gamma, double *x) {
  const int64_t d = p->d;
  double *g = (double *)malloc((size_t)d * sizeof(double));
  int bad = 0;
  project_p(p, x, x);
  for (int t = 1; t <= T && !bad; ++t) {
    oracle_objective(p, mode, x, g, NULL);
    for (int64_t k = 0; k < d; ++k) x[k] = x[k] - gamma * g[k];
    project_p(p, x, x);
    for (int64_t k = 0; k < d; ++k)
      if (!isfinite(x[k])) { bad = t; break; }
  }
  free(g);
  return bad;
}

/* ------------------------------------------------------------------ NEXT-2
 * The paper's CT constraint set X = X1 ∩ X2, X1 = {||x||_TV <= τ},
 * X2 = R_+^d, for a side x side image stored row-major
 * (pixel (r, c) at r*side + c).  Readings (R19-R21, after
 * SPEC.md:214-282): anisotropic TV with forward differences; the TV prox by
 * FISTA on the dual; λ bracketed by doubling from 1 then bisected. */

/* D x: horizontal differences h(r,c) = x[r][c+1] - x[r][c] at index
 * r*(side-1) + c (c < side-1), then vertical v(r,c) = x[r+1][c] - x[r][c] at
 * index side*(side-1) + r*side + c (r < side-1). */
static void tv_D(int side, const double *x, double *dx) {
  const int nh = side * (side - 1);
  for (int r = 0; r < side; ++r)
    for (int c = 0; c + 1 < side; ++c) dx[r * (side - 1) + c] = x[r * side + c + 1] - x[r * side + c];
  for (int r = 0; r + 1 < side; ++r)
    for (int c = 0; c < side; ++c) dx[nh + r * side + c] = x[(r + 1) * side + c] - x[r * side + c];
}

/* D^T u (the adjoint of tv_D). */
static void tv_Dt(int side, const double *u, double *out) {
  const int nh = side * (side - 1);
  for (int k = 0; k < side * side; ++k) out[k] = 0.0;
  for (int r = 0; r < side; ++r)
    for (int c = 0; c + 1 < side; ++c) {
      const double uh = u[r * (side - 1) + c];
      out[r * side + c + 1] += uh;
      out[r * side + c] -= uh;
    }
  for (int r = 0; r + 1 < side; ++r)
    for (int c = 0; c < side; ++c) {
      const double uv = u[nh + r * side + c];
      out[(r + 1) * side + c] += uv;
      out[r * side + c] -= uv;
    }
}

/* ||x||_TV = Σ |D x|. */
double oracle_tv_norm(int side, const double *x) {
  const int m = 2 * side * (side - 1);
  double *dx = (double *)malloc((size_t)(m > 0 ? m : 1) * sizeof(double));
  tv_D(side, x, dx);
  double t = 0.0;
  for (int k = 0; k < m; ++k) t += fabs(dx[k]);
  free(dx);
  return t;
}

/* x = argmin ||x - z||^2 + λ ||x||_TV, Eq.(TV-regularization) PAPER.md:1257-1259.
 * Dual: x = z - D^T u with u = argmin_{|u_k| <= λ/2} ½||z - D^T u||^2,
 * solved by FISTA (Beck-Teboulle) with step 1/8 (||D||^2 <= 8): from w,
 *   x_w = z - D^T w,  u+ = clip(w + D x_w / 8, ±λ/2),  t+ = (1 + sqrt(1 + 4t^2))/2,
 *   w = u+ + ((t - 1)/t+)(u+ - u);
 * stop when the primal x(u) = z - D^T u moves by <= rtol ||x(u)|| or after
 * max_it iterations.  u_out (may be NULL) receives u [2 side (side-1)].
 * Returns the iterations used. */
int oracle_prox_tv_from(int side, const double *z, double lam, double rtol, int max_it, double *x,
                        double *u_out, const double *u_in);

int oracle_prox_tv(int side, const double *z, double lam, double rtol, int max_it, double *x,
                   double *u_out) {
  return oracle_prox_tv_from(side, z, lam, rtol, max_it, x, u_out, NULL);
}

/* FISTA iterations run by all proxes since the last reset (statistics only). */
static long long g_fista_iters = 0;
long long oracle_fista_iterations(int reset) {
  const long long v = g_fista_iters;
  if (reset) g_fista_iters = 0;
  return v;
}

/* The same FISTA started from the dual point clip(u_in, ±λ/2) (u_in NULL: 0). */
int oracle_prox_tv_from(int side, const double *z, double lam, double rtol, int max_it, double *x,
                        double *u_out, const double *u_in) {
  const int d = side * side, m = 2 * side * (side - 1);
  double *u = (double *)calloc((size_t)(m > 0 ? m : 1), sizeof(double));
  double *w = (double *)calloc((size_t)(m > 0 ? m : 1), sizeof(double));
  if (u_in)
    for (int k = 0; k < m; ++k) {
      const double v = u_in[k];
      u[k] = w[k] = v > lam / 2.0 ? lam / 2.0 : (v < -lam / 2.0 ? -lam / 2.0 : v);
    }
  double *un = (double *)malloc((size_t)(m > 0 ? m : 1) * sizeof(double));
  double *dx = (double *)malloc((size_t)(m > 0 ? m : 1) * sizeof(double));
  double *xw = (double *)malloc((size_t)d * sizeof(double));
  double *xp = (double *)malloc((size_t)d * sizeof(double));
  double t = 1.0;
  int it = 0;
  /* the primal of the starting dual: x(u0) = z - Dᵀu0 (= z from u0 = 0) */
  tv_Dt(side, u, x);
  for (int k = 0; k < d; ++k) x[k] = z[k] - x[k];
  if (lam > 0.0 && m > 0) {
    for (it = 1; it <= max_it; ++it) {
      tv_Dt(side, w, xw);
      for (int k = 0; k < d; ++k) xw[k] = z[k] - xw[k];
      tv_D(side, xw, dx);
      for (int k = 0; k < m; ++k) {
        double v = w[k] + dx[k] / 8.0;
        un[k] = v > lam / 2.0 ? lam / 2.0 : (v < -lam / 2.0 ? -lam / 2.0 : v);
      }
      const double tn = (1.0 + sqrt(1.0 + 4.0 * t * t)) / 2.0;
      for (int k = 0; k < m; ++k) {
        w[k] = un[k] + ((t - 1.0) / tn) * (un[k] - u[k]);
        u[k] = un[k];
      }
      t = tn;
      for (int k = 0; k < d; ++k) xp[k] = x[k];
      tv_Dt(side, u, x);
      for (int k = 0; k < d; ++k) x[k] = z[k] - x[k];
      double dn = 0.0, xn = 0.0;
      for (int k = 0; k < d; ++k) {
        dn += (x[k] - xp[k]) * (x[k] - xp[k]);
        xn += x[k] * x[k];
      }
      if (sqrt(dn) <= rtol * sqrt(xn)) break;
    }
    if (it > max_it) it = max_it;
  }
  g_fista_iters += it;
  if (u_out)
    for (int k = 0; k < m; ++k) u_out[k] = u[k];
  free(u);
  free(w);
  free(un);
  free(dx);
  free(xw);
  free(xp);
  return it;
}

/* Approximate projection onto X1 = {||x||_TV <= τ}: z
 * itself if ||z||_TV <= τ; else the prox of Eq.(TV-regularization) with λ
 * "tuned via a binary search" until | ||x̄||_TV - τ | <= tv_tol (0.01 in the
 * paper).  Bracket: λ_hi = 1, doubled while ||prox(z, λ_hi)||_TV
 * > τ; bisection of [λ_lo, λ_hi] for at most 60 steps.  Returns the bisection
 * steps used (0 if z ∈ X1).
 *
 * Reading R22: the search may evaluate K values of λ per round
 * (the GPU evaluates them at once, one thread-block cluster each).  With
 * K = 1 this is exactly the search above.  For K > 1:
 *   bracket round g: λ = 2^(gK + k), k = 0..K-1; the first k with TV <= τ
 *     gives hi = 2^(gK + k), lo = 2^(gK + k - 1) (0 when gK + k = 0);
 *     at most 200 values, as the doubling loop;
 *   search round: λ_k = lo + (hi - lo)(k + 1)/(K + 1) (K = 1: (lo + hi)/2);
 *     stop at the smallest k with |TV_k - τ| <= tv_tol (its prox is the
 *     result); else, with k* the smallest k with TV_k <= τ, the new bracket
 *     is [λ_{k*-1} (lo if k* = 0), λ_{k*}], or [λ_{K-1}, hi] if there is none;
 *     at most 60 rounds, after which the result is the prox at λ_{k*} (at
 *     λ_{K-1} if there is none).
 * Returns the rounds used. */
static int project_tv_core(int side, const double *z, double tau, double tv_tol, double rtol, int max_it,
                           int K, double *ustate, double *x);

int oracle_project_tv_k(int side, const double *z, double tau, double tv_tol, double rtol,
                        int max_it, int K, double *x) {
  return project_tv_core(side, z, tau, tv_tol, rtol, max_it, K, NULL, x);
}

/* The same with warm-started proxes (reading R23): ustate [K][2 side (side-1)]
 * holds, per λ slot k, the dual solution of the slot's last prox; each prox
 * starts from it (clipped to the new box by oracle_prox_tv_from) and leaves
 * its own solution there.  ustate all zeros = cold starts for the first
 * round.  NULL: every prox starts from 0 (the search above). */
int oracle_project_tv_k_warm(int side, const double *z, double tau, double tv_tol, double rtol,
                             int max_it, int K, double *ustate, double *x) {
  return project_tv_core(side, z, tau, tv_tol, rtol, max_it, K, ustate, x);
}

static int project_tv_core(int side, const double *z, double tau, double tv_tol, double rtol, int max_it,
                           int K, double *ustate, double *x) {
  const int d = side * side;
  const size_t m = (size_t)2 * side * (side - 1);
  if (K < 1) K = 1;
  if (oracle_tv_norm(side, z) <= tau) {
    for (int k = 0; k < d; ++k) x[k] = z[k];
    return 0;
  }
  double *xs = (double *)malloc((size_t)K * d * sizeof(double));
  double *tv = (double *)malloc((size_t)K * sizeof(double));
  double *lam = (double *)malloc((size_t)K * sizeof(double));
  double lo = 0.0, hi = 1.0;
  int found = 0;
  for (int g = 0; g * K < 200 && !found; ++g) {
    for (int k = 0; k < K; ++k) {
      const int e = g * K + k;
      if (e >= 200) { tv[k] = INFINITY; continue; }
      lam[k] = ldexp(1.0, e);
      oracle_prox_tv_from(side, z, lam[k], rtol, max_it, xs + (size_t)k * d, ustate ? ustate + k * m : NULL,
                          ustate ? ustate + k * m : NULL);
      tv[k] = oracle_tv_norm(side, xs + (size_t)k * d);
    }
    for (int k = 0; k < K; ++k) {
      const int e = g * K + k;
      if (e < 200 && tv[k] <= tau) {
        hi = lam[k];
        lo = e == 0 ? 0.0 : ldexp(1.0, e - 1);
        found = 1;
        break;
      }
    }
    if (!found) {
      const int e = (g + 1) * K - 1 < 199 ? (g + 1) * K - 1 : 199;
      lo = ldexp(1.0, e);
      hi = 2.0 * lo;
    }
  }
  int rounds, sel = K - 1;
  for (rounds = 1; rounds <= 60; ++rounds) {
    for (int k = 0; k < K; ++k) {
      lam[k] = K == 1 ? 0.5 * (lo + hi) : lo + (hi - lo) * (double)(k + 1) / (double)(K + 1);
      oracle_prox_tv_from(side, z, lam[k], rtol, max_it, xs + (size_t)k * d, ustate ? ustate + k * m : NULL,
                          ustate ? ustate + k * m : NULL);
      tv[k] = oracle_tv_norm(side, xs + (size_t)k * d);
    }
    int hit = -1, ks = -1;
    for (int k = 0; k < K && hit < 0; ++k)
      if (fabs(tv[k] - tau) <= tv_tol) hit = k;
    for (int k = 0; k < K && ks < 0; ++k)
      if (tv[k] <= tau) ks = k;
    if (hit >= 0) {
      sel = hit;
      break;
    }
    sel = ks >= 0 ? ks : K - 1;
    if (ks >= 0) {
      const double nlo = ks > 0 ? lam[ks - 1] : lo;
      hi = lam[ks];
      lo = nlo;
    } else {
      lo = lam[K - 1];
    }
  }
  if (rounds > 60) rounds = 60;
  for (int k = 0; k < d; ++k) x[k] = xs[(size_t)sel * d + k];
  free(xs);
  free(tv);
  free(lam);
  return rounds;
}

int oracle_project_tv(int side, const double *z, double tau, double tv_tol, double rtol,
                      int max_it, double *x) {
  return oracle_project_tv_k(side, z, tau, tv_tol, rtol, max_it, 1, x);
}

/* Dykstra's algorithm for X1 ∩ X2, Eq.(projection-intersection)
 * z_0 = z, p_0 = q_0 = 0,
 *   y_k = P_X1(z_k + p_k),  p_{k+1} = z_k + p_k - y_k,
 *   z_{k+1} = P_X2(y_k + q_k),  q_{k+1} = y_k + q_k - z_{k+1},
 * stopping at ||z_{k+1} - z_k||_2 <= tol (1e-4 in the paper) or max_outer.
 * P_X2 keeps the positive entries.  Returns the sweeps. */
int oracle_project_tv_nonneg_k(int side, const double *z, double tau, double tv_tol, double rtol,
                               int max_it, double tol, int max_outer, int K, double *out) {
  return oracle_project_tv_nonneg_kw(side, z, tau, tv_tol, rtol, max_it, tol, max_outer, K, 0, out);
}

/* warm = 1: the proxes of the whole projection — all Dykstra sweeps — share
 * one warm-start state per λ slot (reading R23), zero at the start. */
int oracle_project_tv_nonneg_kw(int side, const double *z, double tau, double tv_tol, double rtol,
                                int max_it, double tol, int max_outer, int K, int warm, double *out) {
  const int d = side * side;
  double *ust = warm ? (double *)calloc((size_t)(K < 1 ? 1 : K) * 2 * side * (side - 1) + 1, sizeof(double))
                     : NULL;
  double *zk = (double *)malloc((size_t)d * sizeof(double));
  double *p = (double *)calloc((size_t)d, sizeof(double));
  double *q = (double *)calloc((size_t)d, sizeof(double));
  double *y = (double *)malloc((size_t)d * sizeof(double));
  double *v = (double *)malloc((size_t)d * sizeof(double));
  for (int k = 0; k < d; ++k) zk[k] = z[k];
  int it;
  for (it = 1; it <= max_outer; ++it) {
    for (int k = 0; k < d; ++k) v[k] = zk[k] + p[k];
    project_tv_core(side, v, tau, tv_tol, rtol, max_it, K, ust, y);
    for (int k = 0; k < d; ++k) p[k] = zk[k] + p[k] - y[k];
    double dn = 0.0;
    for (int k = 0; k < d; ++k) {
      const double s = y[k] + q[k];
      const double zn = s > 0.0 ? s : 0.0;
      q[k] = y[k] + q[k] - zn;
      dn += (zn - zk[k]) * (zn - zk[k]);
      zk[k] = zn;
    }
    if (sqrt(dn) <= tol) break;
  }
  if (it > max_outer) it = max_outer;
  for (int k = 0; k < d; ++k) out[k] = zk[k];
  free(zk);
  free(p);
  free(q);
  free(y);
  free(v);
  free(ust);
  return it;
}

int oracle_project_tv_nonneg(int side, const double *z, double tau, double tv_tol, double rtol,
                             int max_it, double tol, int max_outer, double *out) {
  return oracle_project_tv_nonneg_k(side, z, tau, tv_tol, rtol, max_it, tol, max_outer, 1, out);
}
