/*
 * smo_oracle.c -- plain, slow, fp64 CPU oracle of the binary SMO solve.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  The product path
 * (paper_2311_14908_b200/, libsvmb200.so) never links, imports or calls it, and it
 * shares no code, header, table or constant with the CUDA path.
 *
 * What it follows (PAPER.md = "P:L<line>", SPEC.md = "S:L<line>"):
 *   - problem: binary soft-margin kernel SVM dual QP, y in {+1,-1}     P:L132-133 (§3.1)
 *   - kernels: linear x.y, Gaussian RBF exp(-gamma ||x-y||^2)
 *   - SMO: two multipliers per step "under the KKT constraints"         P:L140 (§3.2)
 *     with the maximal-violating-pair rule, f, I_up/I_low, tie-break,
 *     stopping rule, bias, eta-degenerate rule
 *   - "convergence checks ... for every set of iterations"              P:L144; tested
 *     every iteration here (reading R6)
 *
 * Everything is fp64; X is read as float32 and widened exactly.  Rounding-order
 * readings: squared distance and dot product accumulate in
 * ascending feature order, one fma per term; exp is correctly rounded (computed in
 * double-double and rounded once); kernel arguments below -708 give K = 0.
 *
 * Pins (tests/test_oracle_*.py): closed-form two/three-point duals, RBF two-point,
 * eta = 0 duplicates, separable toy with known margin, brute-force active-set QP,
 * KKT at convergence, invariants per step, mpmath-rounded exp; the second-order working
 * set (oracle_select_second_order, wss = 2) against scikit-learn's libsvm; the projected-GD
 * trainer (oracle_gd_train) against a brute-force box-constrained QP and closed forms.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_LINEAR 0
#define ORACLE_RBF 1

/* ------------------------------------------------------------------ double-double */
typedef struct { double hi, lo; } dd_t;

static dd_t fast_two_sum(double a, double b) {   /* |a| >= |b| */
    dd_t r; r.hi = a + b; r.lo = b - (r.hi - a); return r;
}
static dd_t two_sum(double a, double b) {
    dd_t r; r.hi = a + b; double bb = r.hi - a; r.lo = (a - (r.hi - bb)) + (b - bb); return r;
}
static dd_t two_prod(double a, double b) {
    dd_t r; r.hi = a * b; r.lo = fma(a, b, -r.hi); return r;
}
static dd_t dd_add(dd_t a, dd_t b) {
    dd_t s = two_sum(a.hi, b.hi), t = two_sum(a.lo, b.lo);
    s.lo += t.hi; s = fast_two_sum(s.hi, s.lo);
    s.lo += t.lo; return fast_two_sum(s.hi, s.lo);
}
static dd_t dd_mul(dd_t a, dd_t b) {
    dd_t p = two_prod(a.hi, b.hi);
    p.lo += a.hi * b.lo + a.lo * b.hi;
    return fast_two_sum(p.hi, p.lo);
}
static dd_t dd_div_d(dd_t a, double b) {          /* a / b, ~2^-104 relative */
    double q1 = a.hi / b;
    dd_t p = two_prod(q1, b);
    double r = ((a.hi - p.hi) - p.lo + a.lo) / b;
    return fast_two_sum(q1, r);
}

/* ln 2 and 1/i! in double-double, computed here from their series (no tables). */
static dd_t g_ln2;
static dd_t g_invfact[16];
static int g_init = 0;
static long g_exp_ambiguous = 0;

static void oracle_init(void) {
    if (g_init) return;
    /* ln 2 = sum_{k>=1} 1 / (k 2^k); 120 terms reach far below 2^-110. */
    dd_t s = {0.0, 0.0};
    for (int k = 120; k >= 1; --k) {
        dd_t term = {ldexp(1.0, -k), 0.0};
        s = dd_add(s, dd_div_d(term, (double)k));
    }
    g_ln2 = s;
    g_invfact[0].hi = 1.0; g_invfact[0].lo = 0.0;
    for (int i = 1; i < 16; ++i) g_invfact[i] = dd_div_d(g_invfact[i - 1], (double)i);
    g_init = 1;
}

/*
 * Correctly rounded exp(x) for x in [-708, 0] (the RBF argument range); the
 * reading of "exp" in P:L179 / S:L120 is the exact exponential rounded once.
 *   x = k ln2 + r, |r| <= ln2/2          (r in double-double)
 *   exp(r) = (sum_{i<=12} (r/256)^i / i!)^(2^8)    (double-double, ~2^-96 rel.)
 *   exp(x) = 2^k exp(r), then one rounding to double.
 * A result whose double-double value lies within 2^-88 (relative) of a rounding
 * boundary is counted in g_exp_ambiguous (tests assert it stays 0).
 */
double oracle_exp_cr(double x) {
    oracle_init();
    if (x == 0.0) return 1.0;
    if (x < -708.0) return 0.0;
    double k = nearbyint(x / g_ln2.hi);
    dd_t kl = two_prod(k, g_ln2.hi);                    /* exact */
    dd_t r = two_sum(x, -kl.hi);                        /* exact */
    r = dd_add(r, (dd_t){-kl.lo, 0.0});
    r = dd_add(r, (dd_t){-k * g_ln2.lo, 0.0});
    dd_t y = {ldexp(r.hi, -8), ldexp(r.lo, -8)};
    dd_t p = g_invfact[12];
    for (int i = 11; i >= 0; --i) p = dd_add(dd_mul(p, y), g_invfact[i]);
    for (int i = 0; i < 8; ++i) p = dd_mul(p, p);
    /* p is normalised (p.hi = RN(p.hi + p.lo)); 2^k scaling is exact because
     * x >= -708 keeps the result >= 2^-1021 (normal). */
    if (p.lo != 0.0) {
        double nb = p.lo > 0 ? nextafter(p.hi, INFINITY) : nextafter(p.hi, -INFINITY);
        double half_gap = fabs(nb - p.hi) * 0.5;
        if (fabs(fabs(p.lo) - half_gap) <= ldexp(p.hi, -88)) g_exp_ambiguous++;
    }
    return ldexp(p.hi, (int)k);
}

long oracle_exp_ambiguous_count(void) { return g_exp_ambiguous; }

/* ------------------------------------------------------------------------ kernels */
/* ||a - b||^2, ascending k, one fma per term (reading R13). */
static double sqdist(const float* a, const float* b, int64_t d) {
    double acc = 0.0;
    for (int64_t k = 0; k < d; ++k) {
        double t = (double)a[k] - (double)b[k];   /* exact */
        acc = fma(t, t, acc);
    }
    return acc;
}
/* a . b, ascending k (fp32 x fp32 products are exact in fp64). */
static double dot(const float* a, const float* b, int64_t d) {
    double acc = 0.0;
    for (int64_t k = 0; k < d; ++k) acc = fma((double)a[k], (double)b[k], acc);
    return acc;
}

/* K(a, b): S:L119-127.  same != 0 marks the diagonal (RBF K_ii == 1). */
double oracle_kernel(int kernel, double gamma, const float* a, const float* b, int64_t d, int same) {
    if (kernel == ORACLE_LINEAR) return dot(a, b, d);
    if (same) return 1.0;
    double arg = -(gamma * sqdist(a, b, d));
    return oracle_exp_cr(arg);
}

/* row i of K over all n samples: S:L128-136 (kernel_row). */
void oracle_kernel_row(int kernel, double gamma, const float* X, int64_t n, int64_t d,
                       int64_t i, double* out) {
    for (int64_t j = 0; j < n; ++j)
        out[j] = oracle_kernel(kernel, gamma, X + i * d, X + j * d, d, i == j);
}

/* --------------------------------------------------------------------- selection */
/* i_up = argmin f over I_up, i_low = argmax f over I_low, ties -> lowest
 * index.  Returns 0 when either set is empty. */
int oracle_select(const double* f, const int8_t* y, const double* alpha, double C, int64_t n,
                  int64_t* i_up, int64_t* i_low, double* b_up, double* b_low) {
    int64_t u = -1, l = -1;
    double fu = 0.0, fl = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        int in_up = (y[j] == 1 && alpha[j] < C) || (y[j] == -1 && alpha[j] > 0.0);
        int in_low = (y[j] == 1 && alpha[j] > 0.0) || (y[j] == -1 && alpha[j] < C);
        if (in_up && (u < 0 || f[j] < fu)) { u = j; fu = f[j]; }
        if (in_low && (l < 0 || f[j] > fl)) { l = j; fl = f[j]; }
    }
    *i_up = u; *i_low = l; *b_up = fu; *b_low = fl;
    return (u >= 0 && l >= 0);
}

/* ------------------------------------------------------------------------- train */
/*
 * SMO, step by step (SURVEY.md §8(c) pseudo-code):
 *   alpha = 0, f = -y
 *   loop: select (u, l); if b_low - b_up <= 2 tol: converged
 *         if it == max_iter: stop, not converged
 *         eta = K_uu + K_ll - 2 K_ul
 *         t = min(t_u, t_l, gap / max(eta, 1e-12))        (clip to the box; eta rule S:L251)
 *         alpha_u += y_u t, alpha_l -= y_l t, snapped to the bound when clipped
 *         f_j += c_u K(u, j) + c_l K(l, j)
 *   b = -(b_up + b_low) / 2
 * Optional warm start (alpha0 and f0 both non-NULL) resumes a saved state.
 * pair_trace (nullable) receives (i_up, i_low) per update.
 * Returns 0 on success, -3 on a single-class problem, -1 on bad arguments.
 */
/* Second-order working-set selection (WSS2; the method of Fan, Chen and Lin 2005 that
 * P:L140 cites as "fan2005working").  Given the first-order u (the
 * minimum f over I_up), choose l among t in I_low with f_t > f_u maximising the gain of
 * the unconstrained pair step,
 *     g_t = (f_t - f_u)^2 / a_t,   a_t = K_uu + K_tt - 2 K_ut  (a_t <= 1e-12 -> 1e-12),
 * ties to the lowest index (reading R4).  Returns -1 when no t qualifies. */
static int64_t select_second_order_masked(const float* X, const int8_t* y, const double* alpha,
                                          const double* f, double C, int64_t n, int64_t d,
                                          int kernel, double gamma, int64_t u, const uint8_t* active);

int64_t oracle_select_second_order(const float* X, const int8_t* y, const double* alpha,
                                   const double* f, double C, int64_t n, int64_t d,
                                   int kernel, double gamma, int64_t u) {
    return select_second_order_masked(X, y, alpha, f, C, n, d, kernel, gamma, u, NULL);
}

/* the same over the rows with active[t] != 0 (NULL: all rows; R29 windows) */
static int64_t select_second_order_masked(const float* X, const int8_t* y, const double* alpha,
                                          const double* f, double C, int64_t n, int64_t d,
                                          int kernel, double gamma, int64_t u, const uint8_t* active) {
    const float* xu = X + u * d;
    const double Kuu = oracle_kernel(kernel, gamma, xu, xu, d, 1);
    int64_t best = -1;
    double best_g = 0.0;
    for (int64_t t = 0; t < n; ++t) {
        if (active && !active[t]) continue;
        const int pos = y[t] == 1;
        const int low = pos ? (alpha[t] > 0.0) : (alpha[t] < C);
        if (!low) continue;
        const double b = f[t] - f[u];
        if (!(b > 0.0)) continue;
        const float* xt = X + t * d;
        const double Kut = oracle_kernel(kernel, gamma, xu, xt, d, t == u);
        const double Ktt = oracle_kernel(kernel, gamma, xt, xt, d, 1);
        double a = Kuu + Ktt - 2.0 * Kut;
        if (!(a > 1e-12)) a = 1e-12;
        const double g = (b * b) / a;
        if (best < 0 || g > best_g) { best = t; best_g = g; }
    }
    return best;
}

int oracle_svm_train(const float* X, const int8_t* y, int64_t n, int64_t d, double C,
                     int kernel, double gamma, double tol, int64_t max_iter,
                     const double* alpha0, const double* f0,
                     double* alpha, double* f, double* b_out, int64_t* iters_out,
                     int* converged_out, double* b_up_out, double* b_low_out,
                     int64_t* pair_trace, int64_t trace_cap);

/* Window shrinking (reading R29; the shrinking heuristic of the SMO
 * improvements P:L140 cites, "keerthi2001improvements" / "fan2005working", in the form of
 * Joachims / LIBSVM, with f kept exact): the solve runs in windows of H updates.  At a
 * window start every row is active; the pair is selected over all rows and the stopping
 * test taken; then the rows that cannot form a violating pair are set aside for the
 * window -- i in I_up only with f_i > b_low, and i in I_low only with f_i < b_up.  Inside
 * the window the pair is selected over the active rows only; when their gap falls to
 * 2 tol, or after H updates, the window ends (the next selection is over all rows
 * again).  Every update is applied to every row's f (rows set aside are only excluded
 * from the selection), so f stays the exact incremental value. */
static void shrink_mark(const double* f, const int8_t* y, const double* alpha, double C, int64_t n,
                        double b_up, double b_low, uint8_t* active) {
    for (int64_t j = 0; j < n; ++j) {
        int in_up = (y[j] == 1 && alpha[j] < C) || (y[j] == -1 && alpha[j] > 0.0);
        int in_low = (y[j] == 1 && alpha[j] > 0.0) || (y[j] == -1 && alpha[j] < C);
        int out = (in_up && !in_low && f[j] > b_low) || (in_low && !in_up && f[j] < b_up);
        active[j] = (uint8_t)!out;
    }
}

/* S:L194-202 selection restricted to the rows with active[j] != 0 (NULL: all rows). */
static int select_active(const double* f, const int8_t* y, const double* alpha, double C, int64_t n,
                         const uint8_t* active, int64_t* i_up, int64_t* i_low, double* b_up, double* b_low) {
    int64_t u = -1, l = -1;
    double fu = 0.0, fl = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        if (active && !active[j]) continue;
        int in_up = (y[j] == 1 && alpha[j] < C) || (y[j] == -1 && alpha[j] > 0.0);
        int in_low = (y[j] == 1 && alpha[j] > 0.0) || (y[j] == -1 && alpha[j] < C);
        if (in_up && (u < 0 || f[j] < fu)) { u = j; fu = f[j]; }
        if (in_low && (l < 0 || f[j] > fl)) { l = j; fl = f[j]; }
    }
    *i_up = u; *i_low = l; *b_up = fu; *b_low = fl;
    return (u >= 0 && l >= 0);
}

int oracle_svm_train_full(const float* X, const int8_t* y, int64_t n, int64_t d, double C,
                          int kernel, double gamma, double tol, int64_t max_iter,
                          const double* alpha0, const double* f0,
                          double* alpha, double* f, double* b_out, int64_t* iters_out,
                          int* converged_out, double* b_up_out, double* b_low_out,
                          int64_t* pair_trace, int64_t trace_cap, int wss, int64_t shrink_window);

/* The SMO solve with working-set rule wss (1: maximal violating pair, S:L197 -- the
 * default reading R1; 2: second-order selection of l above).  The stopping test is the
 * first-order gap in both. */
int oracle_svm_train_wss(const float* X, const int8_t* y, int64_t n, int64_t d, double C,
                         int kernel, double gamma, double tol, int64_t max_iter,
                         const double* alpha0, const double* f0,
                         double* alpha, double* f, double* b_out, int64_t* iters_out,
                         int* converged_out, double* b_up_out, double* b_low_out,
                         int64_t* pair_trace, int64_t trace_cap, int wss) {
    return oracle_svm_train_full(X, y, n, d, C, kernel, gamma, tol, max_iter, alpha0, f0, alpha, f, b_out,
                                 iters_out, converged_out, b_up_out, b_low_out, pair_trace, trace_cap, wss, 0);
}

/* wss as above; shrink_window H > 0 turns on window shrinking (R29), 0 = off. */
int oracle_svm_train_full(const float* X, const int8_t* y, int64_t n, int64_t d, double C,
                          int kernel, double gamma, double tol, int64_t max_iter,
                          const double* alpha0, const double* f0,
                          double* alpha, double* f, double* b_out, int64_t* iters_out,
                          int* converged_out, double* b_up_out, double* b_low_out,
                          int64_t* pair_trace, int64_t trace_cap, int wss, int64_t shrink_window) {
    oracle_init();
    if (n < 2 || d < 1 || !(C > 0.0) || !(tol > 0.0)) return -1;
    if (kernel == ORACLE_RBF && !(gamma > 0.0)) return -1;
    int has_pos = 0, has_neg = 0;
    for (int64_t j = 0; j < n; ++j) {
        if (y[j] == 1) has_pos = 1; else if (y[j] == -1) has_neg = 1; else return -2;
    }
    if (!has_pos || !has_neg) return -3;
    if (max_iter <= 0) max_iter = (10 * n > 10000) ? 10 * n : 10000;

    for (int64_t j = 0; j < n; ++j) {
        alpha[j] = alpha0 ? alpha0[j] : 0.0;
        f[j] = f0 ? f0[j] : -(double)y[j];
    }
    int64_t it = 0;
    int converged = 0;
    double b_up = 0.0, b_low = 0.0;
    uint8_t* active = shrink_window > 0 ? (uint8_t*)malloc((size_t)n) : NULL;
    int64_t window_left = 0;                  /* updates left in the current window (R29) */
    for (;;) {
        int64_t u, l;
        if (!active || window_left == 0) {
            /* every row: the selection, the stopping test, then (R29) the rows set aside */
            if (!oracle_select(f, y, alpha, C, n, &u, &l, &b_up, &b_low)) { converged = 1; break; }
            if (b_low - b_up <= 2.0 * tol) { converged = 1; break; }
            if (it == max_iter) break;
            if (active) { shrink_mark(f, y, alpha, C, n, b_up, b_low, active); window_left = shrink_window; }
        } else {
            /* inside a window: the active rows only; their convergence ends the window */
            if (!select_active(f, y, alpha, C, n, active, &u, &l, &b_up, &b_low) || b_low - b_up <= 2.0 * tol) {
                window_left = 0;
                continue;
            }
            if (it == max_iter) break;
        }
        if (wss == 2) l = select_second_order_masked(X, y, alpha, f, C, n, d, kernel, gamma, u, active);

        const float* xu = X + u * d;
        const float* xl = X + l * d;
        double Kuu = oracle_kernel(kernel, gamma, xu, xu, d, 1);
        double Kll = oracle_kernel(kernel, gamma, xl, xl, d, 1);
        double Kul = oracle_kernel(kernel, gamma, xu, xl, d, u == l);
        double eta = Kuu + Kll - 2.0 * Kul;
        double gap = f[l] - f[u];             /* = b_low - b_up for the first-order pair */
        double yu = (double)y[u], yl = (double)y[l];
        double tu = (y[u] == 1) ? C - alpha[u] : alpha[u];
        double tl = (y[l] == 1) ? alpha[l] : C - alpha[l];
        double t = gap / (eta > 1e-12 ? eta : 1e-12);
        if (tu < t) t = tu;
        if (tl < t) t = tl;
        double au = (t == tu) ? (y[u] == 1 ? C : 0.0) : alpha[u] + yu * t;
        double al = (t == tl) ? (y[l] == 1 ? 0.0 : C) : alpha[l] - yl * t;
        double cu = yu * (au - alpha[u]);
        double cl = yl * (al - alpha[l]);
        alpha[u] = au;
        alpha[l] = al;
        if (pair_trace && it < trace_cap) { pair_trace[2 * it] = u; pair_trace[2 * it + 1] = l; }

        #pragma omp parallel for schedule(static) if (n * d > 65536)
        for (int64_t j = 0; j < n; ++j) {
            double ku = oracle_kernel(kernel, gamma, xu, X + j * d, d, j == u);
            double kl = oracle_kernel(kernel, gamma, xl, X + j * d, d, j == l);
            f[j] = fma(cl, kl, fma(cu, ku, f[j]));
        }
        ++it;
        if (active) --window_left;
    }
    free(active);
    *b_out = -(b_up + b_low) / 2.0;
    *iters_out = it;
    *converged_out = converged;
    *b_up_out = b_up;
    *b_low_out = b_low;
    return 0;
}

/* dec(x) = sum_s coef_s K(x_s, x) + b, coef = alpha * y, ascending s. */
void oracle_decision(const float* Xsv, const double* coef, int64_t nsv, int64_t d, double b,
                     int kernel, double gamma, const float* Xt, int64_t m, double* dec) {
    oracle_init();
    #pragma omp parallel for schedule(static) if (m * nsv * d > 65536)
    for (int64_t i = 0; i < m; ++i) {
        double acc = 0.0;
        for (int64_t s = 0; s < nsv; ++s)
            acc += coef[s] * oracle_kernel(kernel, gamma, Xsv + s * d, Xt + i * d, d, 0);
        dec[i] = acc + b;
    }
}

/* W(alpha) = sum alpha - 1/2 sum_ij alpha_i alpha_j y_i y_j K_ij, O(n^2 d). */
double oracle_dual_objective(const float* X, const int8_t* y, const double* alpha, int64_t n,
                             int64_t d, int kernel, double gamma) {
    oracle_init();
    double lin = 0.0, quad = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        lin += alpha[i];
        if (alpha[i] == 0.0) continue;
        for (int64_t j = 0; j < n; ++j) {
            if (alpha[j] == 0.0) continue;
            quad += alpha[i] * alpha[j] * (double)y[i] * (double)y[j]
                    * oracle_kernel(kernel, gamma, X + i * d, X + j * d, d, i == j);
        }
    }
    return lin - 0.5 * quad;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

int oracle_svm_train(const float* X, const int8_t* y, int64_t n, int64_t d, double C,
                     int kernel, double gamma, double tol, int64_t max_iter,
                     const double* alpha0, const double* f0,
                     double* alpha, double* f, double* b_out, int64_t* iters_out,
                     int* converged_out, double* b_up_out, double* b_low_out,
                     int64_t* pair_trace, int64_t trace_cap) {
    return oracle_svm_train_wss(X, y, n, d, C, kernel, gamma, tol, max_iter, alpha0, f0, alpha, f,
                                b_out, iters_out, converged_out, b_up_out, b_low_out, pair_trace,
                                trace_cap, 1);
}

/* ---------------------------------------------------------------- projected-GD dual trainer
 * The paper's TensorFlow path (§3.3, Fig. 5: "describing the Gaussian RBF kernel
 * function ... declaring the gradient descent optimizer algorithm") read as full-batch
 * projected gradient ascent on the same dual W(alpha) (DESIGN.md
 * readings R23-R26), step by step:
 *   alpha^0 = 0
 *   epoch:  v_j = alpha_j y_j
 *           g_i = sum_j K_ij v_j            (ascending j, one fma per term)       R24
 *           grad_i = 1 - y_i g_i            (dW/dalpha_i)
 *           alpha_i <- min(C, max(0, fma(lr, grad_i, alpha_i)))  (box projection)  R23
 *   after the last epoch g = K (alpha o y) for the final alpha, and
 *   b = mean over {1e-8 < alpha_i < C - 1e-8} of (y_i - g_i)  (ascending i)        R25
 *       else -(max g_i + min g_i)/2 over {alpha_i > 1e-8}, else over all i
 *   W = sum alpha_i - 1/2 sum_i v_i g_i
 * K is the full kernel matrix of oracle_kernel (R13, R14, R16). */
int oracle_gd_train(const float* X, const int8_t* y, int64_t n, int64_t d, double C, int kernel,
                    double gamma, double lr, int64_t epochs, double* alpha, double* g,
                    double* b_out, double* W_out) {
    oracle_init();
    double* K = (double*)malloc((size_t)n * (size_t)n * sizeof(double));
    double* v = (double*)malloc((size_t)n * sizeof(double));
    double* an = (double*)malloc((size_t)n * sizeof(double));
    if (!K || !v || !an) { free(K); free(v); free(an); return -5; }
    #pragma omp parallel for schedule(static) if (n * n * d > 65536)
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j)
            K[i * n + j] = oracle_kernel(kernel, gamma, X + i * d, X + j * d, d, i == j);
    for (int64_t i = 0; i < n; ++i) alpha[i] = 0.0;
    for (int64_t e = 0; e <= epochs; ++e) {
        for (int64_t j = 0; j < n; ++j) v[j] = y[j] > 0 ? alpha[j] : -alpha[j];
        #pragma omp parallel for schedule(static) if (n * n > 65536)
        for (int64_t i = 0; i < n; ++i) {
            double acc = 0.0;
            for (int64_t j = 0; j < n; ++j) acc = fma(K[i * n + j], v[j], acc);
            g[i] = acc;
        }
        if (e == epochs) break;                     /* the final pass only evaluates g */
        for (int64_t i = 0; i < n; ++i) {
            const double grad = 1.0 - (y[i] > 0 ? g[i] : -g[i]);
            double a = fma(lr, grad, alpha[i]);
            if (a < 0.0) a = 0.0;
            if (a > C) a = C;
            an[i] = a;
        }
        for (int64_t i = 0; i < n; ++i) alpha[i] = an[i];
    }
    const double eps = 1e-8;
    double sum = 0.0;
    int64_t cnt = 0;
    for (int64_t i = 0; i < n; ++i)
        if (alpha[i] > eps && alpha[i] < C - eps) { sum += (double)y[i] - g[i]; ++cnt; }
    double b;
    if (cnt > 0) {
        b = sum / (double)cnt;
    } else {
        int any = 0;
        for (int64_t i = 0; i < n; ++i) any |= alpha[i] > eps;
        double mx = -INFINITY, mn = INFINITY;
        for (int64_t i = 0; i < n; ++i)
            if (!any || alpha[i] > eps) { if (g[i] > mx) mx = g[i]; if (g[i] < mn) mn = g[i]; }
        b = -(mx + mn) / 2.0;
    }
    double lin = 0.0, quad = 0.0;
    for (int64_t i = 0; i < n; ++i) { lin += alpha[i]; quad += v[i] * g[i]; }
    *b_out = b;
    *W_out = lin - 0.5 * quad;
    free(K); free(v); free(an);
    return 0;
}
