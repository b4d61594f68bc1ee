/*
 * ad2_oracle.c — fp64 CPU ORACLE for the modified B-ADMM barycenter path of
 * AD2-clustering (Ye, Wu, Wang, Li; arXiv 1510.00012).  "P:n" = /root/reference/PAPER.md line n.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code, header,
 * table or helper with the CUDA path (paper_1510_00012_b200/csrc) and never reads its output.
 *
 * Plain and slow on purpose: every function is the paper's formula written out in its own
 * order, in double precision, one member matrix at a time.  Matrices are ROW-MAJOR m x m_k
 * (entry (i,j) at [i*mk + j]), i = centroid support point, j = member support point, the
 * paper's Pi^(k) in R^{m x m_k}.  The only parallelism is an OpenMP loop over
 * members inside a phase, where members are independent; every cross-member
 * sum is serial in member order, so the result does not depend on the thread count.
 *
 * Readings of the paper frozen here:
 *   X1 rho = rho0 * mean over all plan entries of C (the extra 1/N in Eq.rho is a typo)
 *   X2 rho per cluster, computed once from the initial x, fixed through support updates
 *   X3 eps added exactly where Eq.badmmc0b / Eq.badmmc1b add it (default 1e-16)
 *   X4 Eq.badmmc1b uses Lambda^n (before this iteration's dual step)
 *   X5 x update uses Pi^(2), normalised by its actual row mass
 *   X6 support update after every tau completed iterations, never before iteration 1
 *   X12 keep x_i if w_i < 1e-12
 *   X14 surrogate objective with the last Pi^(1) and the current x
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define AD2O_OK 0
#define AD2O_ERR_ARG 1
#define AD2O_ERR_ZERO_RHO 2
#define AD2O_ERR_NONFINITE 3
#define AD2O_ERR_OOM 4

/* ---------------------------------------------------------------------------------------
 * Ground cost.  c(x_i, x_j^(k)) = ||x_i - x_j^(k)||_2^2  (P:239 with p = 2);
 * C(x, x^(k)) = (||x_i - x_j^(k)||^2)_{i,j} in R^{m x m_k}.
 * x: m x d row-major, y: mk x d row-major, C: m x mk row-major.
 * ------------------------------------------------------------------------------------- */
void ad2o_cost(int m, int mk, int d, const double *x, const double *y, double *C)
{
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < mk; ++j) {
            double c = 0.0;
            for (int t = 0; t < d; ++t) {
                double diff = x[i * d + t] - y[j * d + t];
                c += diff * diff;
            }
            C[i * mk + j] = c;
        }
}

/* ---------------------------------------------------------------------------------------
 * Eq.rho, reading X1: rho = rho0 * (sum_k sum_i sum_j c(x_i, x_j^(k))) / (m * n),
 * n = sum_k m_k, i.e. rho0 times the mean plan-entry cost.
 * Returns the sum of costs in *sumC_out (may be NULL).
 * ------------------------------------------------------------------------------------- */
double ad2o_rho(int m, int d, const double *x, int N, const int64_t *off, const double *Y,
                double rho0, double *sumC_out)
{
    double s = 0.0;
    for (int k = 0; k < N; ++k) {
        int mk = (int)(off[k + 1] - off[k]);
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < mk; ++j) {
                double c = 0.0;
                for (int t = 0; t < d; ++t) {
                    double diff = x[i * d + t] - Y[(off[k] + j) * d + t];
                    c += diff * diff;
                }
                s += c;
            }
    }
    if (sumC_out) *sumC_out = s;
    double n = (double)(off[N] - off[0]);
    return rho0 * s / ((double)m * n);
}

/* ---------------------------------------------------------------------------------------
 * Eq.badmmc0b + Eq.badmmc0:
 *   pt_ij   = pi2_ij * exp[ (c_ij + lambda_ij) / (-rho) ] + eps
 *   pi1_ij  = pt_ij / (sum_{l=1..m} pt_lj) * w_j^(k)
 * ------------------------------------------------------------------------------------- */
void ad2o_pi1(int m, int mk, const double *Pi2, const double *Lam, const double *C,
              const double *omega, double rho, double eps, double *Pi1)
{
    double *pt = (double *)malloc(sizeof(double) * (size_t)m * mk);
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < mk; ++j)
            pt[i * mk + j] = Pi2[i * mk + j] * exp((C[i * mk + j] + Lam[i * mk + j]) / (-rho)) + eps;
    for (int j = 0; j < mk; ++j) {
        double colsum = 0.0;
        for (int l = 0; l < m; ++l) colsum += pt[l * mk + j];
        for (int i = 0; i < m; ++i) Pi1[i * mk + j] = pt[i * mk + j] / colsum * omega[j];
    }
    free(pt);
}

/* Eq.badmmc1b: pt1_ij = pi1_ij * exp[ lambda_ij / rho ] + eps   (X4: lambda^n) */
void ad2o_pi1_tilde(int m, int mk, const double *Pi1, const double *Lam, double rho, double eps,
                    double *B)
{
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < mk; ++j)
            B[i * mk + j] = Pi1[i * mk + j] * exp(Lam[i * mk + j] / rho) + eps;
}

/* r_i = sum_{j=1..m_k} pt1_ij ;  wt_i = r_i / sum_i r_i  (normalised row mass) */
void ad2o_rowmass(int m, int mk, const double *B, double *r, double *wt)
{
    double tot = 0.0;
    for (int i = 0; i < m; ++i) {
        double s = 0.0;
        for (int j = 0; j < mk; ++j) s += B[i * mk + j];
        r[i] = s;
        tot += s;
    }
    for (int i = 0; i < m; ++i) wt[i] = r[i] / tot;
}

/* ---------------------------------------------------------------------------------------
 * Consensus over the N members of one cluster, wt: N x m (member-major), members summed in
 * ascending order.
 *   rule 0, (R1) Eq.badmmw: w_i ∝ (1/N) sum_k wt_i^(k),            sum_i w_i = 1
 *   rule 1, (R2) Eq.badmmw2: w_i^(1/2) ∝ (1/N) sum_k (wt_i^(k))^(1/2), sum_i w_i = 1
 * ------------------------------------------------------------------------------------- */
void ad2o_consensus(int N, int m, const double *wt, int rule, double *w)
{
    for (int i = 0; i < m; ++i) {
        double s = 0.0;
        for (int k = 0; k < N; ++k) s += (rule == 1) ? sqrt(wt[(size_t)k * m + i]) : wt[(size_t)k * m + i];
        s /= (double)N;
        w[i] = (rule == 1) ? s * s : s;
    }
    double tot = 0.0;
    for (int i = 0; i < m; ++i) tot += w[i];
    for (int i = 0; i < m; ++i) w[i] /= tot;
}

/* Eq.badmmc1: pi2_ij = pt1_ij / (sum_{l=1..m_k} pt1_il) * w_i */
void ad2o_pi2(int m, int mk, const double *B, const double *w, double *Pi2)
{
    for (int i = 0; i < m; ++i) {
        double rowsum = 0.0;
        for (int l = 0; l < mk; ++l) rowsum += B[i * mk + l];
        for (int j = 0; j < mk; ++j) Pi2[i * mk + j] = B[i * mk + j] / rowsum * w[i];
    }
}

/* Eq.badmm2 / Alg. 4 line: Lambda := Lambda + rho (Pi^(1) - Pi^(2)) */
void ad2o_dual(int m, int mk, double *Lam, const double *Pi1, const double *Pi2, double rho)
{
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < mk; ++j)
            Lam[i * mk + j] = Lam[i * mk + j] + rho * (Pi1[i * mk + j] - Pi2[i * mk + j]);
}

/* ---------------------------------------------------------------------------------------
 * Eq.updatex: x_i := 1/(N w_i) sum_k sum_j pi_ij^(k) x_j^(k), with X5: pi = Pi^(2)
 * whose rows sum to w_i, so N w_i = sum_k sum_j pi_ij^(k) (the actual row mass is used);
 * X12: x_i kept when w_i < 1e-12.  Pi2cat: concatenation of the N member matrices
 * (member k at offset m*off[k], row-major m x m_k).
 * ------------------------------------------------------------------------------------- */
void ad2o_update_support(int m, int d, double *x, const double *w, int N, const int64_t *off,
                         const double *Y, const double *Pi2cat)
{
    for (int i = 0; i < m; ++i) {
        if (w[i] < 1e-12) continue;
        double mass = 0.0;
        double *num = (double *)calloc((size_t)d, sizeof(double));
        for (int k = 0; k < N; ++k) {
            int mk = (int)(off[k + 1] - off[k]);
            const double *P = Pi2cat + (size_t)m * (off[k] - off[0]);
            for (int j = 0; j < mk; ++j) {
                double p = P[i * mk + j];
                mass += p;
                for (int t = 0; t < d; ++t) num[t] += p * Y[(off[k] + j) * d + t];
            }
        }
        for (int t = 0; t < d; ++t) x[i * d + t] = num[t] / mass;
        free(num);
    }
}

/* Surrogate objective (X14): F = (1/N) sum_k <C(x, x^(k)), Pi^(k,1)>,  <A,B> = tr(A B^t) */
double ad2o_surrogate(int m, int d, const double *x, int N, const int64_t *off, const double *Y,
                      const double *Pi1cat)
{
    double s = 0.0;
    for (int k = 0; k < N; ++k) {
        int mk = (int)(off[k + 1] - off[k]);
        double *C = (double *)malloc(sizeof(double) * (size_t)m * mk);
        ad2o_cost(m, mk, d, x, Y + off[k] * d, C);
        const double *P = Pi1cat + (size_t)m * (off[k] - off[0]);
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < mk; ++j) s += C[i * mk + j] * P[i * mk + j];
        free(C);
    }
    return s / (double)N;
}

static int all_finite(const double *v, size_t n)
{
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(v[i])) return 0;
    return 1;
}

/* The iterations of Alg. 4 from the initial Pi2 / Lambda already in place, with C
 * the members' cost matrices.  x != NULL: "Update x per tau loops" (X6) with Eq.updatex
 * and the C rebuild; x == NULL: fixed (symbolic) support, the update is skipped. */
static int alg4_iterations(int m, int N, const int64_t *off, const double *omega, double *C, double *Pi1,
                           double *Pi2, double *Lam, double *B, double *r, double *wt, double *w, int T,
                           int tau, int rule, double rho, double eps, double *x, int d, const double *Y)
{
    int status = AD2O_OK;
    for (int t = 1; t <= T && status == AD2O_OK; ++t) {
        /* for k: Pi^(k,1), pt^(k,1) (Alg. 4) */
#pragma omp parallel for schedule(dynamic, 64)
        for (int k = 0; k < N; ++k) {
            int mk = (int)(off[k + 1] - off[k]);
            size_t b = (size_t)m * off[k];
            ad2o_pi1(m, mk, Pi2 + b, Lam + b, C + b, omega + off[k], rho, eps, Pi1 + b);
            ad2o_pi1_tilde(m, mk, Pi1 + b, Lam + b, rho, eps, B + b);
            ad2o_rowmass(m, mk, B + b, r + (size_t)k * m, wt + (size_t)k * m);
        }
        /* w (Alg. 4) */
        ad2o_consensus(N, m, wt, rule, w);
        /* for k: Pi^(k,2), Lambda^(k) (Alg. 4) */
#pragma omp parallel for schedule(dynamic, 64)
        for (int k = 0; k < N; ++k) {
            int mk = (int)(off[k + 1] - off[k]);
            size_t b = (size_t)m * off[k];
            ad2o_pi2(m, mk, B + b, w, Pi2 + b);
            ad2o_dual(m, mk, Lam + b, Pi1 + b, Pi2 + b, rho);
        }
        if (!all_finite(w, (size_t)m)) status = AD2O_ERR_NONFINITE;
        /* "Update x from Eq.updatex per tau loops", X6: after every tau iterations */
        if (x && t % tau == 0 && status == AD2O_OK) {
            ad2o_update_support(m, d, x, w, N, off, Y, Pi2);
#pragma omp parallel for schedule(dynamic, 64)
            for (int k = 0; k < N; ++k) {
                int mk = (int)(off[k + 1] - off[k]);
                ad2o_cost(m, mk, d, x, Y + off[k] * d, C + (size_t)m * off[k]);
            }
        }
    }
    return status;
}

/* ---------------------------------------------------------------------------------------
 * Algorithm 4 "Centroid Update with B-ADMM" for ONE cluster of N members.
 *
 *   inputs : members (off[N+1], relative or absolute; Y rows off[k]..off[k+1]-1; omega),
 *            centroid x (m x d, in/out), w (m, in/out);
 *            warm: optional Pi^(2) start (concatenated, row-major per member) used for members
 *            with warm_mask[k] != 0, else Pi^(2),0 = w_i w_j^(k).
 *   schedule: T iterations; support update after every tau completed iterations (X6);
 *            rule 0 = R1, 1 = R2; rho0; eps.
 *   outputs: Pi1/Pi2/Lam (concatenated row-major, may be NULL), rho, surrogate objective.
 *   member weights are renormalised to the simplex; |sum-1| > wtol -> ERR_ARG.
 *
 * Alg. 4 body, per iteration:
 *   for k: Pi^(k,1) by Eq.badmmc0b/c0; pt^(k,1) by Eq.badmmc1b
 *   w by Eq.badmmw (R1) or Eq.badmmw2 (R2)
 *   for k: Pi^(k,2) by Eq.badmmc1; Lambda^(k) += rho (Pi^(k,1) - Pi^(k,2))
 * ------------------------------------------------------------------------------------- */
int ad2o_badmm_centroid(int m, int d, int N, const int64_t *off_in, const double *Y_in,
                        const double *omega_in, double *x, double *w,
                        const double *Pi2_warm, const uint8_t *warm_mask,
                        int T, int tau, int rule, double rho0, double eps, double wtol,
                        double *Pi1_out, double *Pi2_out, double *Lam_out,
                        double *rho_out, double *obj_out, int nthreads)
{
    if (m < 1 || d < 1 || N < 1 || T < 0 || tau < 1 || rho0 <= 0.0) return AD2O_ERR_ARG;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    /* relative offsets */
    int64_t *off = (int64_t *)malloc(sizeof(int64_t) * (size_t)(N + 1));
    for (int k = 0; k <= N; ++k) off[k] = off_in[k] - off_in[0];
    const double *Y = Y_in + off_in[0] * d;
    size_t n = (size_t)off[N];
    for (int k = 0; k < N; ++k)
        if (off[k + 1] - off[k] < 1) { free(off); return AD2O_ERR_ARG; }
    size_t E = (size_t)m * n;

    double *omega = (double *)malloc(sizeof(double) * n);
    double *C = (double *)malloc(sizeof(double) * E);
    double *Pi1 = (double *)malloc(sizeof(double) * E);
    double *Pi2 = (double *)malloc(sizeof(double) * E);
    double *Lam = (double *)malloc(sizeof(double) * E);
    double *B = (double *)malloc(sizeof(double) * E);
    double *r = (double *)malloc(sizeof(double) * (size_t)N * m);
    double *wt = (double *)malloc(sizeof(double) * (size_t)N * m);
    if (!omega || !C || !Pi1 || !Pi2 || !Lam || !B || !r || !wt) {
        free(off); free(omega); free(C); free(Pi1); free(Pi2); free(Lam); free(B); free(r); free(wt);
        return AD2O_ERR_OOM;
    }
    int status = AD2O_OK;

    /* O1: member weights on the simplex, renormalised */
    for (int k = 0; k < N && status == AD2O_OK; ++k) {
        double s = 0.0;
        for (int64_t j = off[k]; j < off[k + 1]; ++j) s += omega_in[off_in[0] + j];
        if (!(fabs(s - 1.0) <= wtol)) status = AD2O_ERR_ARG;
        for (int64_t j = off[k]; j < off[k + 1]; ++j) omega[j] = omega_in[off_in[0] + j] / s;
    }

    /* cost matrices C(x, x^(k)) */
#pragma omp parallel for schedule(dynamic, 64)
    for (int k = 0; k < N; ++k) {
        int mk = (int)(off[k + 1] - off[k]);
        ad2o_cost(m, mk, d, x, Y + off[k] * d, C + (size_t)m * off[k]);
    }

    /* Eq.rho with X1, X2: once from the initial x */
    double sumC = 0.0;
    for (size_t e = 0; e < E; ++e) sumC += C[e];
    double rho = rho0 * sumC / ((double)m * (double)n);
    if (rho_out) *rho_out = rho;
    if (status == AD2O_OK && !(rho > 0.0 && isfinite(rho))) status = AD2O_ERR_ZERO_RHO;

    /* Alg. 4 line "Lambda := 0; Pi^(2),0 := Pi" with the P:842-850 initialisation */
    for (int k = 0; k < N; ++k) {
        int mk = (int)(off[k + 1] - off[k]);
        size_t b = (size_t)m * off[k];
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < mk; ++j) {
                Lam[b + i * mk + j] = 0.0;
                if (Pi2_warm && warm_mask && warm_mask[k])
                    Pi2[b + i * mk + j] = Pi2_warm[b + i * mk + j];
                else
                    Pi2[b + i * mk + j] = w[i] * omega[off[k] + j];
                Pi1[b + i * mk + j] = 0.0;
            }
    }

    if (status == AD2O_OK)
        status = alg4_iterations(m, N, off, omega, C, Pi1, Pi2, Lam, B, r, wt, w, T, tau, rule, rho, eps, x, d, Y);
    if (status == AD2O_OK && !all_finite(Pi1, E)) status = AD2O_ERR_NONFINITE;
    if (obj_out) *obj_out = (T > 0) ? ad2o_surrogate(m, d, x, N, off, Y, Pi1) : NAN;
    if (Pi1_out) memcpy(Pi1_out, Pi1, sizeof(double) * E);
    if (Pi2_out) memcpy(Pi2_out, Pi2, sizeof(double) * E);
    if (Lam_out) memcpy(Lam_out, Lam, sizeof(double) * E);
    free(off); free(omega); free(C); free(Pi1); free(Pi2); free(Lam); free(B); free(r); free(wt);
    return status;
}

int ad2o_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Symbolic supports: the support points are symbols of a fixed set with a given
 * symbol-to-symbol cost table D (V x V, row-major, D[a*V + b] = cost of centroid symbol a to
 * member symbol b).  C^(k)_ij = D[xs_i, ys_j]; Alg. 4 runs with the support update skipped
 * (the symbols are fixed).  Otherwise identical to ad2o_badmm_centroid (same O1, Eq.rho X1,
 * initialisation, outputs); the objective is (1/N) sum_k <C^(k), Pi^(k,1)>. */
int ad2o_badmm_table(int m, int N, const int64_t *off_in, const int32_t *ys_in, const double *omega_in,
                     const int32_t *xs, double *w, const double *D, int V, const double *Pi2_warm,
                     const uint8_t *warm_mask, int T, int rule, double rho0, double eps, double wtol,
                     double *Pi1_out, double *Pi2_out, double *Lam_out, double *rho_out, double *obj_out)
{
    if (m < 1 || N < 1 || T < 0 || V < 1 || rho0 <= 0.0) return AD2O_ERR_ARG;
    int64_t *off = (int64_t *)malloc(sizeof(int64_t) * (size_t)(N + 1));
    for (int k = 0; k <= N; ++k) off[k] = off_in[k] - off_in[0];
    const int32_t *ys = ys_in + off_in[0];
    size_t n = (size_t)off[N], E = (size_t)m * n;
    for (int i = 0; i < m; ++i)
        if (xs[i] < 0 || xs[i] >= V) { free(off); return AD2O_ERR_ARG; }
    for (size_t j = 0; j < n; ++j)
        if (ys[j] < 0 || ys[j] >= V) { free(off); return AD2O_ERR_ARG; }
    double *omega = (double *)malloc(sizeof(double) * n);
    double *C = (double *)malloc(sizeof(double) * E);
    double *Pi1 = (double *)calloc(E, sizeof(double));
    double *Pi2 = (double *)malloc(sizeof(double) * E);
    double *Lam = (double *)calloc(E, sizeof(double));
    double *B = (double *)malloc(sizeof(double) * E);
    double *r = (double *)malloc(sizeof(double) * (size_t)N * m);
    double *wt = (double *)malloc(sizeof(double) * (size_t)N * m);
    int status = AD2O_OK;
    for (int k = 0; k < N && status == AD2O_OK; ++k) {
        double s = 0.0;
        for (int64_t j = off[k]; j < off[k + 1]; ++j) s += omega_in[off_in[0] + j];
        if (!(fabs(s - 1.0) <= wtol)) status = AD2O_ERR_ARG;
        for (int64_t j = off[k]; j < off[k + 1]; ++j) omega[j] = omega_in[off_in[0] + j] / s;
    }
    double sumC = 0.0;
    for (int k = 0; k < N; ++k) {
        int mk = (int)(off[k + 1] - off[k]);
        size_t b = (size_t)m * off[k];
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < mk; ++j) {
                C[b + i * mk + j] = D[(size_t)xs[i] * V + ys[off[k] + j]];
                sumC += C[b + i * mk + j];
                Pi2[b + i * mk + j] = (Pi2_warm && warm_mask && warm_mask[k]) ? Pi2_warm[b + i * mk + j]
                                                                              : w[i] * omega[off[k] + j];
            }
    }
    double rho = rho0 * sumC / ((double)m * (double)n);
    if (rho_out) *rho_out = rho;
    if (status == AD2O_OK && !(rho > 0.0 && isfinite(rho))) status = AD2O_ERR_ZERO_RHO;
    if (status == AD2O_OK)
        status = alg4_iterations(m, N, off, omega, C, Pi1, Pi2, Lam, B, r, wt, w, T, 1, rule, rho, eps, NULL, 0, NULL);
    if (status == AD2O_OK && !all_finite(Pi1, E)) status = AD2O_ERR_NONFINITE;
    if (obj_out) {
        double s = 0.0;
        for (size_t e = 0; e < E; ++e) s += C[e] * Pi1[e];
        *obj_out = (T > 0) ? s / (double)N : NAN;
    }
    if (Pi1_out) memcpy(Pi1_out, Pi1, sizeof(double) * E);
    if (Pi2_out) memcpy(Pi2_out, Pi2, sizeof(double) * E);
    if (Lam_out) memcpy(Lam_out, Lam, sizeof(double) * E);
    free(off); free(omega); free(C); free(Pi1); free(Pi2); free(Lam); free(B); free(r); free(wt);
    return status;
}
