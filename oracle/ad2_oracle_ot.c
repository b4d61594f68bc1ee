/*
 * ad2_oracle_ot.c — exact optimal transport for the ORACLE (test infrastructure only; see
 * ad2_oracle.c header for the import rule).  "P:n" = /root/reference/PAPER.md line n.
 *
 * Solves the transport LP Eq.primal:
 *     min_{pi >= 0} sum_ij pi_ij c_ij   s.t.  sum_j pi_ij = a_i,  sum_i pi_ij = b_j
 * by the textbook transportation simplex (north-west-corner start, u-v potentials on the
 * basis tree, entering cell by Bland's smallest-index rule, leaving cell = smallest-index
 * minimiser on the cycle, as suggested for anti-cycling by SPEC.md S:73).  The paper used
 * Mosek's transportation simplex; this is an independent textbook restatement.
 * With c_ij = ||x_i - y_j||^2 the optimum is W_2^2.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { int i, j; } cell_t;

/* find the tree path from row node ri to column node cj; nodes: rows 0..ma-1, cols ma..ma+mb-1.
 * Returns number of edges written to path (as basis indices), in order from cj back to ri. */
static int tree_path(int ma, int mb, int nb, const cell_t *basis, int ri, int cj, int *path,
                     int *parent_node, int *parent_edge, int *queue)
{
    int nn = ma + mb;
    for (int v = 0; v < nn; ++v) parent_node[v] = -2;
    int qh = 0, qt = 0;
    queue[qt++] = ri;
    parent_node[ri] = -1;
    int target = ma + cj;
    while (qh < qt) {
        int v = queue[qh++];
        if (v == target) break;
        for (int e = 0; e < nb; ++e) {
            int a = basis[e].i, b = ma + basis[e].j, u;
            if (a == v) u = b;
            else if (b == v) u = a;
            else continue;
            if (parent_node[u] != -2) continue;
            parent_node[u] = v;
            parent_edge[u] = e;
            queue[qt++] = u;
        }
    }
    if (parent_node[target] == -2) return -1;
    int len = 0;
    for (int v = target; v != ri; v = parent_node[v]) path[len++] = parent_edge[v];
    return len;
}

/* returns W = sum c*pi (>= 0), or NAN on failure; plan (ma x mb row-major) may be NULL */
double ad2o_transport(int ma, int mb, const double *a_in, const double *b_in, const double *c,
                      double *plan, int *iters_out)
{
    if (ma < 1 || mb < 1) return NAN;
    int nb = ma + mb - 1;
    double *x = (double *)calloc((size_t)ma * mb, sizeof(double));
    char *isb = (char *)calloc((size_t)ma * mb, 1);
    cell_t *basis = (cell_t *)malloc(sizeof(cell_t) * nb);
    double *ra = (double *)malloc(sizeof(double) * ma);
    double *rb = (double *)malloc(sizeof(double) * mb);
    double *u = (double *)malloc(sizeof(double) * ma);
    double *v = (double *)malloc(sizeof(double) * mb);
    int *path = (int *)malloc(sizeof(int) * (ma + mb));
    int *pn = (int *)malloc(sizeof(int) * (ma + mb));
    int *pe = (int *)malloc(sizeof(int) * (ma + mb));
    int *queue = (int *)malloc(sizeof(int) * (ma + mb));
    char *known_u = (char *)malloc(ma), *known_v = (char *)malloc(mb);
    double cmax = 0.0;
    for (int e = 0; e < ma * mb; ++e) cmax = fmax(cmax, fabs(c[e]));
    double tol = 1e-13 * (cmax > 0 ? cmax : 1.0);

    /* north-west corner: exactly ma+mb-1 basic cells */
    memcpy(ra, a_in, sizeof(double) * ma);
    memcpy(rb, b_in, sizeof(double) * mb);
    {
        int i = 0, j = 0, e = 0;
        for (;;) {
            double q = fmin(ra[i], rb[j]);
            if (q < 0) q = 0;
            x[i * mb + j] = q;
            isb[i * mb + j] = 1;
            basis[e].i = i; basis[e].j = j; ++e;
            int down = ra[i] <= rb[j];
            ra[i] -= q; rb[j] -= q;
            if (i == ma - 1 && j == mb - 1) break;
            if (i == ma - 1) ++j;
            else if (j == mb - 1) ++i;
            else if (down) ++i;
            else ++j;
        }
    }

    int it = 0, ok = 1;
    for (; it < 1000000; ++it) {
        /* potentials: u_i + v_j = c_ij on basic cells, u_0 = 0 */
        memset(known_u, 0, ma); memset(known_v, 0, mb);
        u[0] = 0.0; known_u[0] = 1;
        int changed = 1;
        while (changed) {
            changed = 0;
            for (int e = 0; e < nb; ++e) {
                int i = basis[e].i, j = basis[e].j;
                if (known_u[i] && !known_v[j]) { v[j] = c[i * mb + j] - u[i]; known_v[j] = 1; changed = 1; }
                else if (!known_u[i] && known_v[j]) { u[i] = c[i * mb + j] - v[j]; known_u[i] = 1; changed = 1; }
            }
        }
        /* Bland: first nonbasic cell (row-major index) with negative reduced cost */
        int ie = -1, je = -1;
        for (int i = 0; i < ma && ie < 0; ++i)
            for (int j = 0; j < mb; ++j) {
                if (isb[i * mb + j]) continue;
                if (c[i * mb + j] - u[i] - v[j] < -tol) { ie = i; je = j; break; }
            }
        if (ie < 0) break;                                   /* optimal */
        int len = tree_path(ma, mb, nb, basis, ie, je, path, pn, pe, queue);
        if (len < 0) { ok = 0; break; }
        /* path[0] is the edge at column je: sign -, then alternating */
        double theta = INFINITY;
        int leave = -1;
        for (int s = 0; s < len; s += 2) {
            int e = path[s];
            double xv = x[basis[e].i * mb + basis[e].j];
            int idx = basis[e].i * mb + basis[e].j;
            if (xv < theta || (xv == theta && leave >= 0 &&
                               idx < basis[leave].i * mb + basis[leave].j)) { theta = xv; leave = e; }
        }
        for (int s = 0; s < len; ++s) {
            int e = path[s];
            double *xp = &x[basis[e].i * mb + basis[e].j];
            *xp += (s % 2 == 0) ? -theta : theta;
            if (*xp < 0) *xp = 0;
        }
        isb[basis[leave].i * mb + basis[leave].j] = 0;
        x[basis[leave].i * mb + basis[leave].j] = 0.0;
        basis[leave].i = ie; basis[leave].j = je;
        isb[ie * mb + je] = 1;
        x[ie * mb + je] = theta;
    }
    double W = NAN;
    if (ok) {
        W = 0.0;
        for (int e = 0; e < ma * mb; ++e) W += c[e] * x[e];
        if (plan) memcpy(plan, x, sizeof(double) * ma * mb);
    }
    if (iters_out) *iters_out = it;
    free(x); free(isb); free(basis); free(ra); free(rb); free(u); free(v);
    free(path); free(pn); free(pe); free(queue); free(known_u); free(known_v);
    return W;
}

/* W_2^2 between (xa, wa) (ma x d) and (xb, wb) (mb x d), Eq.primal with c = ||.||^2 */
double ad2o_w2sq(int ma, int mb, int d, const double *xa, const double *wa, const double *xb,
                 const double *wb, double *plan)
{
    double *c = (double *)malloc(sizeof(double) * (size_t)ma * mb);
    for (int i = 0; i < ma; ++i)
        for (int j = 0; j < mb; ++j) {
            double s = 0.0;
            for (int t = 0; t < d; ++t) {
                double df = xa[i * d + t] - xb[j * d + t];
                s += df * df;
            }
            c[i * mb + j] = s;
        }
    double W = ad2o_transport(ma, mb, wa, wb, c, plan, NULL);
    free(c);
    return W;
}

/* Exact objective Eq.centroid: (1/N) sum_k W^2(P, P^(k)) for one cluster */
double ad2o_exact_objective(int m, int d, const double *x, const double *w, int N,
                            const int64_t *off, const double *Y, const double *omega)
{
    double s = 0.0;
    for (int k = 0; k < N; ++k) {
        int mk = (int)(off[k + 1] - off[k]);
        s += ad2o_w2sq(m, mk, d, x, w, Y + off[k] * d, omega + off[k], NULL);
    }
    return s / (double)N;
}

/* Assignment step of AD2-clustering (Alg. 1, reading X13):
 * l^(k) = argmin_c W^2(P_c, P^(k)) by exact OT against EVERY centroid (no pruning), ties to the
 * lowest c.  Centroid weights w_c and member weights are renormalised by their fp64 sums
 * (O1).  best[k] = the minimum W^2, second[k] = the runner-up (gap = second - best; +inf if K = 1).
 * Members are independent: OpenMP over k, no cross-member arithmetic. */
void ad2o_assign(int K, int m, int d, const double *x, const double *w, int N, const int64_t *off,
                 const double *Y, const double *omega, int32_t *labels, double *best, double *second)
{
    double *wn = (double *)malloc(sizeof(double) * (size_t)K * m);
    for (int c = 0; c < K; ++c) {
        double s = 0.0;
        for (int i = 0; i < m; ++i) s += w[c * m + i];
        for (int i = 0; i < m; ++i) wn[c * m + i] = w[c * m + i] / s;
    }
    #pragma omp parallel for schedule(dynamic, 4)
    for (int k = 0; k < N; ++k) {
        const int mk = (int)(off[k + 1] - off[k]);
        double *om = (double *)malloc(sizeof(double) * (size_t)mk);
        double s = 0.0;
        for (int j = 0; j < mk; ++j) s += omega[off[k] + j];
        for (int j = 0; j < mk; ++j) om[j] = omega[off[k] + j] / s;
        double b1 = INFINITY, b2 = INFINITY;
        int lab = -1;
        for (int c = 0; c < K; ++c) {
            double W = ad2o_w2sq(m, mk, d, x + (size_t)c * m * d, wn + (size_t)c * m, Y + off[k] * d, om, NULL);
            if (W < b1) {
                b2 = b1;
                b1 = W;
                lab = c;
            } else if (W < b2) {
                b2 = W;
            }
        }
        labels[k] = lab;
        best[k] = b1;
        second[k] = b2;
        free(om);
    }
    free(wn);
}

/* Centroid initialisation (§V, Eq.merge): from a chosen member's support
 * (y [mk][d], weights w renormalised to sum 1), recursively merge the pair (i, j), i < j,
 * minimising w_i w_j |x_i - x_j|^2 / (w_i + w_j) (first pair in (i, j) order on ties) into
 * x = (w_i x_i + w_j x_j) / (w_i + w_j) with weight w_i + w_j, kept at position i (j removed,
 * the later points move up), until m points remain.  With fewer than m points (reading X19,
 * SPEC's fallback): repeatedly split the heaviest point (first on ties) into two copies of half
 * its weight, the copy appended at the end.  Outputs xout [m][d], wout [m] (sum 1). */
void ad2o_merge(int mk, int d, const double *y, const double *w_in, int m, double *xout, double *wout)
{
    int cap = mk > m ? mk : m;
    double *x = (double *)malloc(sizeof(double) * (size_t)cap * d);
    double *w = (double *)malloc(sizeof(double) * (size_t)cap);
    double s = 0.0;
    for (int j = 0; j < mk; ++j) s += w_in[j];
    for (int j = 0; j < mk; ++j) {
        w[j] = w_in[j] / s;
        for (int t = 0; t < d; ++t) x[j * d + t] = y[j * d + t];
    }
    int n = mk;
    while (n > m) {
        double best = INFINITY;
        int bi = 0, bj = 1;
        for (int i = 0; i < n; ++i)
            for (int j = i + 1; j < n; ++j) {
                double dd = 0.0;
                for (int t = 0; t < d; ++t) {
                    double df = x[i * d + t] - x[j * d + t];
                    dd += df * df;
                }
                double c = w[i] * w[j] * dd / (w[i] + w[j]);
                if (c < best) { best = c; bi = i; bj = j; }
            }
        double wb = w[bi] + w[bj];
        for (int t = 0; t < d; ++t) x[bi * d + t] = (w[bi] * x[bi * d + t] + w[bj] * x[bj * d + t]) / wb;
        w[bi] = wb;
        for (int j = bj; j < n - 1; ++j) {
            w[j] = w[j + 1];
            for (int t = 0; t < d; ++t) x[j * d + t] = x[(j + 1) * d + t];
        }
        --n;
    }
    while (n < m) {
        int h = 0;
        for (int j = 1; j < n; ++j)
            if (w[j] > w[h]) h = j;
        w[h] *= 0.5;
        w[n] = w[h];
        for (int t = 0; t < d; ++t) x[n * d + t] = x[h * d + t];
        ++n;
    }
    double tot = 0.0;
    for (int i = 0; i < m; ++i) tot += w[i];
    for (int i = 0; i < m; ++i) {
        wout[i] = w[i] / tot;
        for (int t = 0; t < d; ++t) xout[i * d + t] = x[i * d + t];
    }
    free(x);
    free(w);
}
