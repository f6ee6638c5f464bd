/*
 * nurbs_oracle.c — plain, slow, double-precision CPU oracle for the NURBS-Diff hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_2104_14547_b200/) never imports, links or calls it, and shares no code,
 * header, table or constant generator with it.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (NURBS-Diff, arXiv 2104.14547).
 * Readings of garbled / silent passages are the numbered items of DESIGN.md §3
 * (= SURVEY.md §8(c)); they are cited here as "R<k>".
 *
 * Conventions:
 *   n, m   control-point COUNTS in u, v (R6); knot vectors have n+p+1 / m+q+1 entries;
 *          the valid domain is [U[p], U[n]].
 *   ctrl   [B][n][m][4] = (x, y, z, w), Cartesian control points and weights.
 *   out    [B][n_u][n_v][3], u-major (R17).
 *   grad   [B][n][m][4] = (dL/dx, dL/dy, dL/dz, dL/dw).
 *   All arithmetic is IEEE double, no reordering beyond what each cited formula states.
 *
 * Pins: tests/test_oracle_pins.py checks every function below against closed forms,
 * the paper's worked identities, brute force and finite differences. No function here is
 * "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define REF_MAX_DEG 16

enum {
    REF_OK = 0,
    REF_E_ARG = 1,
    REF_E_KNOTS = 3,
    REF_E_DOMAIN = 4,
    REF_E_WEIGHT = 5,
};

/* ------------------------------------------------------------------------------------ */
/* Knot-vector validity: non-decreasing, n > p, non-empty domain U[p] < U[n].    */
/* ------------------------------------------------------------------------------------ */
int nurbs_ref_check_knots(int n, int p, const double* U)
{
    if (p < 0 || p > REF_MAX_DEG || n <= p) return REF_E_ARG;
    for (int k = 0; k + 1 < n + p + 1; ++k)
        if (!(U[k] <= U[k + 1])) return REF_E_KNOTS;      /* P:132 "non-decreasing" */
    if (!(U[p] < U[n])) return REF_E_KNOTS;                /* R6: domain [U[p], U[n]] */
    return REF_OK;
}

/* ------------------------------------------------------------------------------------ */
/* FindSpan — §3.1.2 step 1: the span s with u in [U[s], U[s+1]).                */
/* Piegl–Tiller A2.1 bisection for the largest s in [p, n-1] with U[s] <= u; then the    */
/* right-end rule (R3): if that interval is empty (only possible at u == U[n]) step down */
/* to the last non-empty one, which is treated as closed on the right.                   */
/* Returns -1 if u lies outside [U[p], U[n]] (S:64 domain error).                        */
/* ------------------------------------------------------------------------------------ */
int nurbs_ref_find_span(int n, int p, const double* U, double u)
{
    if (!(u >= U[p] && u <= U[n])) return -1;
    int lo = p, hi = n - 1;                 /* answer in [lo, hi]; U[p] <= u holds */
    while (lo < hi) {
        int mid = (lo + hi + 1) / 2;
        if (U[mid] <= u) lo = mid; else hi = mid - 1;
    }
    int s = lo;
    while (s > p && U[s] == U[s + 1]) --s;  /* R3 / R4 */
    return s;
}

/* ------------------------------------------------------------------------------------ */
/* BasisFuns — §3.1.2 step 2, Cox–de Boor Eq.4 evaluated on the p+1     */
/* non-zero functions N_{s-p..s}^p(u) in the Piegl–Tiller A2.2 triangular order.         */
/* ------------------------------------------------------------------------------------ */
void nurbs_ref_basis_funs(int s, double u, int p, const double* U, double* N)
{
    double left[REF_MAX_DEG + 1], right[REF_MAX_DEG + 1];
    N[0] = 1.0;
    for (int j = 1; j <= p; ++j) {
        left[j] = u - U[s + 1 - j];
        right[j] = U[s + j] - u;
        double saved = 0.0;
        for (int r = 0; r < j; ++r) {
            double temp = N[r] / (right[r + 1] + left[j - r]);
            N[r] = saved + right[r + 1] * temp;
            saved = left[j - r] * temp;
        }
        N[j] = saved;
    }
}

/* ------------------------------------------------------------------------------------ */
/* Dense basis — the literal recursion Eq.4 from Eq.5 for ALL n          */
/* functions, with the half-open degree-0 interval (R2), the right-end rule (R3) and     */
/* 0/0 := 0 (R5). Brute force used only to pin BasisFuns and for the dense Jacobian.     */
/* N_out[0..n-1].                                                                       */
/* ------------------------------------------------------------------------------------ */
void nurbs_ref_basis_dense(int n, int p, const double* U, double u, double* N_out)
{
    int nk = n + p + 1;                 /* number of knots */
    int n0 = nk - 1;                    /* number of degree-0 functions */
    double* N = (double*)calloc((size_t)n0, sizeof(double));
    if (u == U[n]) {
        /* R3: at the right end the last non-empty interval with index <= n-1 is closed */
        int s = n - 1;
        while (s > p && U[s] == U[s + 1]) --s;
        N[s] = 1.0;
    } else {
        for (int i = 0; i < n0; ++i)
            N[i] = (U[i] <= u && u < U[i + 1]) ? 1.0 : 0.0;     /* Eq.5, half-open (R2) */
    }
    for (int k = 1; k <= p; ++k) {
        for (int i = 0; i < n0 - k; ++i) {
            double d1 = U[i + k] - U[i];
            double d2 = U[i + k + 1] - U[i + 1];
            double a = (d1 != 0.0) ? (u - U[i]) / d1 * N[i] : 0.0;          /* R5 */
            double b = (d2 != 0.0) ? (U[i + k + 1] - u) / d2 * N[i + 1] : 0.0;
            N[i] = a + b;                                                    /* Eq.4 */
        }
    }
    for (int i = 0; i < n; ++i) N_out[i] = N[i];
    free(N);
}

/* Spans + local basis for an array of parameters (the per-grid "tape" of Alg.1). */
int nurbs_ref_spans(int n, int p, const double* U, int n_s, const double* s_in,
                    int32_t* span_out, double* N_out /* [n_s][p+1] */)
{
    int st = nurbs_ref_check_knots(n, p, U);
    if (st) return st;
    for (int a = 0; a < n_s; ++a) {
        int s = nurbs_ref_find_span(n, p, U, s_in[a]);
        if (s < 0) return REF_E_DOMAIN;
        span_out[a] = s;
        nurbs_ref_basis_funs(s, s_in[a], p, U, N_out + (size_t)a * (p + 1));
    }
    return REF_OK;
}

static int check_common(int B, int n, int m, int p, int q, int n_u, int n_v, int kb,
                        const double* ctrl, const double* U, const double* V,
                        const double* u, const double* v)
{
    if (B < 0 || n_u < 0 || n_v < 0) return REF_E_ARG;
    int nU = n + p + 1, nV = m + q + 1;
    for (int k = 0; k < (kb ? B : (B > 0 ? 1 : 0)); ++k) {
        int st = nurbs_ref_check_knots(n, p, U + (size_t)k * nU);
        if (st) return st;
        st = nurbs_ref_check_knots(m, q, V + (size_t)k * nV);
        if (st) return st;
        for (int a = 0; a < n_u; ++a)
            if (nurbs_ref_find_span(n, p, U + (size_t)k * nU, u[a]) < 0) return REF_E_DOMAIN;
        for (int b = 0; b < n_v; ++b)
            if (nurbs_ref_find_span(m, q, V + (size_t)k * nV, v[b]) < 0) return REF_E_DOMAIN;
    }
    for (size_t t = 0; t < (size_t)B * n * m; ++t)
        if (!(ctrl[4 * t + 3] > 0.0)) return REF_E_WEIGHT;   /* R15: w > 0 */
    return REF_OK;
}

/* ------------------------------------------------------------------------------------ */
/* Surface forward — Eq.3 (denominator read as the double sum, R1) via §3.1.2     */
/* steps 1-3: homogeneous P^w = (wP, w), S' = sum_r sum_h Nu[r] Nv[h] P^w,   */
/* S = S'_xyz / S'_w. Every point is evaluated independently (Alg.1).          */
/* ------------------------------------------------------------------------------------ */
int nurbs_ref_surface_fwd(int B, int n, int m, int p, int q, int n_u, int n_v, int knots_batched,
                          const double* ctrl, const double* U, const double* V,
                          const double* u, const double* v, double* out)
{
    if (p > REF_MAX_DEG || q > REF_MAX_DEG) return REF_E_ARG;
    int st = check_common(B, n, m, p, q, n_u, n_v, knots_batched, ctrl, U, V, u, v);
    if (st) return st;
    double Nu[REF_MAX_DEG + 1], Nv[REF_MAX_DEG + 1];
    for (int k = 0; k < B; ++k) {
        const double* Uk = U + (knots_batched ? (size_t)k * (n + p + 1) : 0);
        const double* Vk = V + (knots_batched ? (size_t)k * (m + q + 1) : 0);
        const double* Pk = ctrl + (size_t)k * n * m * 4;
        for (int a = 0; a < n_u; ++a) {
            int su = nurbs_ref_find_span(n, p, Uk, u[a]);
            nurbs_ref_basis_funs(su, u[a], p, Uk, Nu);
            for (int b = 0; b < n_v; ++b) {
                int sv = nurbs_ref_find_span(m, q, Vk, v[b]);
                nurbs_ref_basis_funs(sv, v[b], q, Vk, Nv);
                double Sw[4] = {0.0, 0.0, 0.0, 0.0};
                for (int r = 0; r <= p; ++r)
                    for (int h = 0; h <= q; ++h) {
                        const double* P = Pk + ((size_t)(su - p + r) * m + (sv - q + h)) * 4;
                        double Nrh = Nu[r] * Nv[h];
                        Sw[0] += Nrh * (P[3] * P[0]);
                        Sw[1] += Nrh * (P[3] * P[1]);
                        Sw[2] += Nrh * (P[3] * P[2]);
                        Sw[3] += Nrh * P[3];
                    }
                double* o = out + (((size_t)k * n_u + a) * n_v + b) * 3;
                o[0] = Sw[0] / Sw[3];
                o[1] = Sw[1] / Sw[3];
                o[2] = Sw[2] / Sw[3];
            }
        }
    }
    return REF_OK;
}

/* ------------------------------------------------------------------------------------ */
/* Surface backward, Form E — the literal Eq.8 and Eq.9 accumulated over */
/* all points with the upstream factor (R11, "we multiply dL/dS to dS/dPsi"):      */
/*   dL/dP_ij += R_ij * g                 R_ij = N_i N_j w_ij / W        (Eq.8)          */
/*   dL/dw_ij += g . (NR_{,w} W - NR w_{,w}) / W^2,  NR_{,w} = N_i N_j P_ij,             */
/*                                       w_{,w} = N_i N_j                (Eq.9)          */
/* Control index s-p+r (R10), r = 0..p, h = 0..q (R9). Points in row-major (a,b) order.  */
/* Knot gradients are zero by definition (§3.2.2; R14).                           */
/* ------------------------------------------------------------------------------------ */
int nurbs_ref_surface_bwd_eq89(int B, int n, int m, int p, int q, int n_u, int n_v, int knots_batched,
                               const double* ctrl, const double* U, const double* V,
                               const double* u, const double* v, const double* gout,
                               double* grad /* [B][n][m][4] */)
{
    if (p > REF_MAX_DEG || q > REF_MAX_DEG) return REF_E_ARG;
    int st = check_common(B, n, m, p, q, n_u, n_v, knots_batched, ctrl, U, V, u, v);
    if (st) return st;
    memset(grad, 0, sizeof(double) * (size_t)B * n * m * 4);
    double Nu[REF_MAX_DEG + 1], Nv[REF_MAX_DEG + 1];
    for (int k = 0; k < B; ++k) {
        const double* Uk = U + (knots_batched ? (size_t)k * (n + p + 1) : 0);
        const double* Vk = V + (knots_batched ? (size_t)k * (m + q + 1) : 0);
        const double* Pk = ctrl + (size_t)k * n * m * 4;
        double* Gk = grad + (size_t)k * n * m * 4;
        for (int a = 0; a < n_u; ++a) {
            int su = nurbs_ref_find_span(n, p, Uk, u[a]);
            nurbs_ref_basis_funs(su, u[a], p, Uk, Nu);
            for (int b = 0; b < n_v; ++b) {
                int sv = nurbs_ref_find_span(m, q, Vk, v[b]);
                nurbs_ref_basis_funs(sv, v[b], q, Vk, Nv);
                /* NR(u,v) and w(u,v) of Eq.6 */
                double NR[3] = {0.0, 0.0, 0.0}, W = 0.0;
                for (int r = 0; r <= p; ++r)
                    for (int h = 0; h <= q; ++h) {
                        const double* P = Pk + ((size_t)(su - p + r) * m + (sv - q + h)) * 4;
                        double Nrh = Nu[r] * Nv[h];
                        NR[0] += Nrh * P[3] * P[0];
                        NR[1] += Nrh * P[3] * P[1];
                        NR[2] += Nrh * P[3] * P[2];
                        W += Nrh * P[3];
                    }
                const double* g = gout + (((size_t)k * n_u + a) * n_v + b) * 3;
                for (int r = 0; r <= p; ++r)
                    for (int h = 0; h <= q; ++h) {
                        size_t idx = (size_t)(su - p + r) * m + (sv - q + h);
                        const double* P = Pk + idx * 4;
                        double Nrh = Nu[r] * Nv[h];
                        double R = Nrh * P[3] / W;                               /* Eq.8 */
                        double* d = Gk + idx * 4;
                        d[0] += R * g[0];
                        d[1] += R * g[1];
                        d[2] += R * g[2];
                        double dw = 0.0;
                        for (int c = 0; c < 3; ++c) {
                            double NRw = Nrh * P[c];                             /* NR_{,w_ij} */
                            double ww = Nrh;                                     /* w_{,w_ij}  */
                            dw += g[c] * (NRw * W - NR[c] * ww) / (W * W);       /* Eq.9 */
                        }
                        d[3] += dw;
                    }
            }
        }
    }
    return REF_OK;
}

/* ------------------------------------------------------------------------------------ */
/* Surface backward, Form H — the same gradient through the homogeneous point           */
/* Q = (wP, w): with S' = sum N N Q, W = S'_w, S = S'_xyz/W, G = (g/W, -(g.S)/W),        */
/* dQ_ij = sum_pts N_i N_j G, then dP = w dQ_xyz, dw = P.dQ_xyz + dQ_w.                  */
/* Algebraically Eq.8/9; pinned against Form E and finite differences.    */
/* ------------------------------------------------------------------------------------ */
int nurbs_ref_surface_bwd(int B, int n, int m, int p, int q, int n_u, int n_v, int knots_batched,
                          const double* ctrl, const double* U, const double* V,
                          const double* u, const double* v, const double* gout,
                          double* grad /* [B][n][m][4] */)
{
    if (p > REF_MAX_DEG || q > REF_MAX_DEG) return REF_E_ARG;
    int st = check_common(B, n, m, p, q, n_u, n_v, knots_batched, ctrl, U, V, u, v);
    if (st) return st;
    double* dQ = (double*)calloc((size_t)n * m * 4 + 1, sizeof(double));
    double Nu[REF_MAX_DEG + 1], Nv[REF_MAX_DEG + 1];
    for (int k = 0; k < B; ++k) {
        const double* Uk = U + (knots_batched ? (size_t)k * (n + p + 1) : 0);
        const double* Vk = V + (knots_batched ? (size_t)k * (m + q + 1) : 0);
        const double* Pk = ctrl + (size_t)k * n * m * 4;
        memset(dQ, 0, sizeof(double) * (size_t)n * m * 4);
        for (int a = 0; a < n_u; ++a) {
            int su = nurbs_ref_find_span(n, p, Uk, u[a]);
            nurbs_ref_basis_funs(su, u[a], p, Uk, Nu);
            for (int b = 0; b < n_v; ++b) {
                int sv = nurbs_ref_find_span(m, q, Vk, v[b]);
                nurbs_ref_basis_funs(sv, v[b], q, Vk, Nv);
                double Sw[4] = {0.0, 0.0, 0.0, 0.0};
                for (int r = 0; r <= p; ++r)
                    for (int h = 0; h <= q; ++h) {
                        const double* P = Pk + ((size_t)(su - p + r) * m + (sv - q + h)) * 4;
                        double Nrh = Nu[r] * Nv[h];
                        Sw[0] += Nrh * (P[3] * P[0]);
                        Sw[1] += Nrh * (P[3] * P[1]);
                        Sw[2] += Nrh * (P[3] * P[2]);
                        Sw[3] += Nrh * P[3];
                    }
                double W = Sw[3];
                double S[3] = {Sw[0] / W, Sw[1] / W, Sw[2] / W};
                const double* g = gout + (((size_t)k * n_u + a) * n_v + b) * 3;
                double G[4] = {g[0] / W, g[1] / W, g[2] / W,
                               -(g[0] * S[0] + g[1] * S[1] + g[2] * S[2]) / W};
                for (int r = 0; r <= p; ++r)
                    for (int h = 0; h <= q; ++h) {
                        double* d = dQ + ((size_t)(su - p + r) * m + (sv - q + h)) * 4;
                        double Nrh = Nu[r] * Nv[h];
                        for (int c = 0; c < 4; ++c) d[c] += Nrh * G[c];
                    }
            }
        }
        double* Gk = grad + (size_t)k * n * m * 4;
        for (size_t t = 0; t < (size_t)n * m; ++t) {
            const double* P = Pk + t * 4;
            const double* d = dQ + t * 4;
            Gk[t * 4 + 0] = P[3] * d[0];
            Gk[t * 4 + 1] = P[3] * d[1];
            Gk[t * 4 + 2] = P[3] * d[2];
            Gk[t * 4 + 3] = P[0] * d[0] + P[1] * d[1] + P[2] * d[2] + d[3];
        }
    }
    free(dQ);
    return REF_OK;
}

/* ------------------------------------------------------------------------------------ */
/* Selected-control-point backward — Eq.8/9 (Form E) for a list of control points only, */
/* summing over the points where N_i(u_a) N_j(v_b) != 0 (local support). Used   */
/* to check full-size GPU gradients at sampled control points. out4[t] = grad of        */
/* (sel_k[t], sel_i[t], sel_j[t]).                                                      */
/* ------------------------------------------------------------------------------------ */
int nurbs_ref_surface_bwd_selected(int B, int n, int m, int p, int q, int n_u, int n_v, int knots_batched,
                                   const double* ctrl, const double* U, const double* V,
                                   const double* u, const double* v, const double* gout,
                                   int n_sel, const int32_t* sel_k, const int32_t* sel_i,
                                   const int32_t* sel_j, double* out4)
{
    if (p > REF_MAX_DEG || q > REF_MAX_DEG) return REF_E_ARG;
    int st = check_common(B, n, m, p, q, n_u, n_v, knots_batched, ctrl, U, V, u, v);
    if (st) return st;
    int32_t* su = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_u + 1));
    int32_t* sv = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_v + 1));
    double* Nu = (double*)malloc(sizeof(double) * (size_t)(n_u + 1) * (p + 1));
    double* Nv = (double*)malloc(sizeof(double) * (size_t)(n_v + 1) * (q + 1));
    int last_k = -1;
    for (int t = 0; t < n_sel; ++t) {
        int k = sel_k[t], i = sel_i[t], j = sel_j[t];
        const double* Uk = U + (knots_batched ? (size_t)k * (n + p + 1) : 0);
        const double* Vk = V + (knots_batched ? (size_t)k * (m + q + 1) : 0);
        const double* Pk = ctrl + (size_t)k * n * m * 4;
        if (k != last_k) {
            nurbs_ref_spans(n, p, Uk, n_u, u, su, Nu);
            nurbs_ref_spans(m, q, Vk, n_v, v, sv, Nv);
            last_k = k;
        }
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        const double* Pij = Pk + ((size_t)i * m + j) * 4;
        for (int a = 0; a < n_u; ++a) {
            int r = i - (su[a] - p);
            if (r < 0 || r > p) continue;
            for (int b = 0; b < n_v; ++b) {
                int h = j - (sv[b] - q);
                if (h < 0 || h > q) continue;
                const double* Na = Nu + (size_t)a * (p + 1);
                const double* Nb = Nv + (size_t)b * (q + 1);
                double NR[3] = {0.0, 0.0, 0.0}, W = 0.0;
                for (int rr = 0; rr <= p; ++rr)
                    for (int hh = 0; hh <= q; ++hh) {
                        const double* P = Pk + ((size_t)(su[a] - p + rr) * m + (sv[b] - q + hh)) * 4;
                        double Nrh = Na[rr] * Nb[hh];
                        NR[0] += Nrh * P[3] * P[0];
                        NR[1] += Nrh * P[3] * P[1];
                        NR[2] += Nrh * P[3] * P[2];
                        W += Nrh * P[3];
                    }
                const double* g = gout + (((size_t)k * n_u + a) * n_v + b) * 3;
                double Nij = Na[r] * Nb[h];
                double R = Nij * Pij[3] / W;                                     /* Eq.8 */
                acc[0] += R * g[0];
                acc[1] += R * g[1];
                acc[2] += R * g[2];
                for (int c = 0; c < 3; ++c)
                    acc[3] += g[c] * (Nij * Pij[c] * W - NR[c] * Nij) / (W * W); /* Eq.9 */
            }
        }
        for (int c = 0; c < 4; ++c) out4[(size_t)t * 4 + c] = acc[c];
    }
    free(su); free(sv); free(Nu); free(Nv);
    return REF_OK;
}

/* ------------------------------------------------------------------------------------ */
/* Dense forward + dense Jacobian (Eq.10) from the dense basis, for tiny      */
/* inputs. J has n_u*n_v*3 rows and n*m*4 columns; column (i*m+j)*4+c is dS/dP_ij[c]     */
/* for c < 3 (R_ij on the diagonal, Eq.8) and dS/dw_ij for c == 3 (Eq.9).               */
/* One surface (B = 1).                                                                 */
/* ------------------------------------------------------------------------------------ */
int nurbs_ref_surface_dense(int n, int m, int p, int q, int n_u, int n_v,
                            const double* ctrl, const double* U, const double* V,
                            const double* u, const double* v, double* out /* [n_u][n_v][3] */,
                            double* J /* nullable: [n_u*n_v*3][n*m*4] */)
{
    int st = check_common(1, n, m, p, q, n_u, n_v, 0, ctrl, U, V, u, v);
    if (st) return st;
    double* Nu = (double*)malloc(sizeof(double) * (size_t)n);
    double* Nv = (double*)malloc(sizeof(double) * (size_t)m);
    size_t ncol = (size_t)n * m * 4;
    for (int a = 0; a < n_u; ++a) {
        nurbs_ref_basis_dense(n, p, U, u[a], Nu);
        for (int b = 0; b < n_v; ++b) {
            nurbs_ref_basis_dense(m, q, V, v[b], Nv);
            double NR[3] = {0.0, 0.0, 0.0}, W = 0.0;
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < m; ++j) {
                    const double* P = ctrl + ((size_t)i * m + j) * 4;
                    double Nij = Nu[i] * Nv[j];
                    NR[0] += Nij * P[3] * P[0];
                    NR[1] += Nij * P[3] * P[1];
                    NR[2] += Nij * P[3] * P[2];
                    W += Nij * P[3];                                    /* Eq.6 w(u,v) */
                }
            double* o = out + ((size_t)a * n_v + b) * 3;
            for (int c = 0; c < 3; ++c) o[c] = NR[c] / W;               /* Eq.6 S = NR/w */
            if (!J) continue;
            for (int c = 0; c < 3; ++c) {
                double* row = J + (((size_t)a * n_v + b) * 3 + c) * ncol;
                for (int i = 0; i < n; ++i)
                    for (int j = 0; j < m; ++j) {
                        const double* P = ctrl + ((size_t)i * m + j) * 4;
                        double Nij = Nu[i] * Nv[j];
                        size_t col = ((size_t)i * m + j) * 4;
                        row[col + c] = Nij * P[3] / W;                             /* Eq.8 */
                        row[col + 3] = (Nij * P[c] * W - NR[c] * Nij) / (W * W);   /* Eq.9 */
                    }
            }
        }
    }
    free(Nu); free(Nv);
    return REF_OK;
}

/* ------------------------------------------------------------------------------------ */
/* Curves — §3: "directly used for curves ... by suitably adjusting the           */
/* dimensions": C(u) = sum_i N_i w_i P_i / sum_i N_i w_i, ctrl [B][n][4], out [B][n_u][3]. */
/* A 2-D curve uses z = 0 (R18).                                                         */
/* ------------------------------------------------------------------------------------ */
int nurbs_ref_curve_fwd(int B, int n, int p, int n_u, int knots_batched,
                        const double* ctrl, const double* U, const double* u, double* out)
{
    if (p > REF_MAX_DEG || B < 0 || n_u < 0) return REF_E_ARG;
    double N[REF_MAX_DEG + 1];
    for (int k = 0; k < B; ++k) {
        const double* Uk = U + (knots_batched ? (size_t)k * (n + p + 1) : 0);
        if (k == 0 || knots_batched) {
            int st = nurbs_ref_check_knots(n, p, Uk);
            if (st) return st;
        }
        const double* Pk = ctrl + (size_t)k * n * 4;
        for (int t = 0; t < n; ++t) if (!(Pk[4 * t + 3] > 0.0)) return REF_E_WEIGHT;
        for (int a = 0; a < n_u; ++a) {
            int s = nurbs_ref_find_span(n, p, Uk, u[a]);
            if (s < 0) return REF_E_DOMAIN;
            nurbs_ref_basis_funs(s, u[a], p, Uk, N);
            double Cw[4] = {0.0, 0.0, 0.0, 0.0};
            for (int r = 0; r <= p; ++r) {
                const double* P = Pk + (size_t)(s - p + r) * 4;
                Cw[0] += N[r] * (P[3] * P[0]);
                Cw[1] += N[r] * (P[3] * P[1]);
                Cw[2] += N[r] * (P[3] * P[2]);
                Cw[3] += N[r] * P[3];
            }
            double* o = out + ((size_t)k * n_u + a) * 3;
            for (int c = 0; c < 3; ++c) o[c] = Cw[c] / Cw[3];
        }
    }
    return REF_OK;
}

/* Curve backward — Eq.8/9 with the v-direction removed (literal form, as Form E). */
int nurbs_ref_curve_bwd(int B, int n, int p, int n_u, int knots_batched,
                        const double* ctrl, const double* U, const double* u,
                        const double* gout, double* grad /* [B][n][4] */)
{
    if (p > REF_MAX_DEG || B < 0 || n_u < 0) return REF_E_ARG;
    memset(grad, 0, sizeof(double) * (size_t)B * n * 4);
    double N[REF_MAX_DEG + 1];
    for (int k = 0; k < B; ++k) {
        const double* Uk = U + (knots_batched ? (size_t)k * (n + p + 1) : 0);
        if (k == 0 || knots_batched) {
            int st = nurbs_ref_check_knots(n, p, Uk);
            if (st) return st;
        }
        const double* Pk = ctrl + (size_t)k * n * 4;
        double* Gk = grad + (size_t)k * n * 4;
        for (int t = 0; t < n; ++t) if (!(Pk[4 * t + 3] > 0.0)) return REF_E_WEIGHT;
        for (int a = 0; a < n_u; ++a) {
            int s = nurbs_ref_find_span(n, p, Uk, u[a]);
            if (s < 0) return REF_E_DOMAIN;
            nurbs_ref_basis_funs(s, u[a], p, Uk, N);
            double NR[3] = {0.0, 0.0, 0.0}, W = 0.0;
            for (int r = 0; r <= p; ++r) {
                const double* P = Pk + (size_t)(s - p + r) * 4;
                NR[0] += N[r] * P[3] * P[0];
                NR[1] += N[r] * P[3] * P[1];
                NR[2] += N[r] * P[3] * P[2];
                W += N[r] * P[3];
            }
            const double* g = gout + ((size_t)k * n_u + a) * 3;
            for (int r = 0; r <= p; ++r) {
                int i = s - p + r;
                const double* P = Pk + (size_t)i * 4;
                double R = N[r] * P[3] / W;                                      /* Eq.8 */
                double* d = Gk + (size_t)i * 4;
                d[0] += R * g[0];
                d[1] += R * g[1];
                d[2] += R * g[2];
                for (int c = 0; c < 3; ++c)
                    d[3] += g[c] * (N[r] * P[c] * W - NR[c] * N[r]) / (W * W);  /* Eq.9 */
            }
        }
    }
    return REF_OK;
}

/* ------------------------------------------------------------------------------------ */
/* NEXT-3: first derivatives. Basis derivatives by differentiating Eq.4 once:             */
/*   N'_{i,p}(u) = p N_{i,p-1}(u)/(U[i+p]-U[i]) - p N_{i+1,p-1}(u)/(U[i+p+1]-U[i+1])     */
/* (0/0 := 0, R5), from the degree p-1 functions at the same span (Piegl–Tiller Eq.2.7).  */
/* dN[r] = N'_{s-p+r,p}(u), r = 0..p.                                                    */
/* ------------------------------------------------------------------------------------ */
void nurbs_ref_basis_ders1(int s, double u, int p, const double* U, double* dN)
{
    if (p == 0) { dN[0] = 0.0; return; }
    double Nm[REF_MAX_DEG + 1];
    nurbs_ref_basis_funs(s, u, p - 1, U, Nm);  /* N_{s-p+1..s, p-1} */
    for (int r = 0; r <= p; ++r) {
        int i = s - p + r;
        double a = 0.0, b = 0.0;
        if (r >= 1) {
            double d = U[i + p] - U[i];
            a = (d != 0.0) ? Nm[r - 1] / d : 0.0;
        }
        if (r <= p - 1) {
            double d = U[i + p + 1] - U[i + 1];
            b = (d != 0.0) ? Nm[r] / d : 0.0;
        }
        dN[r] = p * (a - b);
    }
}

/* Parametric derivatives, Eq.7 and its v analogue:                  */
/*   S_,u = (NR_,u w - NR w_,u) / w^2,  NR_,u = sum N'_i N_j w P,  w_,u = sum N'_i N_j w   */
/* out/out_u/out_v [B][n_u][n_v][3] (out nullable).                                      */
int nurbs_ref_surface_derivs(int B, int n, int m, int p, int q, int n_u, int n_v, int knots_batched,
                             const double* ctrl, const double* U, const double* V,
                             const double* u, const double* v, double* out, double* out_u, double* out_v)
{
    if (p > REF_MAX_DEG || q > REF_MAX_DEG) return REF_E_ARG;
    int st = check_common(B, n, m, p, q, n_u, n_v, knots_batched, ctrl, U, V, u, v);
    if (st) return st;
    double Nu[REF_MAX_DEG + 1], Nv[REF_MAX_DEG + 1], dNu[REF_MAX_DEG + 1], dNv[REF_MAX_DEG + 1];
    for (int k = 0; k < B; ++k) {
        const double* Uk = U + (knots_batched ? (size_t)k * (n + p + 1) : 0);
        const double* Vk = V + (knots_batched ? (size_t)k * (m + q + 1) : 0);
        const double* Pk = ctrl + (size_t)k * n * m * 4;
        for (int a = 0; a < n_u; ++a) {
            int su = nurbs_ref_find_span(n, p, Uk, u[a]);
            nurbs_ref_basis_funs(su, u[a], p, Uk, Nu);
            nurbs_ref_basis_ders1(su, u[a], p, Uk, dNu);
            for (int b = 0; b < n_v; ++b) {
                int sv = nurbs_ref_find_span(m, q, Vk, v[b]);
                nurbs_ref_basis_funs(sv, v[b], q, Vk, Nv);
                nurbs_ref_basis_ders1(sv, v[b], q, Vk, dNv);
                double NR[3] = {0, 0, 0}, W = 0, NRu[3] = {0, 0, 0}, Wu = 0, NRv[3] = {0, 0, 0}, Wv = 0;
                for (int r = 0; r <= p; ++r)
                    for (int h = 0; h <= q; ++h) {
                        const double* P = Pk + ((size_t)(su - p + r) * m + (sv - q + h)) * 4;
                        double w = P[3];
                        double c0 = Nu[r] * Nv[h], cu = dNu[r] * Nv[h], cv = Nu[r] * dNv[h];
                        for (int c = 0; c < 3; ++c) {
                            NR[c] += c0 * w * P[c];
                            NRu[c] += cu * w * P[c];
                            NRv[c] += cv * w * P[c];
                        }
                        W += c0 * w;
                        Wu += cu * w;
                        Wv += cv * w;
                    }
                size_t o = (((size_t)k * n_u + a) * n_v + b) * 3;
                for (int c = 0; c < 3; ++c) {
                    if (out) out[o + c] = NR[c] / W;
                    out_u[o + c] = (NRu[c] * W - NR[c] * Wu) / (W * W);   /* Eq.7 */
                    out_v[o + c] = (NRv[c] * W - NR[c] * Wv) / (W * W);
                }
            }
        }
    }
    return REF_OK;
}

/* ------------------------------------------------------------------------------------ */
/* NEXT-1: paired (scattered) parameter points. Every point k of surface b carries its   */
/* own (u, v) = uv[b][k] (§3.1: S(u,v) for any (u,v) in the domain; Alg.1's    */
/* per-point span and basis). Same steps as the grid functions above: FindSpan */
/* (A2.1), BasisFuns (A2.2), the rational sum of Eq.3 (R1).         */
/* uv [B][N][2]; out / gout [B][N][3]; grad [B][n][m][4].                               */
/* ------------------------------------------------------------------------------------ */
static int check_points(int B, int n, int m, int p, int q, int N, int kb, const double* ctrl,
                        const double* U, const double* V, const double* uv)
{
    if (B < 0 || N < 0 || p > REF_MAX_DEG || q > REF_MAX_DEG) return REF_E_ARG;
    int nU = n + p + 1, nV = m + q + 1;
    for (int k = 0; k < (kb ? B : (B > 0 ? 1 : 0)); ++k) {
        int st = nurbs_ref_check_knots(n, p, U + (size_t)k * nU);
        if (st) return st;
        st = nurbs_ref_check_knots(m, q, V + (size_t)k * nV);
        if (st) return st;
    }
    for (int k = 0; k < B; ++k) {
        const double* Uk = U + (kb ? (size_t)k * nU : 0);
        const double* Vk = V + (kb ? (size_t)k * nV : 0);
        for (int t = 0; t < N; ++t) {
            const double* x = uv + ((size_t)k * N + t) * 2;
            if (nurbs_ref_find_span(n, p, Uk, x[0]) < 0) return REF_E_DOMAIN;
            if (nurbs_ref_find_span(m, q, Vk, x[1]) < 0) return REF_E_DOMAIN;
        }
    }
    for (size_t t = 0; t < (size_t)B * n * m; ++t)
        if (!(ctrl[4 * t + 3] > 0.0)) return REF_E_WEIGHT;   /* R15 */
    return REF_OK;
}

/* Forward at paired points: Eq.3 via P:138-140, point by point (Alg.1). */
int nurbs_ref_surface_fwd_points(int B, int n, int m, int p, int q, int N, int knots_batched,
                                 const double* ctrl, const double* U, const double* V,
                                 const double* uv, double* out)
{
    int st = check_points(B, n, m, p, q, N, knots_batched, ctrl, U, V, uv);
    if (st) return st;
    double Nu[REF_MAX_DEG + 1], Nv[REF_MAX_DEG + 1];
    for (int k = 0; k < B; ++k) {
        const double* Uk = U + (knots_batched ? (size_t)k * (n + p + 1) : 0);
        const double* Vk = V + (knots_batched ? (size_t)k * (m + q + 1) : 0);
        const double* Pk = ctrl + (size_t)k * n * m * 4;
        for (int t = 0; t < N; ++t) {
            const double u = uv[((size_t)k * N + t) * 2], v = uv[((size_t)k * N + t) * 2 + 1];
            int su = nurbs_ref_find_span(n, p, Uk, u);
            int sv = nurbs_ref_find_span(m, q, Vk, v);
            nurbs_ref_basis_funs(su, u, p, Uk, Nu);
            nurbs_ref_basis_funs(sv, v, q, Vk, Nv);
            double Sw[4] = {0.0, 0.0, 0.0, 0.0};
            for (int r = 0; r <= p; ++r)
                for (int h = 0; h <= q; ++h) {
                    const double* P = Pk + ((size_t)(su - p + r) * m + (sv - q + h)) * 4;
                    double Nrh = Nu[r] * Nv[h];
                    Sw[0] += Nrh * (P[3] * P[0]);
                    Sw[1] += Nrh * (P[3] * P[1]);
                    Sw[2] += Nrh * (P[3] * P[2]);
                    Sw[3] += Nrh * P[3];
                }
            double* o = out + ((size_t)k * N + t) * 3;
            o[0] = Sw[0] / Sw[3];
            o[1] = Sw[1] / Sw[3];
            o[2] = Sw[2] / Sw[3];
        }
    }
    return REF_OK;
}

/* Backward at paired points: the literal Eq.8 / Eq.9 (Form E) with the */
/* upstream factor (R11), accumulated over the points in index order t = 0..N-1.       */
int nurbs_ref_surface_bwd_points(int B, int n, int m, int p, int q, int N, int knots_batched,
                                 const double* ctrl, const double* U, const double* V,
                                 const double* uv, const double* gout, double* grad)
{
    int st = check_points(B, n, m, p, q, N, knots_batched, ctrl, U, V, uv);
    if (st) return st;
    memset(grad, 0, sizeof(double) * (size_t)B * n * m * 4);
    double Nu[REF_MAX_DEG + 1], Nv[REF_MAX_DEG + 1];
    for (int k = 0; k < B; ++k) {
        const double* Uk = U + (knots_batched ? (size_t)k * (n + p + 1) : 0);
        const double* Vk = V + (knots_batched ? (size_t)k * (m + q + 1) : 0);
        const double* Pk = ctrl + (size_t)k * n * m * 4;
        double* Gk = grad + (size_t)k * n * m * 4;
        for (int t = 0; t < N; ++t) {
            const double u = uv[((size_t)k * N + t) * 2], v = uv[((size_t)k * N + t) * 2 + 1];
            int su = nurbs_ref_find_span(n, p, Uk, u);
            int sv = nurbs_ref_find_span(m, q, Vk, v);
            nurbs_ref_basis_funs(su, u, p, Uk, Nu);
            nurbs_ref_basis_funs(sv, v, q, Vk, Nv);
            double NR[3] = {0.0, 0.0, 0.0}, W = 0.0;   /* Eq.6 */
            for (int r = 0; r <= p; ++r)
                for (int h = 0; h <= q; ++h) {
                    const double* P = Pk + ((size_t)(su - p + r) * m + (sv - q + h)) * 4;
                    double Nrh = Nu[r] * Nv[h];
                    NR[0] += Nrh * P[3] * P[0];
                    NR[1] += Nrh * P[3] * P[1];
                    NR[2] += Nrh * P[3] * P[2];
                    W += Nrh * P[3];
                }
            const double* g = gout + ((size_t)k * N + t) * 3;
            for (int r = 0; r <= p; ++r)
                for (int h = 0; h <= q; ++h) {
                    size_t idx = (size_t)(su - p + r) * m + (sv - q + h);
                    const double* P = Pk + idx * 4;
                    double Nrh = Nu[r] * Nv[h];
                    double R = Nrh * P[3] / W;                                   /* Eq.8 */
                    double* d = Gk + idx * 4;
                    d[0] += R * g[0];
                    d[1] += R * g[1];
                    d[2] += R * g[2];
                    double dw = 0.0;
                    for (int c = 0; c < 3; ++c)
                        dw += g[c] * (Nrh * P[c] * W - NR[c] * Nrh) / (W * W);    /* Eq.9 */
                    d[3] += dw;
                }
        }
    }
    return REF_OK;
}

/* ------------------------------------------------------------------------------------ */
/* NEXT-4: true knot gradients (the paper sets them to zero, §3.2.2; this extension */
/* is "parity pinned by FD alone" plus two exact invariants).              */
/* dN_{i,p}(u)/dU[kk] for all i (dense), by differentiating the recursion Eq.4   */
/* with the quotient rule; Eq.5's degree-0 functions are piecewise constant, so their     */
/* knot derivative is 0 (u is never at an interval end the derivative is taken at). With  */
/*   N_{i,k} = a N_{i,k-1} + b N_{i+1,k-1},                                               */
/*   a = (u - U_i)/(U_{i+k} - U_i),  b = (U_{i+k+1} - u)/(U_{i+k+1} - U_{i+1})  (0/0 := 0): */
/*   da/dU_i = (u - U_{i+k})/d1^2,   da/dU_{i+k} = -(u - U_i)/d1^2,                        */
/*   db/dU_{i+1} = (U_{i+k+1} - u)/d2^2,  db/dU_{i+k+1} = (u - U_{i+1})/d2^2.             */
/* dN_out[0..n-1].                                                                       */
/* ------------------------------------------------------------------------------------ */
void nurbs_ref_basis_dknot(int n, int p, const double* U, double u, int kk, double* dN_out)
{
    int nk = n + p + 1, n0 = nk - 1;
    double* N = (double*)calloc((size_t)n0, sizeof(double));
    double* D = (double*)calloc((size_t)n0, sizeof(double));
    if (u == U[n]) {
        int s = n - 1;
        while (s > p && U[s] == U[s + 1]) --s;
        N[s] = 1.0;
    } else {
        for (int i = 0; i < n0; ++i) N[i] = (U[i] <= u && u < U[i + 1]) ? 1.0 : 0.0;
    }
    for (int k = 1; k <= p; ++k) {
        for (int i = 0; i < n0 - k; ++i) {
            double d1 = U[i + k] - U[i], d2 = U[i + k + 1] - U[i + 1];
            double a = 0.0, da = 0.0, b = 0.0, db = 0.0;
            if (d1 != 0.0) {
                a = (u - U[i]) / d1;
                if (kk == i) da += (u - U[i + k]) / (d1 * d1);
                if (kk == i + k) da += -(u - U[i]) / (d1 * d1);
            }
            if (d2 != 0.0) {
                b = (U[i + k + 1] - u) / d2;
                if (kk == i + 1) db += (U[i + k + 1] - u) / (d2 * d2);
                if (kk == i + k + 1) db += (u - U[i + 1]) / (d2 * d2);
            }
            double Nn = a * N[i] + b * N[i + 1];                                   /* Eq.4 */
            double Dn = da * N[i] + a * D[i] + db * N[i + 1] + b * D[i + 1];       /* d/dU_kk */
            N[i] = Nn;
            D[i] = Dn;
        }
    }
    for (int i = 0; i < n; ++i) dN_out[i] = D[i];
    free(N);
    free(D);
}

/* dL/dU, dL/dV for surfaces: dL/dU_kk = sum over points of g . dS/dU_kk with the quotient */
/* rule of Eq.7's form: dS/dU_kk = (dNR W - NR dW) / W^2, where               */
/* NR = sum_ij N_i N_j w_ij P_ij, W = sum_ij N_i N_j w_ij and dNR, dW replace N_i by        */
/* dN_i/dU_kk (all i, j: the literal double sum). Shared knots (knots_batched = 0) give    */
/* one gradient summed over the B surfaces; batched knots one per surface.                */
/* gU [(kb ? B : 1)][n+p+1], gV [(kb ? B : 1)][m+q+1].                                     */
int nurbs_ref_surface_knot_grad(int B, int n, int m, int p, int q, int n_u, int n_v, int knots_batched,
                                const double* ctrl, const double* U, const double* V,
                                const double* u, const double* v, const double* gout,
                                double* gU, double* gV)
{
    if (p > REF_MAX_DEG || q > REF_MAX_DEG) return REF_E_ARG;
    int st = check_common(B, n, m, p, q, n_u, n_v, knots_batched, ctrl, U, V, u, v);
    if (st) return st;
    const int nkU = n + p + 1, nkV = m + q + 1;
    memset(gU, 0, sizeof(double) * (size_t)(knots_batched ? B : 1) * nkU);
    memset(gV, 0, sizeof(double) * (size_t)(knots_batched ? B : 1) * nkV);
    double* Nu = (double*)malloc(sizeof(double) * (size_t)n_u * n);
    double* Nv = (double*)malloc(sizeof(double) * (size_t)n_v * m);
    double* dNu = (double*)malloc(sizeof(double) * (size_t)n_u * n * nkU);
    double* dNv = (double*)malloc(sizeof(double) * (size_t)n_v * m * nkV);
    for (int k = 0; k < B; ++k) {
        const double* Uk = U + (knots_batched ? (size_t)k * nkU : 0);
        const double* Vk = V + (knots_batched ? (size_t)k * nkV : 0);
        const double* Pk = ctrl + (size_t)k * n * m * 4;
        double* gUk = gU + (knots_batched ? (size_t)k * nkU : 0);
        double* gVk = gV + (knots_batched ? (size_t)k * nkV : 0);
        if (k == 0 || knots_batched) {
            for (int a = 0; a < n_u; ++a) {
                nurbs_ref_basis_dense(n, p, Uk, u[a], Nu + (size_t)a * n);
                for (int kk = 0; kk < nkU; ++kk)
                    nurbs_ref_basis_dknot(n, p, Uk, u[a], kk, dNu + ((size_t)a * nkU + kk) * n);
            }
            for (int b = 0; b < n_v; ++b) {
                nurbs_ref_basis_dense(m, q, Vk, v[b], Nv + (size_t)b * m);
                for (int kk = 0; kk < nkV; ++kk)
                    nurbs_ref_basis_dknot(m, q, Vk, v[b], kk, dNv + ((size_t)b * nkV + kk) * m);
            }
        }
        for (int a = 0; a < n_u; ++a)
            for (int b = 0; b < n_v; ++b) {
                const double* g = gout + (((size_t)k * n_u + a) * n_v + b) * 3;
                double NR[3] = {0, 0, 0}, W = 0;
                for (int i = 0; i < n; ++i)
                    for (int j = 0; j < m; ++j) {
                        const double* P = Pk + ((size_t)i * m + j) * 4;
                        double c = Nu[(size_t)a * n + i] * Nv[(size_t)b * m + j] * P[3];
                        NR[0] += c * P[0]; NR[1] += c * P[1]; NR[2] += c * P[2]; W += c;
                    }
                for (int dir = 0; dir < 2; ++dir) {
                    const int nk = dir == 0 ? nkU : nkV;
                    for (int kk = 0; kk < nk; ++kk) {
                        double dNR[3] = {0, 0, 0}, dW = 0;
                        for (int i = 0; i < n; ++i)
                            for (int j = 0; j < m; ++j) {
                                const double* P = Pk + ((size_t)i * m + j) * 4;
                                double c = dir == 0
                                    ? dNu[((size_t)a * nkU + kk) * n + i] * Nv[(size_t)b * m + j] * P[3]
                                    : Nu[(size_t)a * n + i] * dNv[((size_t)b * nkV + kk) * m + j] * P[3];
                                dNR[0] += c * P[0]; dNR[1] += c * P[1]; dNR[2] += c * P[2]; dW += c;
                            }
                        double acc = 0.0;
                        for (int cc = 0; cc < 3; ++cc) acc += g[cc] * (dNR[cc] * W - NR[cc] * dW) / (W * W);
                        (dir == 0 ? gUk : gVk)[kk] += acc;
                    }
                }
            }
    }
    free(Nu); free(Nv); free(dNu); free(dNv);
    return REF_OK;
}

/* Curves: the same with the v-direction removed. gU [(kb ? B : 1)][n+p+1]. */
int nurbs_ref_curve_knot_grad(int B, int n, int p, int n_u, int knots_batched, const double* ctrl,
                              const double* U, const double* u, const double* gout, double* gU)
{
    if (p > REF_MAX_DEG || B < 0 || n_u < 0) return REF_E_ARG;
    const int nk = n + p + 1;
    memset(gU, 0, sizeof(double) * (size_t)(knots_batched ? B : 1) * nk);
    double* N = (double*)malloc(sizeof(double) * (size_t)n);
    double* dN = (double*)malloc(sizeof(double) * (size_t)n);
    for (int k = 0; k < B; ++k) {
        const double* Uk = U + (knots_batched ? (size_t)k * nk : 0);
        if (k == 0 || knots_batched) {
            int st = nurbs_ref_check_knots(n, p, Uk);
            if (st) { free(N); free(dN); return st; }
        }
        const double* Pk = ctrl + (size_t)k * n * 4;
        double* gUk = gU + (knots_batched ? (size_t)k * nk : 0);
        for (int a = 0; a < n_u; ++a) {
            if (nurbs_ref_find_span(n, p, Uk, u[a]) < 0) { free(N); free(dN); return REF_E_DOMAIN; }
            nurbs_ref_basis_dense(n, p, Uk, u[a], N);
            const double* g = gout + ((size_t)k * n_u + a) * 3;
            double NR[3] = {0, 0, 0}, W = 0;
            for (int i = 0; i < n; ++i) {
                const double* P = Pk + (size_t)i * 4;
                double c = N[i] * P[3];
                NR[0] += c * P[0]; NR[1] += c * P[1]; NR[2] += c * P[2]; W += c;
            }
            for (int kk = 0; kk < nk; ++kk) {
                nurbs_ref_basis_dknot(n, p, Uk, u[a], kk, dN);
                double dNR[3] = {0, 0, 0}, dW = 0;
                for (int i = 0; i < n; ++i) {
                    const double* P = Pk + (size_t)i * 4;
                    double c = dN[i] * P[3];
                    dNR[0] += c * P[0]; dNR[1] += c * P[1]; dNR[2] += c * P[2]; dW += c;
                }
                for (int cc = 0; cc < 3; ++cc) gUk[kk] += g[cc] * (dNR[cc] * W - NR[cc] * dW) / (W * W);
            }
        }
    }
    free(N); free(dN);
    return REF_OK;
}
