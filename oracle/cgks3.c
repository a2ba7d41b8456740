/*
 * cgks3.c -- CPU oracle for the third-order compact gas-kinetic fine operator
 * (§2.3-§3) that the V-cycle
 * uses as the fine-level pre-smoother residual.
 *
 * TEST INFRASTRUCTURE ONLY (same rules as gmg_oracle.c): only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it; it shares no code with the CUDA path and never includes it.
 *
 * Every step follows the paper's order and notation; the parts the paper
 * defers to earlier work (nonlinear weights, collision time, the equilibrium
 * slopes, boundary gradients, the time step) follow the readings C1-C14 of
 * DESIGN.md §12, cited below.  fp64, natural order, no blocking or fusion,
 * built with -ffp-contract=off.
 *
 * Velocity-space moments are evaluated generically: a polynomial in
 * (u1, u2, u3, xi^2) is a list of monomial terms, and the moment of a
 * monomial under a (half-)Maxwellian factorises into 1D Gaussian moments
 * (textbook recurrences).  There are no hand-expanded moment formulas, so a
 * reader can check each flux term against Eqs. (dis1), (dis2), (co) by eye.
 *
 * Pins (tests/test_oracle_cgks3.py, -m "not gpu"): 1D moments vs numerical
 * quadrature; micro-slope solves vs quadrature of <a psi>; GKS flux of equal
 * uniform states = dt * Euler flux (free stream); flux and Gauss-point state
 * vs a brute-force velocity-space + time quadrature of Eqs. (dis1)+(dis2);
 * conservation (side swap) and rotation invariance; p2 exact for quadratic
 * fields; Green-Gauss p1 exact for linear fields on uniform grids;
 * free-stream preservation of the whole residual on every mesh family.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* exported by gmg_oracle.c (same library) */
double orc_df_face(int dim, double gamma, const double *WL, const double *WR, const double *n);
double orc_spectral_radius(int dim, double gamma, double omega, const double *WL, const double *WR, const double *n);
void orc_ghost(int dim, int kind, const double *Wi, const double *Winf, const double *n, double *Wg);

enum { C3_FARFIELD = 0, C3_SLIP = 1, C3_NOSLIP = 2, C3_EXTRAP = 3 };

/* fine level with its high-order geometry (natural order, SoA) */
typedef struct {
    int dim, n_patches, G;       /* G: Gauss slots per face (2 in 2D, 4 in 3D) */
    int64_t n, nf;
    const double *vol;           /* [n] */
    const double *ctr;           /* [dim][n] */
    const double *m2;            /* [nq][n] central second moments (xx, xy, (xz), yy, (yz, zz)) */
    const int64_t *left, *right; /* [nf]; right < 0: -(patch+1) */
    const double *avec;          /* [dim][nf] S n, left -> right */
    const double *gp;            /* [dim][G][nf] Gauss points */
    const double *gw;            /* [G][nf] weights, sum 1 per face */
    const int32_t *patch_kind;
} orc3_mesh;

typedef struct {
    double gamma;
    double cfl_exp;              /* C8: dt_i = CFL_exp V_i / Sigma_i */
    double c1, c2;               /* C9: tau = c1 dt + c2 dt |pl-pr|/(pl+pr) */
    double gam0;                 /* C5: linear weight of the large stencil (gamma_1 = 1 - gam0) */
    double eps;                  /* C5: WENO-Z epsilon */
    int p2min;                   /* C3: p2 needs >= p2min interior neighbours (0: d + 1; C3b: d + 2) */
} orc3_opt;

/* ===================================================================== */
/* small dense solver: Gaussian elimination with partial pivoting          */
/* A [m][m] row major (destroyed), b [m] -> x (in place).  Returns 0 on a   */
/* zero pivot.                                                             */
/* ===================================================================== */
static int solve_dense(int m, double *A, double *b)
{
    for (int k = 0; k < m; ++k) {
        int p = k;
        for (int r = k + 1; r < m; ++r) if (fabs(A[r * m + k]) > fabs(A[p * m + k])) p = r;
        if (A[p * m + k] == 0.0) return 0;
        if (p != k) {
            for (int c = 0; c < m; ++c) { double t = A[k * m + c]; A[k * m + c] = A[p * m + c]; A[p * m + c] = t; }
            double t = b[k]; b[k] = b[p]; b[p] = t;
        }
        for (int r = k + 1; r < m; ++r) {
            double f = A[r * m + k] / A[k * m + k];
            for (int c = k; c < m; ++c) A[r * m + c] -= f * A[k * m + c];
            b[r] -= f * b[k];
        }
    }
    for (int k = m - 1; k >= 0; --k) {
        double s = b[k];
        for (int c = k + 1; c < m; ++c) s -= A[k * m + c] * b[c];
        b[k] = s / A[k * m + k];
    }
    return 1;
}

/* ===================================================================== */
/* Velocity-space polynomials and Maxwellian moments */
/* ===================================================================== */
#define MAXT 512
typedef struct { double c; int e[4]; } term;          /* c u1^e0 u2^e1 u3^e2 (xi^2)^e3 */
typedef struct { int n; term t[MAXT]; } vpoly;

static void vp_zero(vpoly *p) { p->n = 0; }
static void vp_add(vpoly *p, double c, int a, int b, int cc, int d)
{
    if (c == 0.0) return;
    term *t = &p->t[p->n++];
    t->c = c; t->e[0] = a; t->e[1] = b; t->e[2] = cc; t->e[3] = d;
}
/* out = x * y (no combining of like terms: every term kept as written) */
static void vp_mul(const vpoly *x, const vpoly *y, vpoly *out)
{
    vp_zero(out);
    for (int i = 0; i < x->n; ++i)
        for (int j = 0; j < y->n; ++j)
            vp_add(out, x->t[i].c * y->t[j].c, x->t[i].e[0] + y->t[j].e[0], x->t[i].e[1] + y->t[j].e[1],
                   x->t[i].e[2] + y->t[j].e[2], x->t[i].e[3] + y->t[j].e[3]);
}

/* psi_a: (1, u1, u2, [u3,] 1/2 (u1^2 + u2^2 [+ u3^2] + xi^2)) */
static void vp_psi(int dim, int a, vpoly *p)
{
    vp_zero(p);
    int nv = dim + 2;
    if (a == 0) vp_add(p, 1.0, 0, 0, 0, 0);
    else if (a < nv - 1) vp_add(p, 1.0, a == 1, a == 2, a == 3, 0);
    else {
        vp_add(p, 0.5, 2, 0, 0, 0);
        vp_add(p, 0.5, 0, 2, 0, 0);
        if (dim == 3) vp_add(p, 0.5, 0, 0, 2, 0);
        vp_add(p, 0.5, 0, 0, 0, 1);
    }
}

/* s = s_j psi_j: the polynomial of micro-slope coefficients */
static void vp_slope(int dim, const double *s, vpoly *p)
{
    vp_zero(p);
    vpoly q;
    for (int a = 0; a < dim + 2; ++a) {
        vp_psi(dim, a, &q);
        for (int i = 0; i < q.n; ++i) vp_add(p, s[a] * q.t[i].c, q.t[i].e[0], q.t[i].e[1], q.t[i].e[2], q.t[i].e[3]);
    }
}

/* Maxwellian g = rho (lambda/pi)^{(K+D)/2} exp(-lambda(|u-U|^2 + xi^2)),
 * lambda = rho / (2p); 1D moments of the normalised Gaussian:
 *   <u^0> = 1, <u^1> = U, <u^{k+2}> = U <u^{k+1}> + (k+1)/(2 lambda) <u^k>;
 * half range u > 0: <u^0> = erfc(-sqrt(lambda) U)/2,
 *   <u^1> = U <u^0> + exp(-lambda U^2) / (2 sqrt(pi lambda)), same recurrence;
 * u < 0: erfc(+sqrt(lambda) U)/2 and  - exp(...)/(2 sqrt(pi lambda)).
 * internal: <xi^0> = 1, <xi^2> = K/(2 lambda), <xi^4> = (K^2 + 2K)/(4 lambda^2). */
#define NMOM 12
typedef struct {
    double rho, U[3], lambda;
    double Mu[3][NMOM];          /* u1 moments: [0] full, [1] u1 > 0, [2] u1 < 0 */
    double Mv[NMOM], Mw[NMOM], Mxi[3];
} maxw;

static void gauss_moments(double U, double lambda, double m0, double m1, double *M)
{
    M[0] = m0;
    M[1] = m1;
    for (int k = 0; k + 2 < NMOM; ++k) M[k + 2] = U * M[k + 1] + (double)(k + 1) / (2.0 * lambda) * M[k];
}

static double K_internal(int dim, double gamma)
{
    return dim == 3 ? (5.0 - 3.0 * gamma) / (gamma - 1.0) : (4.0 - 2.0 * gamma) / (gamma - 1.0);
}

/* W (conservative, LOCAL frame) -> Maxwellian parameters and moments */
static void maxw_from_W(int dim, double gamma, const double *W, maxw *g)
{
    double rho = W[0], u2 = 0.0;
    g->rho = rho;
    g->U[0] = g->U[1] = g->U[2] = 0.0;
    for (int k = 0; k < dim; ++k) { g->U[k] = W[1 + k] / rho; u2 += g->U[k] * g->U[k]; }
    double p = (gamma - 1.0) * (W[dim + 1] - 0.5 * rho * u2);
    double lam = rho / (2.0 * p);
    g->lambda = lam;
    double U = g->U[0], sl = sqrt(lam);
    double e = exp(-lam * U * U) / (2.0 * sqrt(M_PI * lam));
    gauss_moments(U, lam, 1.0, U, g->Mu[0]);
    double h0 = 0.5 * erfc(-sl * U);
    gauss_moments(U, lam, h0, U * h0 + e, g->Mu[1]);
    double l0 = 0.5 * erfc(sl * U);
    gauss_moments(U, lam, l0, U * l0 - e, g->Mu[2]);
    gauss_moments(g->U[1], lam, 1.0, g->U[1], g->Mv);
    if (dim == 3) gauss_moments(g->U[2], lam, 1.0, g->U[2], g->Mw);
    else { memset(g->Mw, 0, sizeof g->Mw); g->Mw[0] = 1.0; }
    double K = K_internal(dim, gamma);
    g->Mxi[0] = 1.0;
    g->Mxi[1] = K / (2.0 * lam);
    g->Mxi[2] = (K * K + 2.0 * K) / (4.0 * lam * lam);
}

/* normalised moment (1/rho) int p g dXi over range r (0 full, 1 u1>0, 2 u1<0) */
static double moment(const maxw *g, int r, const vpoly *p)
{
    double s = 0.0;
    for (int i = 0; i < p->n; ++i) {
        const term *t = &p->t[i];
        s += t->c * g->Mu[r][t->e[0]] * g->Mv[t->e[1]] * g->Mw[t->e[2]] * g->Mxi[t->e[3]];
    }
    return s;
}

/* <psi_a * X> for a = 0..nv-1 */
static void moment_psi(int dim, const maxw *g, int r, const vpoly *X, double *out)
{
    vpoly q, prod;
    for (int a = 0; a < dim + 2; ++a) {
        vp_psi(dim, a, &q);
        vp_mul(&q, X, &prod);
        out[a] = moment(g, r, &prod);
    }
}

/* Micro-slope solve (Eq.(co)): find s with <s_j psi_j psi_a> = b_a
 * (moment matrix M_ab = <psi_a psi_b>, full range). */
static void micro_solve(int dim, const maxw *g, const double *b, double *s)
{
    int nv = dim + 2;
    double M[25];
    vpoly pa, pb, prod;
    for (int a = 0; a < nv; ++a) {
        vp_psi(dim, a, &pa);
        for (int c = 0; c < nv; ++c) {
            vp_psi(dim, c, &pb);
            vp_mul(&pa, &pb, &prod);
            M[a * nv + c] = moment(g, 0, &prod);
        }
    }
    for (int a = 0; a < nv; ++a) s[a] = b[a];
    solve_dense(nv, M, s);
}

/* sum_e a_e u_e (the spatial part of the expansion, a_e = s_e . psi) */
static void vp_adotu(int dim, const double (*a)[5], vpoly *out)
{
    vp_zero(out);
    vpoly sp, ue, prod;
    for (int e = 0; e < dim; ++e) {
        vp_slope(dim, a[e], &sp);
        vp_zero(&ue);
        vp_add(&ue, 1.0, e == 0, e == 1, e == 2, 0);
        vp_mul(&sp, &ue, &prod);
        for (int i = 0; i < prod.n; ++i) out->t[out->n++] = prod.t[i];
    }
}

/* time-derivative coefficients A from compatibility <A + a_e u_e> = 0
 * (Eq.(co) last line): M A = -<(a.u) psi>. */
static void time_coeffs(int dim, const maxw *g, const double (*a)[5], double *A)
{
    vpoly au;
    double b[5];
    vp_adotu(dim, a, &au);
    moment_psi(dim, g, 0, &au, b);
    for (int q = 0; q < dim + 2; ++q) b[q] = -b[q];
    micro_solve(dim, g, b, A);
}

/* ===================================================================== */
/* Gas-kinetic flux at one Gauss point, LOCAL frame (x1 = face normal)     */
/* (Eqs. (integral1), (dis1), (equli), (compatibility2),        */
/* (dis2), (co); readings C9, C10).                                        */
/* In: W^l, W^r (conservative, local frame), their derivatives             */
/* dW^k[e][q] along the local axes e, dt, tau.                              */
/* Out: F = int_0^dt int u1 psi f dXi dt (time-integrated flux per unit    */
/* area) and Wt = int psi f(dt) dXi.                           */
/* ===================================================================== */
void orc3_gks_local(int dim, double gamma, const double *Wl, const double *dWl, const double *Wr,
                    const double *dWr, double dt, double tau, double *F, double *Wt)
{
    int nv = dim + 2;
    maxw gl, gr, gc;
    maxw_from_W(dim, gamma, Wl, &gl);
    maxw_from_W(dim, gamma, Wr, &gr);

    /* micro slopes a^k_e = M^-1 (dW^k/dx_e)/rho_k and A^k (Eq.(co)) */
    double al[3][5] = {{0}}, ar[3][5] = {{0}}, Al[5], Ar[5];
    for (int e = 0; e < dim; ++e) {
        double bl[5], br[5];
        for (int q = 0; q < nv; ++q) { bl[q] = dWl[e * nv + q] / gl.rho; br[q] = dWr[e * nv + q] / gr.rho; }
        micro_solve(dim, &gl, bl, al[e]);
        micro_solve(dim, &gr, br, ar[e]);
    }
    time_coeffs(dim, &gl, (const double (*)[5])al, Al);
    time_coeffs(dim, &gr, (const double (*)[5])ar, Ar);

    /* W^c (Eq.(compatibility2)): rho_l <psi>_{u>0} + rho_r <psi>_{u<0} */
    vpoly one;
    vp_zero(&one);
    vp_add(&one, 1.0, 0, 0, 0, 0);
    double Wc[5], tl[5], tr[5];
    moment_psi(dim, &gl, 1, &one, tl);
    moment_psi(dim, &gr, 2, &one, tr);
    for (int q = 0; q < nv; ++q) Wc[q] = gl.rho * tl[q] + gr.rho * tr[q];
    maxw_from_W(dim, gamma, Wc, &gc);

    /* equilibrium slopes (reading C10e): dW^c/dx_e = rho_l <a^l_e psi>_{u>0} + rho_r <a^r_e psi>_{u<0} */
    double ac[3][5] = {{0}}, Ac[5];
    for (int e = 0; e < dim; ++e) {
        vpoly sl, sr;
        double b[5];
        vp_slope(dim, al[e], &sl);
        vp_slope(dim, ar[e], &sr);
        moment_psi(dim, &gl, 1, &sl, tl);
        moment_psi(dim, &gr, 2, &sr, tr);
        for (int q = 0; q < nv; ++q) b[q] = (gl.rho * tl[q] + gr.rho * tr[q]) / gc.rho;
        micro_solve(dim, &gc, b, ac[e]);
    }
    time_coeffs(dim, &gc, (const double (*)[5])ac, Ac);

    /* time integrals over [0, dt] of C1, C2, C3 (Eq.(dis2)) and of the
     * kinetic weights e^{-t/tau}, t e^{-t/tau} (Eq.(dis1)) */
    double ex = exp(-dt / tau);
    double q1 = dt - tau * (1.0 - ex);
    double q2 = 2.0 * tau * tau - tau * dt - tau * ex * (dt + 2.0 * tau);
    double q3 = 0.5 * dt * dt - tau * dt + tau * tau * (1.0 - ex);
    double q4 = tau * (1.0 - ex);
    double q5 = tau * tau - tau * ex * (dt + tau);
    /* the same coefficients at t = dt (for W at the Gauss point) */
    double c1 = 1.0 - ex, c2 = (dt + tau) * ex - tau, c3 = dt - tau + tau * ex;

    vpoly u1, acu, Acp, u1acu, u1Ac, alu, Alp, aru, Arp, t1, t2;
    vp_zero(&u1);
    vp_add(&u1, 1.0, 1, 0, 0, 0);
    vp_adotu(dim, (const double (*)[5])ac, &acu);
    vp_slope(dim, Ac, &Acp);
    vp_adotu(dim, (const double (*)[5])al, &alu);
    vp_slope(dim, Al, &Alp);
    vp_adotu(dim, (const double (*)[5])ar, &aru);
    vp_slope(dim, Ar, &Arp);

    double m[5];
    for (int q = 0; q < nv; ++q) { F[q] = 0.0; Wt[q] = 0.0; }
    /* equilibrium part: C1 g^c + C2 a^c_e u_e g^c + C3 A^c g^c */
    moment_psi(dim, &gc, 0, &u1, m);
    for (int q = 0; q < nv; ++q) F[q] += gc.rho * q1 * m[q];
    vp_mul(&u1, &acu, &u1acu);
    moment_psi(dim, &gc, 0, &u1acu, m);
    for (int q = 0; q < nv; ++q) F[q] += gc.rho * q2 * m[q];
    vp_mul(&u1, &Acp, &u1Ac);
    moment_psi(dim, &gc, 0, &u1Ac, m);
    for (int q = 0; q < nv; ++q) F[q] += gc.rho * q3 * m[q];
    moment_psi(dim, &gc, 0, &one, m);
    for (int q = 0; q < nv; ++q) Wt[q] += gc.rho * c1 * m[q];
    moment_psi(dim, &gc, 0, &acu, m);
    for (int q = 0; q < nv; ++q) Wt[q] += gc.rho * c2 * m[q];
    moment_psi(dim, &gc, 0, &Acp, m);
    for (int q = 0; q < nv; ++q) Wt[q] += gc.rho * c3 * m[q];

    /* kinetic part: e^{-t/tau} g^k [1 - tau (a^k_e u_e + A^k) - t a^k_e u_e],
     * k = l on u1 > 0, k = r on u1 < 0 */
    for (int side = 0; side < 2; ++side) {
        const maxw *g = side == 0 ? &gl : &gr;
        int r = side == 0 ? 1 : 2;
        const vpoly *au = side == 0 ? &alu : &aru;
        const vpoly *Ap = side == 0 ? &Alp : &Arp;
        vpoly aupA;                                  /* a.u + A */
        vp_zero(&aupA);
        for (int i = 0; i < au->n; ++i) aupA.t[aupA.n++] = au->t[i];
        for (int i = 0; i < Ap->n; ++i) aupA.t[aupA.n++] = Ap->t[i];
        moment_psi(dim, g, r, &u1, m);
        for (int q = 0; q < nv; ++q) F[q] += g->rho * q4 * m[q];
        vp_mul(&u1, &aupA, &t1);
        moment_psi(dim, g, r, &t1, m);
        for (int q = 0; q < nv; ++q) F[q] -= g->rho * tau * q4 * m[q];
        vp_mul(&u1, au, &t2);
        moment_psi(dim, g, r, &t2, m);
        for (int q = 0; q < nv; ++q) F[q] -= g->rho * q5 * m[q];
        moment_psi(dim, g, r, &one, m);
        for (int q = 0; q < nv; ++q) Wt[q] += g->rho * ex * m[q];
        moment_psi(dim, g, r, &aupA, m);
        for (int q = 0; q < nv; ++q) Wt[q] -= g->rho * ex * tau * m[q];
        moment_psi(dim, g, r, au, m);
        for (int q = 0; q < nv; ++q) Wt[q] -= g->rho * ex * dt * m[q];
    }
}

/* ===================================================================== */
/* Local frame (reading C10a): e_0 = n; 3D: e_1 = normalize(n x x_k) with  */
/* x_k the axis of the smallest |n_k| (first on ties), e_2 = n x e_1;      */
/* 2D: e_1 = (-n_y, n_x).                                                  */
/* ===================================================================== */
static void frame(int dim, const double *n, double E[3][3])
{
    memset(E, 0, sizeof(double) * 9);
    for (int k = 0; k < dim; ++k) E[0][k] = n[k];
    if (dim == 2) { E[1][0] = -n[1]; E[1][1] = n[0]; return; }
    int k = 0;
    for (int j = 1; j < 3; ++j) if (fabs(n[j]) < fabs(n[k])) k = j;
    double x[3] = {0, 0, 0};
    x[k] = 1.0;
    double t[3] = {n[1] * x[2] - n[2] * x[1], n[2] * x[0] - n[0] * x[2], n[0] * x[1] - n[1] * x[0]};
    double tn = sqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
    for (int j = 0; j < 3; ++j) E[1][j] = t[j] / tn;
    E[2][0] = n[1] * E[1][2] - n[2] * E[1][1];
    E[2][1] = n[2] * E[1][0] - n[0] * E[1][2];
    E[2][2] = n[0] * E[1][1] - n[1] * E[1][0];
}

/* global-frame flux through unit normal n: rotate W, dW (q components and
 * derivative directions) into the frame, evaluate, rotate back.
 * dW [d][nv] global (dW[c*nv+q] = dW_q/dx_c). */
void orc3_gks_flux(int dim, double gamma, const double *Wl, const double *dWl, const double *Wr,
                   const double *dWr, const double *n, double dt, double tau, double *F, double *Wt)
{
    int nv = dim + 2;
    double E[3][3];
    frame(dim, n, E);
    double wl[5], wr[5], gl[15], gr[15];
    for (int side = 0; side < 2; ++side) {
        const double *W = side ? Wr : Wl, *dW = side ? dWr : dWl;
        double *w = side ? wr : wl, *g = side ? gr : gl;
        w[0] = W[0];
        w[nv - 1] = W[nv - 1];
        for (int a = 0; a < dim; ++a) {
            w[1 + a] = 0.0;
            for (int d = 0; d < dim; ++d) w[1 + a] += E[a][d] * W[1 + d];
        }
        for (int b = 0; b < dim; ++b) {          /* derivative along e_b */
            double col[5] = {0, 0, 0, 0, 0};     /* global components of d/de_b */
            for (int q = 0; q < nv; ++q)
                for (int c = 0; c < dim; ++c) col[q] += E[b][c] * dW[c * nv + q];
            g[b * nv + 0] = col[0];
            g[b * nv + nv - 1] = col[nv - 1];
            for (int a = 0; a < dim; ++a) {
                g[b * nv + 1 + a] = 0.0;
                for (int d = 0; d < dim; ++d) g[b * nv + 1 + a] += E[a][d] * col[1 + d];
            }
        }
    }
    double Fl[5], Wl_[5];
    orc3_gks_local(dim, gamma, wl, gl, wr, gr, dt, tau, Fl, Wl_);
    F[0] = Fl[0];
    F[nv - 1] = Fl[nv - 1];
    Wt[0] = Wl_[0];
    Wt[nv - 1] = Wl_[nv - 1];
    for (int d = 0; d < dim; ++d) {
        F[1 + d] = 0.0;
        Wt[1 + d] = 0.0;
        for (int a = 0; a < dim; ++a) { F[1 + d] += E[a][d] * Fl[1 + a]; Wt[1 + d] += E[a][d] * Wl_[1 + a]; }
    }
}

/* ===================================================================== */
/* Reconstruction (readings C2-C6)                              */
/* monomials about the cell centroid x0: linear y_e (e < d), quadratic     */
/* y_a y_b (a <= b, row major: xx, xy, (xz,) yy, (yz, zz)) -- the order of  */
/* the m2 components.                                                      */
/* ===================================================================== */
static int nquad(int dim) { return dim * (dim + 1) / 2; }
static void quad_pair(int dim, int k, int *a, int *b)
{
    int idx = 0;
    *a = *b = 0;
    for (int x = 0; x < dim; ++x)
        for (int y = x; y < dim; ++y) { if (idx == k) { *a = x; *b = y; return; } ++idx; }
}

/* per-cell polynomial: p(x) = c0 + sum_e lin[e] y_e + sum_k quad[k] y_a y_b,
 * y = x - x_cell (the final WENO-combined polynomial, reading C5) */
typedef struct { double c0, lin[3], quad[6]; } cpoly;

static double cp_eval(int dim, const cpoly *p, const double *y)
{
    double v = p->c0;
    for (int e = 0; e < dim; ++e) v += p->lin[e] * y[e];
    for (int k = 0; k < nquad(dim); ++k) { int a, b; quad_pair(dim, k, &a, &b); v += p->quad[k] * y[a] * y[b]; }
    return v;
}
static void cp_grad(int dim, const cpoly *p, const double *y, double *gr)
{
    for (int e = 0; e < dim; ++e) gr[e] = p->lin[e];
    for (int k = 0; k < nquad(dim); ++k) {
        int a, b;
        quad_pair(dim, k, &a, &b);
        gr[a] += p->quad[k] * y[b];
        gr[b] += p->quad[k] * y[a];
    }
}

/* cell -> faces, ascending face id */
static void c3_cell_faces(const orc3_mesh *M, int64_t **off_out, int64_t **idx_out)
{
    int64_t *off = calloc((size_t)M->n + 1, sizeof(int64_t));
    for (int64_t f = 0; f < M->nf; ++f) {
        off[M->left[f] + 1]++;
        if (M->right[f] >= 0) off[M->right[f] + 1]++;
    }
    for (int64_t i = 0; i < M->n; ++i) off[i + 1] += off[i];
    int64_t *fill = malloc(sizeof(int64_t) * (size_t)(M->n + 1));
    memcpy(fill, off, sizeof(int64_t) * (size_t)(M->n + 1));
    int64_t *idx = malloc(sizeof(int64_t) * (size_t)(off[M->n] + 1));
    for (int64_t f = 0; f < M->nf; ++f) {
        idx[fill[M->left[f]]++] = f;
        if (M->right[f] >= 0) idx[fill[M->right[f]]++] = f;
    }
    free(fill);
    *off_out = off;
    *idx_out = idx;
}

static double m2_at(const orc3_mesh *M, int64_t i, int a, int b)
{
    if (a > b) { int t = a; a = b; b = t; }
    int k = 0;
    for (int x = 0; x < M->dim; ++x)
        for (int y = x; y < M->dim; ++y) { if (x == a && y == b) return M->m2[(int64_t)k * M->n + i]; ++k; }
    return 0.0;
}

/* C2: p2 of component q of cell i by the constrained least squares of
 * exact averages on the interior von Neumann neighbours m (rows
 * C a = Qm - Q0), least-squares averaged derivatives (rows L a = (Q_e)_m),
 * solved through the KKT system [[2 L^T L, C^T], [C, 0]].  Returns 0 when
 * the cell has fewer than d + 1 interior neighbours (reading C3: p1 only;
 * with d neighbours the averaged-slope rows can leave the Hessian
 * undetermined, e.g. coplanar centroid offsets on structured tets).
 * a = (lin[d], quad[nq]) of p2(x) = Q0 + sum a_k (phi_k(x) - avg_0 phi_k). */
int orc3_p2(const orc3_mesh *M, const int64_t *nb, int nnb, int64_t i, const double *Qbar, const double *Qgrad,
            double *a)
{
    int d = M->dim, nk = d + nquad(d);
    if (nnb < d + 1) return 0;
    int nl = d * nnb, m = nk + nnb;
    double *Cm = calloc((size_t)nnb * nk, sizeof(double)), *L = calloc((size_t)nl * nk, sizeof(double));
    double *q = calloc((size_t)nnb, sizeof(double)), *g = calloc((size_t)nl, sizeof(double));
    for (int r = 0; r < nnb; ++r) {
        int64_t j = nb[r];
        double dl[3];
        for (int e = 0; e < d; ++e) dl[e] = M->ctr[(int64_t)e * M->n + j] - M->ctr[(int64_t)e * M->n + i];
        /* constraint row: avg_m phi_k - avg_0 phi_k */
        for (int e = 0; e < d; ++e) Cm[r * nk + e] = dl[e];
        for (int k = 0; k < nquad(d); ++k) {
            int A, B;
            quad_pair(d, k, &A, &B);
            Cm[r * nk + d + k] = (m2_at(M, j, A, B) + dl[A] * dl[B]) - m2_at(M, i, A, B);
        }
        q[r] = Qbar[j] - Qbar[i];
        /* least-squares rows: avg_m d/dx_e phi_k = (Q_e)_m */
        for (int e = 0; e < d; ++e) {
            double *row = &L[(r * d + e) * nk];
            row[e] = 1.0;
            for (int k = 0; k < nquad(d); ++k) {
                int A, B;
                quad_pair(d, k, &A, &B);
                row[d + k] = (A == e ? dl[B] : 0.0) + (B == e ? dl[A] : 0.0);
            }
            g[r * d + e] = Qgrad[(int64_t)e * M->n + j];
        }
    }
    double *K = calloc((size_t)m * m, sizeof(double)), *rhs = calloc((size_t)m, sizeof(double));
    for (int x = 0; x < nk; ++x) {
        for (int y = 0; y < nk; ++y) {
            double s = 0.0;
            for (int r = 0; r < nl; ++r) s += L[r * nk + x] * L[r * nk + y];
            K[x * m + y] = 2.0 * s;
        }
        double s = 0.0;
        for (int r = 0; r < nl; ++r) s += L[r * nk + x] * g[r];
        rhs[x] = 2.0 * s;
        for (int r = 0; r < nnb; ++r) { K[x * m + nk + r] = Cm[r * nk + x]; K[(nk + r) * m + x] = Cm[r * nk + x]; }
    }
    for (int r = 0; r < nnb; ++r) rhs[nk + r] = q[r];
    int ok = solve_dense(m, K, rhs);
    for (int k = 0; k < nk; ++k) a[k] = rhs[k];
    free(Cm); free(L); free(q); free(g); free(K); free(rhs);
    return ok;
}

/* C6b: a Gauss-point state is admissible if rho > 0 and p > 0; otherwise
 * that side at that point takes the cell average with zero gradient */
static int c3_admissible(int d, double gamma, const double *w)
{
    double m2s = 0.0;
    for (int e = 0; e < d; ++e) m2s += w[1 + e] * w[1 + e];
    double pr = (gamma - 1.0) * (w[d + 1] - 0.5 * m2s / w[0]);
    return w[0] > 0.0 && pr > 0.0;
}

/* ===================================================================== */
/* The fine operator (readings C1-C13):                                    */
/* in: W [nv][n], G [nv][d][n] (cell-averaged slopes), alpha_in [n]        */
/* out: R [nv][n] time-averaged flux sum (A4), Gnew [nv][d][n] the evolved */
/* slopes times DF, alpha [n] DF, Sigma [n] */
/* (first-order, A5/A6), flags [n] (bit 0: p2 used; bit 1 unused)          */
/* unused).  Returns the number of Gauss-point sides that fell back (C6b). */
/* ===================================================================== */
/* C2-C6: the final (WENO-combined, positivity-checked) polynomial of every
 * cell and component: poly [n][nv][1 + d + nq] = (c0, lin[d], quad[nq]) of
 * p(x) = c0 + lin . y + sum_k quad_k y_a y_b, y = x - x_cell.
 * flags [n]: bit 0 p2 used.  Returns 0 (positivity is handled per Gauss
 * point in orc3_residual, reading C6b). */
int64_t orc3_recon(const orc3_mesh *M, const orc3_opt *o, const double *W, const double *G, const double *alpha_in,
                   const double *Winf, double *poly, int32_t *flags)
{
    int d = M->dim, nv = d + 2, nq = nquad(d);
    int64_t n = M->n, nf = M->nf;
    double g0 = o->gam0, g1 = 1.0 - o->gam0;
    int64_t *off, *fidx;
    c3_cell_faces(M, &off, &fidx);
    cpoly *P = calloc((size_t)n * nv, sizeof(cpoly));
    int64_t nfall = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t nb[16];
        int nnb = 0;
        for (int64_t s = off[i]; s < off[i + 1]; ++s) {
            int64_t f = fidx[s];
            if (M->right[f] < 0) continue;
            nb[nnb++] = M->left[f] == i ? M->right[f] : M->left[f];
        }
        double V = M->vol[i];
        int used2 = 0;
        for (int q = 0; q < nv; ++q) {
            const double *Qb = W + (int64_t)q * n;
            /* p1, Green-Gauss with DF; boundary faces take the ghost state (C4) */
            double g1v[3] = {0, 0, 0};
            for (int64_t s = off[i]; s < off[i + 1]; ++s) {
                int64_t f = fidx[s];
                double sg = M->left[f] == i ? 1.0 : -1.0, A[3] = {0, 0, 0}, Sa = 0.0, nn[3] = {0, 0, 0};
                for (int k = 0; k < d; ++k) { A[k] = sg * M->avec[(int64_t)k * nf + f]; Sa += A[k] * A[k]; }
                Sa = sqrt(Sa);
                for (int k = 0; k < d; ++k) nn[k] = A[k] / Sa;
                double Qm;
                if (M->right[f] >= 0) Qm = Qb[M->left[f] == i ? M->right[f] : M->left[f]];
                else {
                    double Wi[5], Wg[5];
                    for (int c = 0; c < nv; ++c) Wi[c] = W[(int64_t)c * n + i];
                    orc_ghost(d, M->patch_kind[-M->right[f] - 1], Wi, Winf, nn, Wg);
                    Qm = Wg[q];
                }
                for (int k = 0; k < d; ++k) g1v[k] += (Qm + Qb[i]) / (2.0 * V) * A[k];
            }
            for (int k = 0; k < d; ++k) g1v[k] *= alpha_in[i];
            cpoly *pp = &P[i * nv + q];
            memset(pp, 0, sizeof *pp);
            double a[9];
            /* C3 / C3b: the compact stencil must hold at least p2min interior neighbours */
            int has2 = nnb >= (o->p2min > 0 ? o->p2min : d + 1) ? orc3_p2(M, nb, nnb, i, Qb, G + (int64_t)q * d * n, a) : 0;
            if (!has2) {                                   /* C3: p1 only */
                pp->c0 = Qb[i];
                for (int k = 0; k < d; ++k) pp->lin[k] = g1v[k];
                continue;
            }
            used2 = 1;
            /* C5: smoothness indicators */
            double Kh[3][3] = {{0}};
            for (int k = 0; k < nq; ++k) {
                int A, B;
                quad_pair(d, k, &A, &B);
                Kh[A][B] += a[d + k];
                Kh[B][A] += a[d + k];
            }
            double grad2 = 0.0;                            /* avg |grad p2|^2 = |a_lin|^2 + tr(K M2 K) */
            for (int e = 0; e < d; ++e) grad2 += a[e] * a[e];
            for (int e = 0; e < d; ++e)
                for (int c = 0; c < d; ++c)
                    for (int c2 = 0; c2 < d; ++c2) grad2 += Kh[e][c] * Kh[e][c2] * m2_at(M, i, c, c2);
            double hess2 = 0.0;                            /* sum over multi-indices |l| = 2 */
            for (int A = 0; A < d; ++A) for (int B = A; B < d; ++B) hess2 += Kh[A][B] * Kh[A][B];
            double beta0 = pow(V, 2.0 / d) * grad2 + pow(V, 4.0 / d) * hess2;
            double gg = 0.0;
            for (int k = 0; k < d; ++k) gg += g1v[k] * g1v[k];
            double beta1 = pow(V, 2.0 / d) * gg;
            double tz = fabs(beta0 - beta1);
            double w0 = g0 * (1.0 + tz / (beta0 + o->eps)), w1 = g1 * (1.0 + tz / (beta1 + o->eps));
            double ws = w0 + w1;
            w0 /= ws;
            w1 /= ws;
            /* p = w0 (p2 - g1 p1)/g0 + w1 p1 */
            double cq = w0 / g0, cl = w1 - w0 * g1 / g0;
            pp->c0 = Qb[i];
            for (int k = 0; k < d; ++k) pp->lin[k] = cq * a[k] + cl * g1v[k];
            for (int k = 0; k < nq; ++k) {
                int A, B;
                quad_pair(d, k, &A, &B);
                pp->quad[k] = cq * a[d + k];
                pp->c0 -= cq * a[d + k] * m2_at(M, i, A, B);
            }
        }
        if (flags) flags[i] = used2;
    }

    int nc = 1 + d + nq;
    for (int64_t i = 0; i < n; ++i)
        for (int q = 0; q < nv; ++q) {
            const cpoly *pp = &P[i * nv + q];
            double *out = poly + (i * nv + q) * nc;
            out[0] = pp->c0;
            for (int e = 0; e < d; ++e) out[1 + e] = pp->lin[e];
            for (int k = 0; k < nq; ++k) out[1 + d + k] = pp->quad[k];
        }
    free(P); free(off); free(fidx);
    return nfall;
}

int64_t orc3_residual(const orc3_mesh *M, const orc3_opt *o, const double *W, const double *G, const double *alpha_in,
                      const double *Winf, double *R, double *Gnew, double *alpha, double *Sigma, int32_t *flags)
{
    int d = M->dim, nv = d + 2, nq = nquad(d), nc = 1 + d + nq;
    int64_t n = M->n, nf = M->nf;
    /* C8: Sigma_i from first-order face spectral radii (A5, A6), dt_i */
    double *dt = malloc(sizeof(double) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) Sigma[i] = 0.0;
    for (int64_t f = 0; f < nf; ++f) {
        int64_t l = M->left[f], r = M->right[f];
        double A[3] = {0, 0, 0}, nn[3] = {0, 0, 0}, S = 0.0, WL[5], WR[5];
        for (int k = 0; k < d; ++k) { A[k] = M->avec[(int64_t)k * nf + f]; S += A[k] * A[k]; }
        S = sqrt(S);
        for (int k = 0; k < d; ++k) nn[k] = A[k] / S;
        for (int q = 0; q < nv; ++q) WL[q] = W[(int64_t)q * n + l];
        if (r >= 0) for (int q = 0; q < nv; ++q) WR[q] = W[(int64_t)q * n + r];
        else orc_ghost(d, M->patch_kind[-r - 1], WL, Winf, nn, WR);
        double rr = orc_spectral_radius(d, o->gamma, 1.0, WL, WR, nn);
        Sigma[l] += S * rr;
        if (r >= 0) Sigma[r] += S * rr;
    }
    for (int64_t i = 0; i < n; ++i) dt[i] = o->cfl_exp * M->vol[i] / Sigma[i];

    double *poly = malloc(sizeof(double) * (size_t)n * nv * nc);
    int64_t nfall = orc3_recon(M, o, W, G, alpha_in, Winf, poly, flags);
    cpoly *P = calloc((size_t)n * nv, sizeof(cpoly));
    for (int64_t i = 0; i < n; ++i)
        for (int q = 0; q < nv; ++q) {
            cpoly *pp = &P[i * nv + q];
            const double *in = poly + (i * nv + q) * nc;
            pp->c0 = in[0];
            for (int e = 0; e < d; ++e) pp->lin[e] = in[1 + e];
            for (int k = 0; k < nq; ++k) pp->quad[k] = in[1 + d + k];
        }
    free(poly);

    /* C7-C13: faces, Gauss points */
    for (int q = 0; q < nv; ++q) for (int64_t i = 0; i < n; ++i) R[(int64_t)q * n + i] = 0.0;
    for (int64_t x = 0; x < (int64_t)nv * d * n; ++x) Gnew[x] = 0.0;
    for (int64_t i = 0; i < n; ++i) alpha[i] = 1.0;
    for (int64_t f = 0; f < nf; ++f) {
        int64_t l = M->left[f], r = M->right[f];
        double A[3] = {0, 0, 0}, nn[3] = {0, 0, 0}, S = 0.0;
        for (int k = 0; k < d; ++k) { A[k] = M->avec[(int64_t)k * nf + f]; S += A[k] * A[k]; }
        S = sqrt(S);
        for (int k = 0; k < d; ++k) nn[k] = A[k] / S;
        double dtf = r >= 0 ? fmin(dt[l], dt[r]) : dt[l];
        double Fs[5] = {0, 0, 0, 0, 0}, Ws[5] = {0, 0, 0, 0, 0}, ap = 1.0;
        for (int k = 0; k < M->G; ++k) {
            double w = M->gw[(int64_t)k * nf + f];
            if (w == 0.0) continue;
            double x[3], yl[3], yr[3], WL[5], WR[5], dWL[15], dWR[15];
            for (int e = 0; e < d; ++e) {
                x[e] = M->gp[((int64_t)e * M->G + k) * nf + f];
                yl[e] = x[e] - M->ctr[(int64_t)e * n + l];
            }
            for (int q = 0; q < nv; ++q) {
                double gr[3];
                WL[q] = cp_eval(d, &P[l * nv + q], yl);
                cp_grad(d, &P[l * nv + q], yl, gr);
                for (int e = 0; e < d; ++e) dWL[e * nv + q] = gr[e];
            }
            if (!c3_admissible(d, o->gamma, WL)) {          /* C6b: this side, this point */
                ++nfall;
                for (int q = 0; q < nv; ++q) WL[q] = W[(int64_t)q * n + l];
                for (int e = 0; e < d * nv; ++e) dWL[e] = 0.0;
            }
            if (r >= 0) {
                for (int e = 0; e < d; ++e) yr[e] = x[e] - M->ctr[(int64_t)e * n + r];
                for (int q = 0; q < nv; ++q) {
                    double gr[3];
                    WR[q] = cp_eval(d, &P[r * nv + q], yr);
                    cp_grad(d, &P[r * nv + q], yr, gr);
                    for (int e = 0; e < d; ++e) dWR[e * nv + q] = gr[e];
                }
                if (!c3_admissible(d, o->gamma, WR)) {
                    ++nfall;
                    for (int q = 0; q < nv; ++q) WR[q] = W[(int64_t)q * n + r];
                    for (int e = 0; e < d * nv; ++e) dWR[e] = 0.0;
                }
            } else {                                       /* C6: ghost value, ghost gradient */
                int kind = M->patch_kind[-r - 1];
                orc_ghost(d, kind, WL, Winf, nn, WR);
                for (int e = 0; e < d * nv; ++e) dWR[e] = kind == C3_EXTRAP ? dWL[e] : 0.0;
            }
            /* C7: DF at the Gauss point */
            ap *= orc_df_face(d, o->gamma, WL, WR, nn);
            /* C9: collision time */
            double m2l = 0.0, m2r = 0.0;
            for (int e = 0; e < d; ++e) { m2l += WL[1 + e] * WL[1 + e]; m2r += WR[1 + e] * WR[1 + e]; }
            double pl = (o->gamma - 1.0) * (WL[nv - 1] - 0.5 * m2l / WL[0]);
            double pr = (o->gamma - 1.0) * (WR[nv - 1] - 0.5 * m2r / WR[0]);
            double tau = o->c1 * dtf + o->c2 * dtf * fabs(pl - pr) / (pl + pr);
            double F[5], Wt[5];
            orc3_gks_flux(d, o->gamma, WL, dWL, WR, dWR, nn, dtf, tau, F, Wt);
            for (int q = 0; q < nv; ++q) { Fs[q] += w * F[q]; Ws[q] += w * Wt[q]; }
        }
        /* C11: time-averaged flux sum; C13: slopes by the divergence theorem */
        for (int q = 0; q < nv; ++q) {
            R[(int64_t)q * n + l] += S * Fs[q] / dtf;
            for (int e = 0; e < d; ++e) Gnew[((int64_t)q * d + e) * n + l] += Ws[q] * A[e];
            if (r >= 0) {
                R[(int64_t)q * n + r] -= S * Fs[q] / dtf;
                for (int e = 0; e < d; ++e) Gnew[((int64_t)q * d + e) * n + r] -= Ws[q] * A[e];
            }
        }
        alpha[l] *= ap;
        if (r >= 0) alpha[r] *= ap;
    }
    for (int q = 0; q < nv; ++q)
        for (int e = 0; e < d; ++e)
            for (int64_t i = 0; i < n; ++i) Gnew[((int64_t)q * d + e) * n + i] *= alpha[i] / M->vol[i];
    free(P); free(dt);
    return nfall;
}
