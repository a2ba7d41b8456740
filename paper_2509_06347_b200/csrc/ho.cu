// ho.cu -- sm_100a kernels of the third-order compact gas-kinetic fine
// operator (§2.3-§3; readings
// C1-C14 of DESIGN.md §12).  FP64.  Four launches per evaluation:
//
//   k_ho_sr     per face   S r_f (first-order spectral radius of the cell averages, A5)
//   k_ho_recon  per cell   Sigma_i, Dt_i, p1 (Green-Gauss x DF), p2 (stored KKT operator x
//                          neighbour averages and slopes), WENO-Z weights, positivity check
//                          -> one polynomial per cell and component
//   k_ho_flux   per face   at every Gauss point: both sides' polynomial values and gradients,
//                          DF, collision time, the BGK flux (Eqs. (dis1), (dis2)) integrated over
//                          Dt_f and the Gauss-point state at Dt_f  -> one face record
//   k_ho_gather per cell   R_i, the evolved slopes, DF; update / restriction outputs
//
// The BGK flux is FP64-ALU bound (moments up to 6th order of three
// Maxwellians, four 5x5 moment solves per Gauss point); the other three are
// gather/stream kernels.  Velocity moments use per-Maxwellian 1D moment
// arrays and compile-time moment indices (everything stays in registers).
#include <cuda_runtime.h>

#include "device_common.cuh"

namespace gmg {

constexpr int kHoRec = 12;

// ------------------------------------------------------------------ moments
// normalised Maxwellian: Mu (full), Mp (u1 > 0), Mm (u1 < 0), Mv, Mw, <xi^2>, <xi^4>
template <int D>
struct Maxw {
    double rho, lam;
    double Mu[7], Mp[7], Mm[7], Mv[6], Mw[6];
    double x1, x2;
};

__device__ __forceinline__ void rec_mom(double U, double inv2l, double *M, int n)
{
#pragma unroll
    for (int k = 2; k < 7; ++k)
        if (k < n) M[k] = U * M[k - 1] + (double)(k - 1) * inv2l * M[k - 2];
}

template <int D>
__device__ __forceinline__ void maxw(const double *w, double gm1, double K, Maxw<D> &g)
{
    g.rho = w[0];
    const double ir = 1.0 / w[0];
    double U[3] = {0, 0, 0}, u2 = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) { U[k] = w[1 + k] * ir; u2 += U[k] * U[k]; }
    const double p = gm1 * (w[D + 1] - 0.5 * w[0] * u2);
    const double lam = 0.5 * w[0] / p;
    const double inv2l = p * ir;                       // 1/(2 lambda)
    g.lam = lam;
    const double sl = sqrt(lam);
    const double e = exp(-lam * U[0] * U[0]) * (0.28209479177387814 / sl);   // e^{-l U^2} / (2 sqrt(pi l))
    g.Mu[0] = 1.0; g.Mu[1] = U[0];
    g.Mp[0] = 0.5 * erfc(-sl * U[0]); g.Mp[1] = U[0] * g.Mp[0] + e;
    g.Mm[0] = 0.5 * erfc(sl * U[0]);  g.Mm[1] = U[0] * g.Mm[0] - e;
    rec_mom(U[0], inv2l, g.Mu, 7);
    rec_mom(U[0], inv2l, g.Mp, 7);
    rec_mom(U[0], inv2l, g.Mm, 7);
    g.Mv[0] = 1.0; g.Mv[1] = U[1];
    rec_mom(U[1], inv2l, g.Mv, 6);
    if constexpr (D == 3) { g.Mw[0] = 1.0; g.Mw[1] = U[2]; rec_mom(U[2], inv2l, g.Mw, 6); }
    g.x1 = K * inv2l;
    g.x2 = (K * K + 2.0 * K) * inv2l * inv2l;
}

// <u^a v^b w^c psi> with the u1 moments of range R (0 full, 1 >0, 2 <0)
template <int D, int R>
__device__ __forceinline__ const double *umom(const Maxw<D> &g) { return R == 0 ? g.Mu : (R == 1 ? g.Mp : g.Mm); }

template <int D, int R, int a, int b, int c>
__device__ __forceinline__ void psi_m(const Maxw<D> &g, double *o)
{
    const double *Mu = umom<D, R>(g);
    const double wc = D == 3 ? g.Mw[c] : 1.0;
    const double base = Mu[a] * g.Mv[b] * wc;
    o[0] = base;
    o[1] = Mu[a + 1] * g.Mv[b] * wc;
    o[2] = Mu[a] * g.Mv[b + 1] * wc;
    if constexpr (D == 3) {
        o[3] = Mu[a] * g.Mv[b] * g.Mw[c + 1];
        o[D + 1] = 0.5 * (Mu[a + 2] * g.Mv[b] * wc + Mu[a] * g.Mv[b + 2] * wc + Mu[a] * g.Mv[b] * g.Mw[c + 2] + g.x1 * base);
    } else {
        o[D + 1] = 0.5 * (Mu[a + 2] * g.Mv[b] + Mu[a] * g.Mv[b + 2] + g.x1 * base);
    }
}
// <xi^2 u^a v^b w^c psi>
template <int D, int R, int a, int b, int c>
__device__ __forceinline__ void psi_xi(const Maxw<D> &g, double *o)
{
    const double *Mu = umom<D, R>(g);
    const double wc = D == 3 ? g.Mw[c] : 1.0;
    const double base = Mu[a] * g.Mv[b] * wc;
    o[0] = g.x1 * base;
    o[1] = g.x1 * Mu[a + 1] * g.Mv[b] * wc;
    o[2] = g.x1 * Mu[a] * g.Mv[b + 1] * wc;
    if constexpr (D == 3) {
        o[3] = g.x1 * Mu[a] * g.Mv[b] * g.Mw[c + 1];
        o[D + 1] = 0.5 * (g.x1 * (Mu[a + 2] * g.Mv[b] * wc + Mu[a] * g.Mv[b + 2] * wc + Mu[a] * g.Mv[b] * g.Mw[c + 2]) +
                          g.x2 * base);
    } else {
        o[D + 1] = 0.5 * (g.x1 * (Mu[a + 2] * g.Mv[b] + Mu[a] * g.Mv[b + 2]) + g.x2 * base);
    }
}
// <(s . psi) u^a v^b w^c psi>
template <int D, int R, int a, int b, int c>
__device__ __forceinline__ void apsi(const Maxw<D> &g, const double *s, double *o)
{
    constexpr int NV = D + 2;
    double t[NV];
    psi_m<D, R, a, b, c>(g, t);
#pragma unroll
    for (int q = 0; q < NV; ++q) o[q] = s[0] * t[q];
    psi_m<D, R, a + 1, b, c>(g, t);
#pragma unroll
    for (int q = 0; q < NV; ++q) o[q] += s[1] * t[q];
    psi_m<D, R, a, b + 1, c>(g, t);
#pragma unroll
    for (int q = 0; q < NV; ++q) o[q] += s[2] * t[q];
    if constexpr (D == 3) {
        psi_m<D, R, a, b, c + 1>(g, t);
#pragma unroll
        for (int q = 0; q < NV; ++q) o[q] += s[3] * t[q];
    }
    const double h = 0.5 * s[D + 1];
    psi_m<D, R, a + 2, b, c>(g, t);
#pragma unroll
    for (int q = 0; q < NV; ++q) o[q] += h * t[q];
    psi_m<D, R, a, b + 2, c>(g, t);
#pragma unroll
    for (int q = 0; q < NV; ++q) o[q] += h * t[q];
    if constexpr (D == 3) {
        psi_m<D, R, a, b, c + 2>(g, t);
#pragma unroll
        for (int q = 0; q < NV; ++q) o[q] += h * t[q];
    }
    psi_xi<D, R, a, b, c>(g, t);
#pragma unroll
    for (int q = 0; q < NV; ++q) o[q] += h * t[q];
}
// sum_e <u_e (s_e . psi) u^a psi>: direction e adds one power of u / v / w
template <int D, int R, int a>
__device__ __forceinline__ void adotu(const Maxw<D> &g, const double (*s)[D + 2], double *o)
{
    constexpr int NV = D + 2;
    double t[NV];
    apsi<D, R, a + 1, 0, 0>(g, s[0], o);
    apsi<D, R, a, 1, 0>(g, s[1], t);
#pragma unroll
    for (int q = 0; q < NV; ++q) o[q] += t[q];
    if constexpr (D == 3) {
        apsi<D, R, a, 0, 1>(g, s[D - 1], t);
#pragma unroll
        for (int q = 0; q < NV; ++q) o[q] += t[q];
    }
}

// moment matrix M_ab = <psi_a psi_b> (full range), factored without pivoting
// (symmetric positive definite): L D L^T in place
template <int D>
__device__ __forceinline__ void mfactor(const Maxw<D> &g, double (*M)[D + 2])
{
    constexpr int NV = D + 2;
    double c[NV];
    psi_m<D, 0, 0, 0, 0>(g, c);
#pragma unroll
    for (int q = 0; q < NV; ++q) M[q][0] = c[q];
    psi_m<D, 0, 1, 0, 0>(g, c);
#pragma unroll
    for (int q = 0; q < NV; ++q) M[q][1] = c[q];
    psi_m<D, 0, 0, 1, 0>(g, c);
#pragma unroll
    for (int q = 0; q < NV; ++q) M[q][2] = c[q];
    if constexpr (D == 3) {
        psi_m<D, 0, 0, 0, 1>(g, c);
#pragma unroll
        for (int q = 0; q < NV; ++q) M[q][3] = c[q];
    }
    {
        double e[NV] = {};
        e[D + 1] = 1.0;
        apsi<D, 0, 0, 0, 0>(g, e, c);
#pragma unroll
        for (int q = 0; q < NV; ++q) M[q][D + 1] = c[q];
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const double piv = 1.0 / M[k][k];
#pragma unroll
        for (int r = k + 1; r < NV; ++r) {
            const double f = M[r][k] * piv;
            M[r][k] = f;
#pragma unroll
            for (int cc = k + 1; cc < NV; ++cc) M[r][cc] -= f * M[k][cc];
        }
    }
}
template <int D>
__device__ __forceinline__ void msolve(const double (*M)[D + 2], double *x)
{
    constexpr int NV = D + 2;
#pragma unroll
    for (int r = 1; r < NV; ++r)
#pragma unroll
        for (int c = 0; c < r; ++c) x[r] -= M[r][c] * x[c];
#pragma unroll
    for (int r = NV - 1; r >= 0; --r) {
#pragma unroll
        for (int c = r + 1; c < NV; ++c) x[r] -= M[r][c] * x[c];
        x[r] /= M[r][r];
    }
}

// micro slopes a_e = M^-1 dW_e / rho and A from <A + a.u> = 0 (Eq.(co))
template <int D>
__device__ __forceinline__ void slopes(const Maxw<D> &g, const double (*M)[D + 2], const double *dW, double (*a)[D + 2],
                                       double *A)
{
    constexpr int NV = D + 2;
    const double ir = 1.0 / g.rho;
#pragma unroll
    for (int e = 0; e < D; ++e) {
#pragma unroll
        for (int q = 0; q < NV; ++q) a[e][q] = dW[e * NV + q] * ir;
        msolve<D>(M, a[e]);
    }
    adotu<D, 0, 0>(g, a, A);
#pragma unroll
    for (int q = 0; q < NV; ++q) A[q] = -A[q];
    msolve<D>(M, A);
}

// BGK flux at one Gauss point in the face frame (x1 = normal): F time-
// integrated over [0, dt], Wt = W(dt).  dW[e*NV+q] = dW_q / dx_e (frame).
template <int D>
__device__ __noinline__ void gks_local(const double *wl, const double *dwl, const double *wr, const double *dwr, double dt,
                                       double tau, double gm1, double K, double *F, double *Wt)
{
    constexpr int NV = D + 2;
    double al[D][NV], ar[D][NV], Al[NV], Ar[NV], ac[D][NV], Ac[NV];
    Maxw<D> gl, gr, gc;
    double M[NV][NV];
    maxw<D>(wl, gm1, K, gl);
    maxw<D>(wr, gm1, K, gr);
    mfactor<D>(gl, M);
    slopes<D>(gl, M, dwl, al, Al);
    mfactor<D>(gr, M);
    slopes<D>(gr, M, dwr, ar, Ar);
    // W^c (Eq.(compatibility2)) and its slopes (reading C10e)
    double wc[NV], t1[NV], t2[NV], dwc[D * NV];
    psi_m<D, 1, 0, 0, 0>(gl, t1);
    psi_m<D, 2, 0, 0, 0>(gr, t2);
#pragma unroll
    for (int q = 0; q < NV; ++q) wc[q] = gl.rho * t1[q] + gr.rho * t2[q];
    maxw<D>(wc, gm1, K, gc);
#pragma unroll
    for (int e = 0; e < D; ++e) {
        apsi<D, 1, 0, 0, 0>(gl, al[e], t1);
        apsi<D, 2, 0, 0, 0>(gr, ar[e], t2);
#pragma unroll
        for (int q = 0; q < NV; ++q) dwc[e * NV + q] = gl.rho * t1[q] + gr.rho * t2[q];
    }
    mfactor<D>(gc, M);
    slopes<D>(gc, M, dwc, ac, Ac);
    // time integrals (Eqs. (dis1), (dis2))
    const double ex = exp(-dt / tau);
    const double q1 = dt - tau * (1.0 - ex);
    const double q2 = 2.0 * tau * tau - tau * dt - tau * ex * (dt + 2.0 * tau);
    const double q3 = 0.5 * dt * dt - tau * dt + tau * tau * (1.0 - ex);
    const double q4 = tau * (1.0 - ex);
    const double q5 = tau * tau - tau * ex * (dt + tau);
    const double c1 = 1.0 - ex, c2 = (dt + tau) * ex - tau, c3 = dt - tau + tau * ex;
    // equilibrium part
    psi_m<D, 0, 1, 0, 0>(gc, t1);
#pragma unroll
    for (int q = 0; q < NV; ++q) F[q] = q1 * t1[q];
    adotu<D, 0, 1>(gc, ac, t1);
    apsi<D, 0, 1, 0, 0>(gc, Ac, t2);
#pragma unroll
    for (int q = 0; q < NV; ++q) F[q] = gc.rho * (F[q] + q2 * t1[q] + q3 * t2[q]);
    psi_m<D, 0, 0, 0, 0>(gc, t1);
#pragma unroll
    for (int q = 0; q < NV; ++q) Wt[q] = c1 * t1[q];
    adotu<D, 0, 0>(gc, ac, t1);
    apsi<D, 0, 0, 0, 0>(gc, Ac, t2);
#pragma unroll
    for (int q = 0; q < NV; ++q) Wt[q] = gc.rho * (Wt[q] + c2 * t1[q] + c3 * t2[q]);
    // kinetic part: e^{-t/tau} g^k [1 - tau (a.u + A) - t a.u], k = l on u1 > 0, r on u1 < 0
    double t3[NV];
    psi_m<D, 1, 1, 0, 0>(gl, t1);
    adotu<D, 1, 1>(gl, al, t2);
    apsi<D, 1, 1, 0, 0>(gl, Al, t3);
#pragma unroll
    for (int q = 0; q < NV; ++q) F[q] += gl.rho * (q4 * t1[q] - (tau * q4 + q5) * t2[q] - tau * q4 * t3[q]);
    psi_m<D, 2, 1, 0, 0>(gr, t1);
    adotu<D, 2, 1>(gr, ar, t2);
    apsi<D, 2, 1, 0, 0>(gr, Ar, t3);
#pragma unroll
    for (int q = 0; q < NV; ++q) F[q] += gr.rho * (q4 * t1[q] - (tau * q4 + q5) * t2[q] - tau * q4 * t3[q]);
    psi_m<D, 1, 0, 0, 0>(gl, t1);
    adotu<D, 1, 0>(gl, al, t2);
    apsi<D, 1, 0, 0, 0>(gl, Al, t3);
#pragma unroll
    for (int q = 0; q < NV; ++q) Wt[q] += gl.rho * ex * (t1[q] - (tau + dt) * t2[q] - tau * t3[q]);
    psi_m<D, 2, 0, 0, 0>(gr, t1);
    adotu<D, 2, 0>(gr, ar, t2);
    apsi<D, 2, 0, 0, 0>(gr, Ar, t3);
#pragma unroll
    for (int q = 0; q < NV; ++q) Wt[q] += gr.rho * ex * (t1[q] - (tau + dt) * t2[q] - tau * t3[q]);
}

// face frame (C10a): e0 = n; 3D e1 = normalise(n x x_k), x_k the axis of the
// smallest |n_k| (first on ties), e2 = n x e1; 2D e1 = (-n_y, n_x)
template <int D>
__device__ __forceinline__ void frame(const double *n, double (*E)[3])
{
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) E[a][b] = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) E[0][k] = n[k];
    if (D == 2) {
        E[1][0] = -n[1];
        E[1][1] = n[0];
    } else {
        const double a0 = fabs(n[0]), a1 = fabs(n[1]), a2 = fabs(n[D - 1]);
        const int k = (a1 < a0) ? ((a2 < a1) ? 2 : 1) : ((a2 < a0) ? 2 : 0);
        double t[3];
        // n x x_k
        if (k == 0) { t[0] = 0.0; t[1] = n[D - 1]; t[2] = -n[1]; }
        else if (k == 1) { t[0] = -n[D - 1]; t[1] = 0.0; t[2] = n[0]; }
        else { t[0] = n[1]; t[1] = -n[0]; t[2] = 0.0; }
        const double it = rsqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
        E[1][0] = t[0] * it; E[1][1] = t[1] * it; E[1][2] = t[2] * it;
        E[2][0] = n[1] * E[1][2] - n[D - 1] * E[1][1];
        E[2][1] = n[D - 1] * E[1][0] - n[0] * E[1][2];
        E[2][2] = n[0] * E[1][1] - n[1] * E[1][0];
    }
}

// global frame: rotate states / gradients in, flux / state out
template <int D>
__device__ __forceinline__ void gks_flux(const double *wl, const double *gl, const double *wr, const double *gr,
                                         const double *n, double dt, double tau, double gm1, double K, double *F,
                                         double *Wt)
{
    constexpr int NV = D + 2;
    double E[3][3];
    frame<D>(n, E);
    double lw[2][NV], lg[2][D * NV];
#pragma unroll
    for (int sd = 0; sd < 2; ++sd) {
        const double *W = sd ? wr : wl, *G = sd ? gr : gl;
        lw[sd][0] = W[0];
        lw[sd][NV - 1] = W[NV - 1];
#pragma unroll
        for (int a = 0; a < D; ++a) {
            double s = 0.0;
#pragma unroll
            for (int b = 0; b < D; ++b) s += E[a][b] * W[1 + b];
            lw[sd][1 + a] = s;
        }
#pragma unroll
        for (int b = 0; b < D; ++b) {
            double col[NV];
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                double s = 0.0;
#pragma unroll
                for (int c = 0; c < D; ++c) s += E[b][c] * G[c * NV + q];
                col[q] = s;
            }
            lg[sd][b * NV] = col[0];
            lg[sd][b * NV + NV - 1] = col[NV - 1];
#pragma unroll
            for (int a = 0; a < D; ++a) {
                double s = 0.0;
#pragma unroll
                for (int c = 0; c < D; ++c) s += E[a][c] * col[1 + c];
                lg[sd][b * NV + 1 + a] = s;
            }
        }
    }
    double Fl[NV], Wl[NV];
    gks_local<D>(lw[0], lg[0], lw[1], lg[1], dt, tau, gm1, K, Fl, Wl);
    F[0] = Fl[0];
    F[NV - 1] = Fl[NV - 1];
    Wt[0] = Wl[0];
    Wt[NV - 1] = Wl[NV - 1];
#pragma unroll
    for (int k = 0; k < D; ++k) {
        double s = 0.0, u = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) { s += E[a][k] * Fl[1 + a]; u += E[a][k] * Wl[1 + a]; }
        F[1 + k] = s;
        Wt[1 + k] = u;
    }
}

// DF at one Gauss point (O5 formula, C7)
template <int D>
__device__ __forceinline__ double df_point(const double *wl, const double *wr, const double *n, const Phys &ph)
{
    const Side<D> sl = side_of<D>(wl, n, ph.gm1), sr = side_of<D>(wr, n, ph.gm1);
    const double ial = rsqrt(ph.gamma * sl.p * sl.ir), iar = rsqrt(ph.gamma * sr.p * sr.ir);
    const double dMn = sl.U * ial - sr.U * iar;
    double dMt2 = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const double t = (sl.u[k] - sl.U * n[k]) * ial - (sr.u[k] - sr.U * n[k]) * iar;
        dMt2 += t * t;
    }
    const double dp = fabs(sl.p - sr.p);
    const double Dv = dp * sl.ip + dp * sr.ip + dMn * dMn + dMt2;
    return 1.0 / (1.0 + Dv * Dv);
}

// ------------------------------------------------------------------ kernels
template <int D>
__global__ void __launch_bounds__(256) k_ho_sr(DevLevel L, HoDev H, Phys ph, BCs bc)
{
    constexpr int NV = D + 2;
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= L.nf) return;
    const int l = __ldg(L.fl + f), r = __ldg(L.fr + f);
    double A[D], S2 = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) { A[k] = __ldg(L.fA + (size_t)k * L.nf + f); S2 += A[k] * A[k]; }
    const double S = sqrt(S2);
    double n[D];
#pragma unroll
    for (int k = 0; k < D; ++k) n[k] = A[k] / S;
    double wl[NV], wr[NV];
    ld_vec<NV>(L.W + (size_t)l * NV, wl);
    if (r >= 0) ld_vec<NV>(L.W + (size_t)r * NV, wr);
    else ghost<D>(bc.kind[-r - 1], wl, bc, n, wr);
    double wb[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) wb[q] = 0.5 * (wl[q] + wr[q]);
    double mb = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) mb += (wb[1 + k] / wb[0]) * n[k];
    const double pb = pressure<D>(wb, ph.gm1);
    H.sr[f] = S * (ph.omega * (fabs(mb) + sqrt(ph.gamma * pb / wb[0])));
}

// positions of the quadratic monomials (a <= b, row major)
template <int D> __device__ __forceinline__ int qa(int k) { return D == 2 ? (k < 2 ? 0 : 1) : (k < 3 ? 0 : (k < 5 ? 1 : 2)); }
template <int D> __device__ __forceinline__ int qb(int k)
{
    return D == 2 ? (k == 0 ? 0 : 1) : (k == 0 ? 0 : (k == 1 ? 1 : (k == 2 ? 2 : (k == 3 ? 1 : (k == 4 ? 2 : 2)))));
}

template <int D>
__global__ void __launch_bounds__(128) k_ho_recon(DevLevel L, HoDev H, Phys ph, BCs bc, double cfl_exp, double gam0,
                                                  double eps)
{
    constexpr int NV = D + 2, NQ = D * (D + 1) / 2, NK = D + NQ, NC = 1 + NK;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= L.n) return;
    const int f0 = __ldg(H.hfoff + i), f1 = __ldg(H.hfoff + i + 1);
    const double V = __ldg(L.vol + i);
    double wi[NV];
    ld_vec<NV>(L.W + (size_t)i * NV, wi);
    // C8: Sigma, Dt; C4: Green-Gauss sums
    double sig = 0.0, g1[NV][D];
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
        for (int k = 0; k < D; ++k) g1[q][k] = 0.0;
    for (int s = f0; s < f1; ++s) {
        const int sf = __ldg(H.hface + s);
        const int f = (sf > 0 ? sf : -sf) - 1;
        const double sg = sf > 0 ? 1.0 : -1.0;
        sig += __ldg(H.sr + f);
        double A[D], S2 = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) { A[k] = sg * __ldg(L.fA + (size_t)k * L.nf + f); S2 += A[k] * A[k]; }
        const int r = __ldg(L.fr + f);
        double wm[NV];
        if (r >= 0) {
            const int j = sf > 0 ? r : __ldg(L.fl + f);
            ld_vec<NV>(L.W + (size_t)j * NV, wm);
        } else {
            const double iS = 1.0 / sqrt(S2);
            double nn[D];
#pragma unroll
            for (int k = 0; k < D; ++k) nn[k] = A[k] * iS;
            ghost<D>(bc.kind[-r - 1], wi, bc, nn, wm);
        }
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const double h = (wm[q] + wi[q]) / (2.0 * V);
#pragma unroll
            for (int k = 0; k < D; ++k) g1[q][k] += h * A[k];
        }
    }
    L.sigma[i] = sig;
    H.dt[i] = cfl_exp * V / sig;
    const double ai = H.alpha[i];
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
        for (int k = 0; k < D; ++k) g1[q][k] *= ai;
    double m2[NQ];
#pragma unroll
    for (int k = 0; k < NQ; ++k) m2[k] = __ldg(H.m2 + (size_t)i * NQ + k);
    double *po = H.poly + (size_t)i * NV * NC;
    const int p0 = __ldg(H.poff + i), p1 = __ldg(H.poff + i + 1);
    int flag = 0;
    if (p1 > p0) {
        flag = 1;
        // C2: a = sum_m Pq_m (Q_m - Q_i) + sum_e Pg_{m,e} (Q_e)_m, neighbours in the operator's order
        double a[NV][NK];
#pragma unroll
        for (int q = 0; q < NV; ++q)
#pragma unroll
            for (int k = 0; k < NK; ++k) a[q][k] = 0.0;
        const double *P = H.P + p0;
        for (int s = f0; s < f1; ++s) {
            const int sf = __ldg(H.hface + s);
            const int f = (sf > 0 ? sf : -sf) - 1;
            const int r = __ldg(L.fr + f);
            if (r < 0) continue;
            const int j = sf > 0 ? r : __ldg(L.fl + f);
            double dq[NV], gj[NV * D];
            ld_vec<NV>(L.W + (size_t)j * NV, dq);
            ld_vec<NV * D>(H.G_ + (size_t)j * NV * D, gj);
#pragma unroll
            for (int q = 0; q < NV; ++q) dq[q] -= wi[q];
#pragma unroll
            for (int k = 0; k < NK; ++k) {
                const double pq = __ldg(P + k);
                double pg[D];
#pragma unroll
                for (int e = 0; e < D; ++e) pg[e] = __ldg(P + (1 + e) * NK + k);
#pragma unroll
                for (int q = 0; q < NV; ++q) {
                    double v = pq * dq[q];
#pragma unroll
                    for (int e = 0; e < D; ++e) v += pg[e] * gj[q * D + e];
                    a[q][k] += v;
                }
            }
            P += (D + 1) * NK;
        }
        // C5: WENO-Z combination per component
        const double V2 = D == 3 ? cbrt(V * V) : V;      // |Omega|^{2/d}
        const double V4 = V2 * V2;                          // |Omega|^{4/d}
        const double g0 = gam0, gg1 = 1.0 - gam0;
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            double Kh[D][D];
#pragma unroll
            for (int x = 0; x < D; ++x)
#pragma unroll
                for (int y = 0; y < D; ++y) Kh[x][y] = 0.0;
#pragma unroll
            for (int k = 0; k < NQ; ++k) {
                Kh[qa<D>(k)][qb<D>(k)] += a[q][D + k];
                Kh[qb<D>(k)][qa<D>(k)] += a[q][D + k];
            }
            double grad2 = 0.0;
#pragma unroll
            for (int e = 0; e < D; ++e) grad2 += a[q][e] * a[q][e];
#pragma unroll
            for (int e = 0; e < D; ++e)
#pragma unroll
                for (int k = 0; k < NQ; ++k) {
                    // sum_{c,c'} K_ec K_ec' M2_cc' over the symmetric M2: off-diagonal pairs twice
                    const int c = qa<D>(k), cc = qb<D>(k);
                    grad2 += (c == cc ? 1.0 : 2.0) * Kh[e][c] * Kh[e][cc] * m2[k];
                }
            double hess2 = 0.0;
#pragma unroll
            for (int k = 0; k < NQ; ++k) hess2 += Kh[qa<D>(k)][qb<D>(k)] * Kh[qa<D>(k)][qb<D>(k)];
            const double beta0 = V2 * grad2 + V4 * hess2;
            double gn = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) gn += g1[q][k] * g1[q][k];
            const double beta1 = V2 * gn;
            const double tz = fabs(beta0 - beta1);
            double w0 = g0 * (1.0 + tz / (beta0 + eps)), w1 = gg1 * (1.0 + tz / (beta1 + eps));
            const double ws = w0 + w1;
            w0 /= ws;
            w1 /= ws;
            const double cq = w0 / g0, cl = w1 - w0 * gg1 / g0;
            double c0 = wi[q];
#pragma unroll
            for (int k = 0; k < NQ; ++k) c0 -= cq * a[q][D + k] * m2[k];
            po[q * NC] = c0;
#pragma unroll
            for (int k = 0; k < D; ++k) po[q * NC + 1 + k] = cq * a[q][k] + cl * g1[q][k];
#pragma unroll
            for (int k = 0; k < NQ; ++k) po[q * NC + 1 + D + k] = cq * a[q][D + k];
        }
    } else {
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            po[q * NC] = wi[q];
#pragma unroll
            for (int k = 0; k < D; ++k) po[q * NC + 1 + k] = g1[q][k];
#pragma unroll
            for (int k = 0; k < NQ; ++k) po[q * NC + 1 + D + k] = 0.0;
        }
    }
    // C6b: positivity at every Gauss point of the cell's faces
    double x0[D];
#pragma unroll
    for (int k = 0; k < D; ++k) x0[k] = __ldg(H.ctr + (size_t)i * D + k);
    bool bad = false;
    for (int s = f0; s < f1 && !bad; ++s) {
        const int sf = __ldg(H.hface + s);
        const int f = (sf > 0 ? sf : -sf) - 1;
        for (int k = 0; k < H.G; ++k) {
            if (__ldg(H.gw + (size_t)f * H.G + k) == 0.0) continue;
            double y[D];
#pragma unroll
            for (int e = 0; e < D; ++e) y[e] = __ldg(H.gp + ((size_t)f * H.G + k) * D + e) - x0[e];
            double w[NV];
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                double v = po[q * NC];
#pragma unroll
                for (int e = 0; e < D; ++e) v += po[q * NC + 1 + e] * y[e];
#pragma unroll
                for (int kk = 0; kk < NQ; ++kk) v += po[q * NC + 1 + D + kk] * y[qa<D>(kk)] * y[qb<D>(kk)];
                w[q] = v;
            }
            const double p = pressure<D>(w, ph.gm1);
            if (!(w[0] > 0.0) || !(p > 0.0)) { bad = true; break; }
        }
    }
    if (bad) {
        flag |= 2;
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            po[q * NC] = wi[q];
#pragma unroll
            for (int k = 1; k < NC; ++k) po[q * NC + k] = 0.0;
        }
    }
    H.flags[i] = flag;
}

// value and gradient of a cell polynomial at y = x - x_cell
template <int D>
__device__ __forceinline__ void peval(const double *po, const double *y, double *w, double *g)
{
    constexpr int NV = D + 2, NQ = D * (D + 1) / 2, NC = 1 + D + NQ;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        double c[NC];
#pragma unroll
        for (int k = 0; k < NC; ++k) c[k] = __ldg(po + q * NC + k);
        double v = c[0];
        double gr[D];
#pragma unroll
        for (int e = 0; e < D; ++e) { v += c[1 + e] * y[e]; gr[e] = c[1 + e]; }
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
            const int a = qa<D>(k), b = qb<D>(k);
            v += c[1 + D + k] * y[a] * y[b];
            gr[a] += c[1 + D + k] * y[b];
            gr[b] += c[1 + D + k] * y[a];
        }
        w[q] = v;
#pragma unroll
        for (int e = 0; e < D; ++e) g[e * NV + q] = gr[e];
    }
}

template <int D>
__global__ void __launch_bounds__(128) k_ho_flux(DevLevel L, HoDev H, Phys ph, BCs bc, double c1, double c2)
{
    constexpr int NV = D + 2, NQ = D * (D + 1) / 2, NC = 1 + D + NQ;
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= L.nf) return;
    const int l = __ldg(L.fl + f), r = __ldg(L.fr + f);
    double A[D], S2 = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) { A[k] = __ldg(L.fA + (size_t)k * L.nf + f); S2 += A[k] * A[k]; }
    const double S = sqrt(S2);
    double n[D];
#pragma unroll
    for (int k = 0; k < D; ++k) n[k] = A[k] / S;
    const double dtl = H.dt[l];
    const double dtf = r >= 0 ? fmin(dtl, H.dt[r]) : dtl;
    double xl[D], xr[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
        xl[k] = __ldg(H.ctr + (size_t)l * D + k);
        xr[k] = r >= 0 ? __ldg(H.ctr + (size_t)r * D + k) : 0.0;
    }
    const int kind = r < 0 ? bc.kind[-r - 1] : 0;
    double Fs[NV], Ws[NV], ap = 1.0;
#pragma unroll
    for (int q = 0; q < NV; ++q) { Fs[q] = 0.0; Ws[q] = 0.0; }
    for (int k = 0; k < H.G; ++k) {
        const double w = __ldg(H.gw + (size_t)f * H.G + k);
        if (w == 0.0) continue;
        double x[D], y[D];
#pragma unroll
        for (int e = 0; e < D; ++e) x[e] = __ldg(H.gp + ((size_t)f * H.G + k) * D + e);
        double wl[NV], gl[D * NV], wr[NV], gr[D * NV];
#pragma unroll
        for (int e = 0; e < D; ++e) y[e] = x[e] - xl[e];
        peval<D>(H.poly + (size_t)l * NV * NC, y, wl, gl);
        if (r >= 0) {
#pragma unroll
            for (int e = 0; e < D; ++e) y[e] = x[e] - xr[e];
            peval<D>(H.poly + (size_t)r * NV * NC, y, wr, gr);
        } else {
            ghost<D>(kind, wl, bc, n, wr);
#pragma unroll
            for (int e = 0; e < D * NV; ++e) gr[e] = kind == GMG_EXTRAP ? gl[e] : 0.0;
        }
        ap *= df_point<D>(wl, wr, n, ph);
        const double pl = pressure<D>(wl, ph.gm1), pr = pressure<D>(wr, ph.gm1);
        const double tau = c1 * dtf + c2 * dtf * fabs(pl - pr) / (pl + pr);
        double F[NV], Wt[NV];
        gks_flux<D>(wl, gl, wr, gr, n, dtf, tau, ph.gm1, ph.K, F, Wt);
#pragma unroll
        for (int q = 0; q < NV; ++q) { Fs[q] += w * F[q]; Ws[q] += w * Wt[q]; }
    }
    double *o = H.frec + (size_t)f * kHoRec;
#pragma unroll
    for (int q = 0; q < NV; ++q) { o[q] = S * Fs[q] / dtf; o[NV + q] = Ws[q]; }
    o[2 * NV] = ap;
}

template <int D>
__global__ void __launch_bounds__(256) k_ho_gather(DevLevel L, HoDev H, int mode, double cfl_exp, double *Rout,
                                                   double *alpha_out, double *partial)
{
    constexpr int NV = D + 2;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double R[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) R[q] = 0.0;
    if (i < L.n) {
        double Gn[NV][D];
#pragma unroll
        for (int q = 0; q < NV; ++q)
#pragma unroll
            for (int e = 0; e < D; ++e) Gn[q][e] = 0.0;
        double al = 1.0;
        const int f0 = __ldg(H.hfoff + i), f1 = __ldg(H.hfoff + i + 1);
        for (int s = f0; s < f1; ++s) {
            const int sf = __ldg(H.hface + s);
            const int f = (sf > 0 ? sf : -sf) - 1;
            const double sg = sf > 0 ? 1.0 : -1.0;
            const double *o = H.frec + (size_t)f * kHoRec;
            double A[D];
#pragma unroll
            for (int k = 0; k < D; ++k) A[k] = sg * __ldg(L.fA + (size_t)k * L.nf + f);
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                R[q] += sg * __ldg(o + q);
                const double ws = __ldg(o + NV + q);
#pragma unroll
                for (int e = 0; e < D; ++e) Gn[q][e] += ws * A[e];
            }
            al *= __ldg(o + 2 * NV);
        }
        const double sc = al / __ldg(L.vol + i);
        const size_t o = (size_t)i * NV;
        if (mode & HO_UPDATE) {
            const double c = cfl_exp / L.sigma[i];
#pragma unroll
            for (int q = 0; q < NV; ++q) L.W[o + q] = L.W[o + q] - c * R[q];
#pragma unroll
            for (int q = 0; q < NV; ++q)
#pragma unroll
                for (int e = 0; e < D; ++e) H.G_[(o + q) * D + e] = Gn[q][e] * sc;
            H.alpha[i] = al;
        }
        if (mode & HO_RT) {
#pragma unroll
            for (int q = 0; q < NV; ++q) L.Rt[o + q] = R[q];
            L.alpha[i] = al;
            H.alpha[i] = al;
        }
        if (mode & HO_OUT) {
#pragma unroll
            for (int q = 0; q < NV; ++q) Rout[o + q] = R[q];
#pragma unroll
            for (int q = 0; q < NV; ++q)
#pragma unroll
                for (int e = 0; e < D; ++e) H.Gout[(o + q) * D + e] = Gn[q][e] * sc;
            alpha_out[i] = al;
        }
    }
    if (mode & HO_NORM) {
        __shared__ double sh[8][NV];
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            double v = R[q] * R[q];
            for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
            if (lane == 0) sh[wid][q] = v;
        }
        __syncthreads();
        if (threadIdx.x < NV) {
            double v = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += sh[w][threadIdx.x];
            partial[(size_t)blockIdx.x * NV + threadIdx.x] = v;
        }
    }
}

// ----------------------------------------------------------------- launches
inline int hblk(int64_t n, int b) { return (int)std::max<int64_t>(1, (n + b - 1) / b); }

template <int D>
void ho_launch_t(int which, const DevLevel &L, const HoDev &H, const Phys &ph, const BCs &bc, const gmg_options &o,
                 int mode, double *Rout, double *aout, cudaStream_t s)
{
    switch (which) {
    case 0: k_ho_sr<D><<<hblk(L.nf, 256), 256, 0, s>>>(L, H, ph, bc); break;
    case 1: k_ho_recon<D><<<hblk(L.n, 128), 128, 0, s>>>(L, H, ph, bc, o.cfl_exp, o.ho_gam0, o.ho_eps); break;
    case 2: k_ho_flux<D><<<hblk(L.nf, 128), 128, 0, s>>>(L, H, ph, bc, o.ho_c1, o.ho_c2); break;
    default: k_ho_gather<D><<<hblk(L.n, 256), 256, 0, s>>>(L, H, mode, o.cfl_exp, Rout, aout, L.partial); break;
    }
}

void ho_launch(int which, const DevLevel &L, const HoDev &H, const Phys &ph, const BCs &bc, const gmg_options &o,
               int mode, double *Rout, double *aout, cudaStream_t s)
{
    if (L.dim == 3) ho_launch_t<3>(which, L, H, ph, bc, o, mode, Rout, aout, s);
    else ho_launch_t<2>(which, L, H, ph, bc, o, mode, Rout, aout, s);
}

}  // namespace gmg
