// ho.cu -- sm_100a kernels of the third-order compact gas-kinetic fine
// operator (§2.3-§3; readings
// C1-C14 of DESIGN.md §12).  FP64.  Four launches per evaluation:
//
//   k_ho_sr     per face   S r_f (first-order spectral radius of the cell averages, A5)
//   k_ho_recon  per cell   Sigma_i, Dt_i, p1 (Green-Gauss x DF), p2 (stored KKT operator x
//                          neighbour averages and slopes), WENO-Z weights
//                          -> one polynomial per cell and component
//   k_ho_flux   per face   at every Gauss point: both sides' polynomial values and gradients,
//                          positivity (C6b), DF, collision time, the BGK flux (Eqs. (dis1), (dis2)) integrated over
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
// normalised Maxwellian moments: Mu (u1, full range), Mh (u1 on the half
// range R: 1 = u1 > 0, 2 = u1 < 0; unused for R = 0), Mv, Mw, <xi^2>, <xi^4>
template <int D, int R>
struct Maxw {
    double rho;
    double Mu[7], Mh[R == 0 ? 1 : 7], Mv[6], Mw[D == 3 ? 6 : 1];
    double x1, x2;
};

template <int N>
__device__ __forceinline__ void rec_mom(double U, double inv2l, double *M)
{
#pragma unroll
    for (int k = 2; k < N; ++k) M[k] = U * M[k - 1] + (double)(k - 1) * inv2l * M[k - 2];
}

// R = 1, 2: the half range u1 > 0 / u1 < 0; sgn (+1 / -1) selects it at run time
// when one copy of the code serves both sides (R = 1 with sgn = -1 is the R = 2 range)
template <int D, int R>
__device__ __forceinline__ void maxw(const double *w, double gm1, double K, Maxw<D, R> &g,
                                     double sgn = R == 2 ? -1.0 : 1.0, bool half = true)
{
    g.rho = w[0];
    const double ir = 1.0 / w[0];
    double U[3] = {0, 0, 0}, u2 = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) { U[k] = w[1 + k] * ir; u2 += U[k] * U[k]; }
    const double p = gm1 * (w[D + 1] - 0.5 * w[0] * u2);
    const double inv2l = p * ir;                       // 1/(2 lambda), lambda = rho / (2p)
    g.Mu[0] = 1.0; g.Mu[1] = U[0];
    rec_mom<7>(U[0], inv2l, g.Mu);
    if (R != 0 && half) {
        const double lam = 0.5 * w[0] / p;
        const double sl = sqrt(lam);
        const double e = exp(-lam * U[0] * U[0]) * (0.28209479177387814 / sl);   // e^{-l U^2} / (2 sqrt(pi l))
        g.Mh[0] = 0.5 * erfc(-sgn * sl * U[0]);
        g.Mh[1] = U[0] * g.Mh[0] + sgn * e;
        rec_mom<7>(U[0], inv2l, g.Mh);
    }
    g.Mv[0] = 1.0; g.Mv[1] = U[1];
    rec_mom<6>(U[1], inv2l, g.Mv);
    if constexpr (D == 3) { g.Mw[0] = 1.0; g.Mw[1] = U[2]; rec_mom<6>(U[2], inv2l, g.Mw); }
    g.x1 = K * inv2l;
    g.x2 = (K * K + 2.0 * K) * inv2l * inv2l;
}

// u1 moments: H = false full range, true the Maxwellian's half range
template <int D, int R, bool H>
__device__ __forceinline__ const double *umom(const Maxw<D, R> &g)
{
    if constexpr (H && R != 0) return g.Mh;
    else return g.Mu;
}

// T^{abc}_{qj} = <psi_q psi_j u^a v^b w^c>: the symmetric moment matrix of a
// monomial weight, built once from products of 1D moments and then applied
// to several micro-slope vectors (every contraction of Eqs. (dis1), (dis2),
// (co) is o += f T^{abc} s).  H: u1 moments over the Maxwellian's half range.
template <int D, int R, bool H, int a, int b, int c>
__device__ __forceinline__ void tmat(const Maxw<D, R> &g, double (*T)[D + 2])
{
    const double *Mu = umom<D, R, H>(g);
    const double x1 = g.x1, x2 = g.x2;
    if constexpr (D == 3) {
        auto P = [&](int i, int j, int k) { return Mu[i] * g.Mv[j] * g.Mw[k]; };
        auto E = [&](int i, int j, int k) { return 0.5 * (P(i + 2, j, k) + P(i, j + 2, k) + P(i, j, k + 2) + x1 * P(i, j, k)); };
        T[0][0] = P(a, b, c);
        T[0][1] = P(a + 1, b, c);
        T[0][2] = P(a, b + 1, c);
        T[0][3] = P(a, b, c + 1);
        T[0][4] = E(a, b, c);
        T[1][1] = P(a + 2, b, c);
        T[1][2] = P(a + 1, b + 1, c);
        T[1][3] = P(a + 1, b, c + 1);
        T[1][4] = E(a + 1, b, c);
        T[2][2] = P(a, b + 2, c);
        T[2][3] = P(a, b + 1, c + 1);
        T[2][4] = E(a, b + 1, c);
        T[3][3] = P(a, b, c + 2);
        T[3][4] = E(a, b, c + 1);
        const double s2 = P(a + 2, b, c) + P(a, b + 2, c) + P(a, b, c + 2);
        T[4][4] = 0.25 * (P(a + 4, b, c) + P(a, b + 4, c) + P(a, b, c + 4) +
                          2.0 * (P(a + 2, b + 2, c) + P(a + 2, b, c + 2) + P(a, b + 2, c + 2)) + 2.0 * x1 * s2 +
                          x2 * P(a, b, c));
    } else {
        auto P = [&](int i, int j) { return Mu[i] * g.Mv[j]; };
        auto E = [&](int i, int j) { return 0.5 * (P(i + 2, j) + P(i, j + 2) + x1 * P(i, j)); };
        T[0][0] = P(a, b);
        T[0][1] = P(a + 1, b);
        T[0][2] = P(a, b + 1);
        T[0][3] = E(a, b);
        T[1][1] = P(a + 2, b);
        T[1][2] = P(a + 1, b + 1);
        T[1][3] = E(a + 1, b);
        T[2][2] = P(a, b + 2);
        T[2][3] = E(a, b + 1);
        T[3][3] = 0.25 * (P(a + 4, b) + P(a, b + 4) + 2.0 * P(a + 2, b + 2) + 2.0 * x1 * (P(a + 2, b) + P(a, b + 2)) +
                          x2 * P(a, b));
    }
#pragma unroll
    for (int q = 1; q < D + 2; ++q)
#pragma unroll
        for (int j = 0; j < q; ++j) T[q][j] = T[j][q];
}
// o += f T s
template <int D>
__device__ __forceinline__ void tmv(const double (*T)[D + 2], const double *s, double f, double *o)
{
#pragma unroll
    for (int q = 0; q < D + 2; ++q) {
        double v = 0.0;
#pragma unroll
        for (int j = 0; j < D + 2; ++j) v += T[q][j] * s[j];
        o[q] += f * v;
    }
}

// in-place factorisation of the SPD moment matrix (no pivoting) and solve
template <int D>
__device__ __forceinline__ void mfactor(double (*M)[D + 2])
{
    constexpr int NV = D + 2;
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

// micro slopes a_e = M^-1 dW_e / rho (M = T^{000}, full range) and A from
// <A + a.u> = 0, i.e. M A = -sum_e T^{e_e} a_e (Eq.(co))
template <int D, int R>
__device__ __forceinline__ void slopes(const Maxw<D, R> &g, const double *dW, double (*a)[D + 2], double *A)
{
    constexpr int NV = D + 2;
    double M[NV][NV], T[NV][NV];
    tmat<D, R, false, 0, 0, 0>(g, M);
    mfactor<D>(M);
    const double ir = 1.0 / g.rho;
#pragma unroll
    for (int e = 0; e < D; ++e) {
#pragma unroll
        for (int q = 0; q < NV; ++q) a[e][q] = dW[e * NV + q] * ir;
        msolve<D>(M, a[e]);
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) A[q] = 0.0;
    tmat<D, R, false, 1, 0, 0>(g, T);
    tmv<D>(T, a[0], -1.0, A);
    tmat<D, R, false, 0, 1, 0>(g, T);
    tmv<D>(T, a[1], -1.0, A);
    if constexpr (D == 3) {
        tmat<D, R, false, 0, 0, 1>(g, T);
        tmv<D>(T, a[2], -1.0, A);
    }
    msolve<D>(M, A);
}

// time coefficients of Eqs. (dis1), (dis2): integrals over [0, dt] (q1..q5)
// and values at dt (c1..c3, ex)
struct TimeC {
    double q1, q2, q3, q4, q5, c1, c2, c3, ex, tau, dt;
};
__device__ __forceinline__ TimeC time_coeffs(double dt, double tau)
{
    TimeC t;
    const double ex = exp(-dt / tau);
    t.q1 = dt - tau * (1.0 - ex);
    t.q2 = 2.0 * tau * tau - tau * dt - tau * ex * (dt + 2.0 * tau);
    t.q3 = 0.5 * dt * dt - tau * dt + tau * tau * (1.0 - ex);
    t.q4 = tau * (1.0 - ex);
    t.q5 = tau * tau - tau * ex * (dt + tau);
    t.c1 = 1.0 - ex;
    t.c2 = (dt + tau) * ex - tau;
    t.c3 = dt - tau + tau * ex;
    t.ex = ex;
    t.tau = tau;
    t.dt = dt;
    return t;
}

// The three kinetic passes of a Gauss point through ONE code copy (round 2:
// a smaller kernel body, fewer instruction-fetch stalls), frame coordinates.
// mode 0 / 1 -- one side of the interface (left state on u1 > 0, right on
// u1 < 0; the half range by its sign): its share of W^c (Eq.(compatibility2)),
// of the equilibrium slopes (reading C10e; dWc in shared memory, component k
// of this thread at dWc[k * blockDim.x]) and its kinetic terms of Eq.(dis1):
//   F  += rho int_0^dt e^{-t/tau} <u1 psi [1 - tau (a.u + A) - t a.u]>_half dt,
//   Wt += rho e^{-dt/tau} <psi [1 - tau (a.u + A) - dt a.u]>_half;
// mode 2 -- the equilibrium part of Eq.(dis2), C1 g^c + C2 a^c.u g^c + C3 A^c g^c
// (full range): the same contractions with the coefficients below.
template <int D>
__device__ __forceinline__ void kin_pass(const double *w, const double *dw, const TimeC &T, double gm1, double K,
                                         int mode, double *Wc, double *dWc, double *F, double *Wt)
{
    constexpr int NV = D + 2;
    const bool side = mode < 2;
    Maxw<D, 1> g;
    maxw<D, 1>(w, gm1, K, g, mode == 0 ? 1.0 : -1.0, side);
    double a[D][NV], A[NV], M[NV][NV];
    slopes<D, 1>(g, dw, a, A);
    if (!side) {   // the equilibrium's weights are full-range moments
#pragma unroll
        for (int i = 0; i < 7; ++i) g.Mh[i] = g.Mu[i];
    }
    const double rho = g.rho;
    const double cW0 = side ? rho * T.ex : rho * T.c1;
    const double cWA = side ? -rho * T.ex * T.tau : rho * T.c3;
    const double cF0 = side ? rho * T.q4 : rho * T.q1;
    const double cWa = side ? -rho * T.ex * (T.tau + T.dt) : rho * T.c2;
    const double cFA = side ? -rho * T.tau * T.q4 : rho * T.q3;
    const double cFa = side ? -rho * (T.tau * T.q4 + T.q5) : rho * T.q2;
    tmat<D, 1, true, 0, 0, 0>(g, M);
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        if (side) Wc[q] += rho * M[q][0];
        Wt[q] += cW0 * M[q][0];
    }
    if (side) {
#pragma unroll
        for (int e = 0; e < D; ++e) {
            double u[NV];
#pragma unroll
            for (int q = 0; q < NV; ++q) u[q] = 0.0;
            tmv<D>(M, a[e], rho, u);
#pragma unroll
            for (int q = 0; q < NV; ++q) dWc[(e * NV + q) * blockDim.x] += u[q];
        }
    }
    tmv<D>(M, A, cWA, Wt);
    tmat<D, 1, true, 1, 0, 0>(g, M);
#pragma unroll
    for (int q = 0; q < NV; ++q) F[q] += cF0 * M[q][0];
    tmv<D>(M, a[0], cWa, Wt);
    tmv<D>(M, A, cFA, F);
    tmat<D, 1, true, 0, 1, 0>(g, M);
    tmv<D>(M, a[1], cWa, Wt);
    if constexpr (D == 3) {
        tmat<D, 1, true, 0, 0, 1>(g, M);
        tmv<D>(M, a[2], cWa, Wt);
    }
    tmat<D, 1, true, 2, 0, 0>(g, M);
    tmv<D>(M, a[0], cFa, F);
    tmat<D, 1, true, 1, 1, 0>(g, M);
    tmv<D>(M, a[1], cFa, F);
    if constexpr (D == 3) {
        tmat<D, 1, true, 1, 0, 1>(g, M);
        tmv<D>(M, a[2], cFa, F);
    }
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
    if constexpr (D == 2) {
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

// rotate a state and its gradient (G[c*NV+q] = dW_q/dx_c, global) into the frame
template <int D>
__device__ __forceinline__ void to_frame(const double (*E)[3], const double *W, const double *G, double *w, double *g)
{
    constexpr int NV = D + 2;
    w[0] = W[0];
    w[NV - 1] = W[NV - 1];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < D; ++b) s += E[a][b] * W[1 + b];
        w[1 + a] = s;
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
        g[b * NV] = col[0];
        g[b * NV + NV - 1] = col[NV - 1];
#pragma unroll
        for (int a = 0; a < D; ++a) {
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < D; ++c) s += E[a][c] * col[1 + c];
            g[b * NV + 1 + a] = s;
        }
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

// one cell per group of NV lanes, one conserved component per lane: the p2
// operator columns are read once per group (same address in the group's
// lanes), neighbour states coalesced across the component lanes, and the
// per-lane state is one component's p1 / p2 / WENO (C4, C2, C5).
template <int NV>
__device__ __forceinline__ double pick(const double *v, int q)   // v[q] without dynamic register indexing
{
    double r = v[0];
#pragma unroll
    for (int k = 1; k < NV; ++k) r = q == k ? v[k] : r;
    return r;
}
template <int D>
__global__ void __launch_bounds__(256, 4) k_ho_recon(DevLevel L, HoDev H, Phys ph, BCs bc, double cfl_exp, double gam0,
                                                  double eps)
{
    constexpr int NV = D + 2, NQ = D * (D + 1) / 2, NK = D + NQ, NC = 1 + NK;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int i0 = t / NV, q = t % NV;                // NV lanes per cell (no shuffles: any alignment)
    const bool live = i0 < L.n;
    const int i = live ? i0 : L.n - 1;
    const bool comp = live && q < NV;
    const int qq = q < NV ? q : 0;
    const int f0 = __ldg(H.hfoff + i), f1 = __ldg(H.hfoff + i + 1);
    const double V = __ldg(L.vol + i);
    double wi[NV];
    ld_vec<NV>(L.W + (size_t)i * NV, wi);
    const double wq = pick<NV>(wi, qq);
    const int p0 = __ldg(H.poff + i), p1 = __ldg(H.poff + i + 1);
    const bool has2 = p1 > p0;
    // one pass over the cell's face slots (record: A outward | neighbour, face):
    // C8 Sigma, C4 Green-Gauss sum of this component, C2 p2 = sum_m Pq_m (Q_m - Q_i) + sum_e Pg_{m,e} (Q_e)_m
    double sig = 0.0, g1[D], a[NK];
#pragma unroll
    for (int k = 0; k < D; ++k) g1[k] = 0.0;
#pragma unroll
    for (int k = 0; k < NK; ++k) a[k] = 0.0;
    const double *P = H.P + p0;
    for (int s = f0; s < f1; ++s) {
        double rc[4];
        ld4na(H.hrec + (size_t)s * 4, rc);   // per-slot records, read once per launch: no L1 allocation
        const int2 jf = *reinterpret_cast<const int2 *>(&rc[3]);
        const int j = jf.x, f = jf.y;
        sig += __ldg(H.sr + f);
        double A[D];
#pragma unroll
        for (int k = 0; k < D; ++k) A[k] = rc[k];
        double qm;
        if (j >= 0) {
            qm = __ldg(L.W + (size_t)j * NV + qq);
            if (has2) {
                const double dq = qm - wq;
                double gj[D];
#pragma unroll
                for (int e = 0; e < D; ++e) gj[e] = __ldg(H.G_ + ((size_t)j * NV + qq) * D + e);
                constexpr int PST = ((D + 1) * NK + 3) & ~3;
                double pb[PST];
#pragma unroll
                for (int k = 0; k < PST; k += 4) ld4na(P + k, pb + k);   // streamed once: no L1 allocation
#pragma unroll
                for (int k = 0; k < NK; ++k) {
                    double v = pb[k] * dq;
#pragma unroll
                    for (int e = 0; e < D; ++e) v += pb[(1 + e) * NK + k] * gj[e];
                    a[k] += v;
                }
                P += PST;
            }
        } else {
            double S2 = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) S2 += A[k] * A[k];
            const double iS = 1.0 / sqrt(S2);
            double nn[D], wg[NV];
#pragma unroll
            for (int k = 0; k < D; ++k) nn[k] = A[k] * iS;
            ghost<D>(bc.kind[-j - 1], wi, bc, nn, wg);
            qm = pick<NV>(wg, qq);
        }
        const double h = (qm + wq) / (2.0 * V);
#pragma unroll
        for (int k = 0; k < D; ++k) g1[k] += h * A[k];
    }
    if (live && q == 0) {
        L.sigma[i] = sig;
        H.dt[i] = cfl_exp * V / sig;
    }
    const double ai = __ldg(H.alpha + i);
#pragma unroll
    for (int k = 0; k < D; ++k) g1[k] *= ai;
    double m2[NQ];
#pragma unroll
    for (int k = 0; k < NQ; ++k) m2[k] = __ldg(H.m2 + (size_t)i * NQ + k);
    double c[NC];                                   // this component's final polynomial
    int flag = 0;
    if (has2) {
        flag = 1;
        // C5: WENO-Z combination
        const double V2 = D == 3 ? cbrt(V * V) : V;      // |Omega|^{2/d}
        const double V4 = V2 * V2;                          // |Omega|^{4/d}
        const double g0 = gam0, gg1 = 1.0 - gam0;
        double Kh[D][D];
#pragma unroll
        for (int x = 0; x < D; ++x)
#pragma unroll
            for (int y = 0; y < D; ++y) Kh[x][y] = 0.0;
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
            Kh[qa<D>(k)][qb<D>(k)] += a[D + k];
            Kh[qb<D>(k)][qa<D>(k)] += a[D + k];
        }
        double grad2 = 0.0;
#pragma unroll
        for (int e = 0; e < D; ++e) grad2 += a[e] * a[e];
#pragma unroll
        for (int e = 0; e < D; ++e)
#pragma unroll
            for (int k = 0; k < NQ; ++k) {
                // sum_{c,c'} K_ec K_ec' M2_cc' over the symmetric M2: off-diagonal pairs twice
                const int x = qa<D>(k), y = qb<D>(k);
                grad2 += (x == y ? 1.0 : 2.0) * Kh[e][x] * Kh[e][y] * m2[k];
            }
        double hess2 = 0.0;
#pragma unroll
        for (int k = 0; k < NQ; ++k) hess2 += Kh[qa<D>(k)][qb<D>(k)] * Kh[qa<D>(k)][qb<D>(k)];
        const double beta0 = V2 * grad2 + V4 * hess2;
        double gn = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) gn += g1[k] * g1[k];
        const double beta1 = V2 * gn;
        const double tz = fabs(beta0 - beta1);
        double w0 = g0 * (1.0 + tz / (beta0 + eps)), w1 = gg1 * (1.0 + tz / (beta1 + eps));
        const double ws = w0 + w1;
        w0 /= ws;
        w1 /= ws;
        const double cq = w0 / g0, cl = w1 - w0 * gg1 / g0;
        c[0] = wq;
#pragma unroll
        for (int k = 0; k < NQ; ++k) c[0] -= cq * a[D + k] * m2[k];
#pragma unroll
        for (int k = 0; k < D; ++k) c[1 + k] = cq * a[k] + cl * g1[k];
#pragma unroll
        for (int k = 0; k < NQ; ++k) c[1 + D + k] = cq * a[D + k];
    } else {
        c[0] = wq;
#pragma unroll
        for (int k = 0; k < D; ++k) c[1 + k] = g1[k];
#pragma unroll
        for (int k = 0; k < NQ; ++k) c[1 + D + k] = 0.0;
    }
    if (comp) {
        double *po = H.poly + ((size_t)i * NV + q) * NC;
#pragma unroll
        for (int k = 0; k < NC; ++k) po[k] = c[k];
        if (q == 0) H.flags[i] = flag;
    }
}

// value (and gradient) of a cell polynomial at y = x - x_cell
template <int D, bool GRAD>
__device__ __forceinline__ void peval(const double *po, const double *y, double *w, double *g)
{
    constexpr int NV = D + 2, NQ = D * (D + 1) / 2, NC = 1 + D + NQ;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        double c[NC];
#pragma unroll
        for (int k = 0; k < NC; ++k) c[k] = __ldg(po + q * NC + k);
        if constexpr (GRAD) {
            double gr[D];
#pragma unroll
            for (int e = 0; e < D; ++e) gr[e] = c[1 + e];
#pragma unroll
            for (int k = 0; k < NQ; ++k) {
                const int a = qa<D>(k), b = qb<D>(k);
                gr[a] += c[1 + D + k] * y[b];
                gr[b] += c[1 + D + k] * y[a];
            }
#pragma unroll
            for (int e = 0; e < D; ++e) g[e * NV + q] = gr[e];
        } else {
            double v = c[0];
#pragma unroll
            for (int e = 0; e < D; ++e) v += c[1 + e] * y[e];
#pragma unroll
            for (int k = 0; k < NQ; ++k) v += c[1 + D + k] * y[qa<D>(k)] * y[qb<D>(k)];
            w[q] = v;
        }
    }
}

// one Gauss point per lane (H.glane: packed, no idle padding lanes for
// triangles; a face's points on consecutive lanes of one warp); the face's
// first lane adds the others' weighted flux / state / DF by shuffles
template <int D>
__global__ void __launch_bounds__(128) k_ho_flux(DevLevel L, HoDev H, Phys ph, BCs bc, double c1, double c2)
{
    constexpr int NV = D + 2, NQ = D * (D + 1) / 2, NC = 1 + D + NQ;
    constexpr int G = D == 3 ? 4 : 2;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int2 gl = t < H.nlane ? __ldg(H.glane + t) : make_int2(-1, 0);
    const bool live = gl.x >= 0;
    const int f = live ? gl.x / G : 0, k = live ? gl.x % G : 0;
    const int fc = live ? f : L.nf - 1;
    const double w = live ? __ldg(H.gw + (size_t)fc * G + k) : 0.0;
    double Fs[NV], Ws[NV], ap = 1.0;
#pragma unroll
    for (int q = 0; q < NV; ++q) { Fs[q] = 0.0; Ws[q] = 0.0; }
    const int l = __ldg(L.fl + fc), r = __ldg(L.fr + fc);
    double A[D], S2 = 0.0;
#pragma unroll
    for (int e = 0; e < D; ++e) { A[e] = __ldg(L.fA + (size_t)e * L.nf + fc); S2 += A[e] * A[e]; }
    const double S = sqrt(S2);
    double n[D];
#pragma unroll
    for (int e = 0; e < D; ++e) n[e] = A[e] / S;
    const double dtl = __ldg(H.dt + l);
    const double dtf = r >= 0 ? fmin(dtl, __ldg(H.dt + r)) : dtl;
    if (w != 0.0) {
        double x[D], yl[D], yr[D];
#pragma unroll
        for (int e = 0; e < D; ++e) {
            x[e] = __ldg(H.gp + ((size_t)fc * G + k) * D + e);
            yl[e] = x[e] - __ldg(H.ctr + (size_t)l * D + e);
            yr[e] = r >= 0 ? x[e] - __ldg(H.ctr + (size_t)r * D + e) : 0.0;
        }
        const int kind = r < 0 ? bc.kind[-r - 1] : 0;
        const double *pl = H.poly + (size_t)l * NV * NC;
        const double *pr = r >= 0 ? H.poly + (size_t)r * NV * NC : pl;
        double wl[NV], wr[NV], gtmp[D * NV];
        // C6b: an inadmissible Gauss-point state (rho <= 0 or p <= 0) takes the
        // cell average with zero gradient, for that side at that point
        peval<D, false>(pl, yl, wl, nullptr);
        const bool badl = !(wl[0] > 0.0) || !(pressure<D>(wl, ph.gm1) > 0.0);
        if (badl) ld_vec<NV>(L.W + (size_t)l * NV, wl);
        bool badr = false;
        if (r >= 0) {
            peval<D, false>(pr, yr, wr, nullptr);
            badr = !(wr[0] > 0.0) || !(pressure<D>(wr, ph.gm1) > 0.0);
            if (badr) ld_vec<NV>(L.W + (size_t)r * NV, wr);
        } else {
            ghost<D>(kind, wl, bc, n, wr);
        }
        ap = df_point<D>(wl, wr, n, ph);
        const double pL = pressure<D>(wl, ph.gm1), pR = pressure<D>(wr, ph.gm1);
        const double tau = c1 * dtf + c2 * dtf * fabs(pL - pR) / (pL + pR);
        const TimeC T = time_coeffs(dtf, tau);
        double E[3][3];
        frame<D>(n, E);
        __shared__ double sh_dwc[D * NV * 128];
        double *dWc = sh_dwc + threadIdx.x;
        double Wc[NV], Fl[NV], Wl[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) { Wc[q] = 0.0; Fl[q] = 0.0; Wl[q] = 0.0; }
#pragma unroll
        for (int q = 0; q < D * NV; ++q) dWc[q * blockDim.x] = 0.0;
        // both sides through ONE copy of the side pass (a loop, not unrolled: half the code body of
        // the kernel, fewer instruction-fetch stalls); the half range by its sign at run time
        // all three kinetic passes through one code copy (pass 2: the equilibrium on the summed W^c, slopes)
#pragma unroll 1
        for (int pass = 0; pass < 3; ++pass) {
            double lw[NV], lg[D * NV];
            if (pass < 2) {
                const bool useg = pass == 0 ? !badl : ((r >= 0 && !badr) || (r < 0 && kind == GMG_EXTRAP && !badl));
                if (useg) {
                    const bool lp = pass == 0 || r < 0;
                    peval<D, true>(lp ? pl : pr, lp ? yl : yr, nullptr, gtmp);
                } else {
#pragma unroll
                    for (int q = 0; q < D * NV; ++q) gtmp[q] = 0.0;
                }
                double ws[NV];
#pragma unroll
                for (int q = 0; q < NV; ++q) ws[q] = pass == 0 ? wl[q] : wr[q];
                to_frame<D>(E, ws, gtmp, lw, lg);
            } else {
#pragma unroll
                for (int q = 0; q < NV; ++q) lw[q] = Wc[q];
#pragma unroll
                for (int q = 0; q < D * NV; ++q) lg[q] = dWc[q * blockDim.x];
            }
            kin_pass<D>(lw, lg, T, ph.gm1, ph.K, pass, Wc, dWc, Fl, Wl);
        }
        // back to the global frame, times the Gauss weight
        Fs[0] = w * Fl[0];
        Fs[NV - 1] = w * Fl[NV - 1];
        Ws[0] = w * Wl[0];
        Ws[NV - 1] = w * Wl[NV - 1];
#pragma unroll
        for (int e = 0; e < D; ++e) {
            double a = 0.0, b = 0.0;
#pragma unroll
            for (int c = 0; c < D; ++c) { a += E[c][e] * Fl[1 + c]; b += E[c][e] * Wl[1 + c]; }
            Fs[1 + e] = w * a;
            Ws[1 + e] = w * b;
        }
    }
    // the face's first lane adds its other points in lane order (deterministic); only first lanes
    // change their values, and they read only their own face's lanes (j < its point count)
#pragma unroll
    for (int j = 1; j < G; ++j) {
        const bool take = j < gl.y;
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const double xf = __shfl_down_sync(0xffffffffu, Fs[q], j);
            const double xw = __shfl_down_sync(0xffffffffu, Ws[q], j);
            if (take) { Fs[q] += xf; Ws[q] += xw; }
        }
        const double xa = __shfl_down_sync(0xffffffffu, ap, j);
        if (take) ap *= xa;
    }
    if (gl.y > 0) {
        double *o = H.frec + (size_t)f * kHoRec;
#pragma unroll
        for (int q = 0; q < NV; ++q) { o[q] = S * Fs[q] / dtf; o[NV + q] = Ws[q]; }
        o[2 * NV] = ap;
    }
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
            double rc[4];
            ld4na(H.hrec + (size_t)s * 4, rc);                       // A outward | neighbour, face
            const int f = reinterpret_cast<const int2 *>(&rc[3])->y;
            const int sf = __ldg(H.hface + s);
            const double sg = sf > 0 ? 1.0 : -1.0;
            const double *o = H.frec + (size_t)f * kHoRec;
            double A[D];
#pragma unroll
            for (int k = 0; k < D; ++k) A[k] = rc[k];
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
    case 1: k_ho_recon<D><<<hblk((int64_t)L.n * (D + 2), 256), 256, 0, s>>>(L, H, ph, bc, o.cfl_exp, o.ho_gam0, o.ho_eps); break;
    case 2: k_ho_flux<D><<<hblk((int64_t)H.nlane, 128), 128, 0, s>>>(L, H, ph, bc, o.ho_c1, o.ho_c2); break;
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
