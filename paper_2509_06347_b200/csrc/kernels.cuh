// kernels.cuh -- sm_100a device kernels of libgmg (FP64, no tensor cores:
// the per-cell implicit "block" is a scalar times identity).
//
// Every kernel is HBM/latency bound gather-streaming work (the face kernel
// leans on the FP64 pipe as well); see DESIGN.md §6.  Cell arrays are AoS
// [n][nv] in color-contiguous internal order (40-B records read and written
// as two aligned 128-bit pairs + one scalar, ld_rec / st_rec).  The sweep
// gathers one state W' per neighbour (Wp<D> layout: one 256-bit + one 64-bit
// load in 3D) and per-slot 32-byte records (A outward | S r); the own cell
// reads its (X, c) record (W' formulation).  The residual gather, restriction
// and prolongation walk the cells in the Morton order across colors (gord /
// ginfo).  The test-only P2P concurrency emulation is p2p_emulate.cuh.
#pragma once
#include <cuda_runtime.h>

#include "device_common.cuh"

namespace gmg {

// one half-range side of the first-order KFVS flux (O4), accumulated into F:
// sgn = +1 -> u.n > 0 half of the left state, sgn = -1 -> u.n < 0 half of the
// right state.  lambda = rho/(2p), <u^0> = erfc(-sgn sqrt(lambda) U)/2,
// <u^1> = U<u^0> + sgn e^{-lambda U^2}/(2 sqrt(pi lambda)), recurrence for k+2.
template <int D>
__device__ __forceinline__ void kfvs_side(const Side<D> &s, const double *n, double sgn, const Phys &ph, double *F)
{
    const double lam = 0.5 * s.rho * s.ip;
    const double inv2l = s.p * s.ir;                     // 1 / (2 lambda)
    const double rl = rsqrt(lam);
    const double sl = lam * rl;                          // sqrt(lambda)
    // erfc(x) = e^{-x^2} erfcx(x) (x >= 0), 2 - e^{-x^2} erfcx(-x) (x < 0) with
    // x = -sgn sqrt(lambda) U: the Gaussian e^{-lambda U^2} is shared with <u^1>
    // instead of being recomputed inside erfc
    const double g = exp(-lam * s.U * s.U);
    const double e = g * (0.28209479177387814 * rl);   // e^{-lambda U^2} / (2 sqrt(pi lambda))
    const double x = -sgn * sl * s.U;
    const double gx = g * erfcx(fabs(x));
    const double m0 = 0.5 * (x >= 0.0 ? gx : 2.0 - gx);
    const double m1 = s.U * m0 + sgn * e;
    const double m2 = s.U * m1 + inv2l * m0;
    const double m3 = s.U * m2 + 2.0 * inv2l * m1;
    const double rm1 = s.rho * m1, rm2 = s.rho * m2;
    F[0] += rm1;
#pragma unroll
    for (int k = 0; k < D; ++k) F[1 + k] += rm2 * n[k] + rm1 * (s.u[k] - s.U * n[k]);
    F[D + 1] += 0.5 * s.rho * (m3 + m1 * (s.u2 - s.U * s.U + ((double)(D - 1) + ph.K) * inv2l));
}

// ---------------------------------------------------------------------------
// Face kernel (a6 + a10 per face): r_f = omega (|u.n| + a) of the average
// state; with FLUX also S F_f (KFVS) and alpha_f^{M_f} (DF helper).  The
// state is read with a stride (NV for W; STRIDE 0 = a W_lin state array, Wp<D> layout).
// Output: one 64-byte record per face, Frec = (S F[nv] | S r | alpha^M | 0..),
// written with two 256-bit stores.
// ---------------------------------------------------------------------------
constexpr int kFaceRec = 8;
template <int D> struct FR { static constexpr int SR = D + 2, AM = D + 3; };

// PREP: also write the sweep slot records (A outward | S r) of the face's
// cells -- whole 32-byte records, so no partial-sector update (the gather
// used to patch S r into each slot)
template <int D, bool FLUX, int STRIDE, bool DF, bool PREP>
__global__ void __launch_bounds__(256, 4) k_face(DevLevel L, const double *__restrict__ Wsrc, Phys ph, BCs bc, int need_sr)
{
    pdl_launch_dependents();
    constexpr int NV = D + 2;
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= L.nf) { pdl_wait(); return; }
    // static face data before the PDL wait (overlaps the predecessor's tail), states after it
    const int l = __ldg(L.fl + f), r = __ldg(L.fr + f);
    double A[D], S2 = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) { A[k] = __ldg(L.fA + (size_t)k * L.nf + f); S2 += A[k] * A[k]; }
    const int M = DF ? (int)L.fM[f] : 0;                              // Gauss points of the face (DF exponent)
    const int2 es = PREP ? __ldg(L.fslot + f) : make_int2(-1, -1);   // its sweep slots (prepare)
    pdl_wait();
    const double iS = rsqrt(S2), S = S2 * iS;
    double n[D];
#pragma unroll
    for (int k = 0; k < D; ++k) n[k] = A[k] * iS;
    double wl[NV], wr[NV];
    if constexpr (STRIDE == 0) {   // a state array (Wp layout): W_lin
        ld_state<D>(Wsrc, (size_t)L.n_loc, l, wl);
        if (r >= 0) ld_state<D>(Wsrc, (size_t)L.n_loc, r, wr);
    } else {
        static_assert(STRIDE == NV, "W arrays are [n][nv]");
        ld_rec<NV, true>(Wsrc, l, wl);
        if (r >= 0) ld_rec<NV, true>(Wsrc, r, wr);
    }
    if (r < 0) ghost<D>(bc.kind[-r - 1], wl, bc, n, wr);

    double out[kFaceRec];
#pragma unroll
    for (int q = 0; q < kFaceRec; ++q) out[q] = 0.0;
    // spectral radius of the conservative average (O6, reading A5); launches whose
    // gather uses no Sigma (restricted residual, R + F, norms) skip it
    if (PREP || need_sr) {
        double wb[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) wb[q] = 0.5 * (wl[q] + wr[q]);
        const double ib = 1.0 / wb[0];
        double mb = 0.0, m2 = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) { mb += wb[1 + k] * n[k]; m2 += wb[1 + k] * wb[1 + k]; }
        const double pb = ph.gm1 * (wb[D + 1] - 0.5 * m2 * ib);
        out[FR<D>::SR] = S * (ph.omega * (fabs(mb * ib) + sqrt(ph.gamma * pb * ib)));
    }
    if (FLUX) {
        const Side<D> sl = side_of<D>(wl, n, ph.gm1), sr = side_of<D>(wr, n, ph.gm1);
        kfvs_side<D>(sl, n, 1.0, ph, out);
        kfvs_side<D>(sr, n, -1.0, ph, out);
#pragma unroll
        for (int q = 0; q < NV; ++q) out[q] *= S;
    }
    if (FLUX && DF) {   // only the fine residual whose alpha is consumed evaluates the DF helper
        const Side<D> sl = side_of<D>(wl, n, ph.gm1), sr = side_of<D>(wr, n, ph.gm1);
        // DF helper (O5): D = |dp|/p_l + |dp|/p_r + (dMa_n)^2 + |dMa_t|^2, alpha = 1/(1+D^2)
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
        const double af = 1.0 / (1.0 + Dv * Dv);
        double aM = 1.0;
        for (int g = 0; g < M; ++g) aM *= af;
        out[FR<D>::AM] = aM;
    }
    if (PREP) {
        const double sr = out[FR<D>::SR];
        if (es.x >= 0) {
            const double v[4] = {A[0], A[1], D == 3 ? A[D - 1] : sr, D == 3 ? sr : 0.0};
            st4(L.sRe + (size_t)es.x * kSlotRec, v);
        }
        if (es.y >= 0) {
            const double v[4] = {-A[0], -A[1], D == 3 ? -A[D - 1] : sr, D == 3 ? sr : 0.0};
            st4(L.sRe + (size_t)es.y * kSlotRec, v);
        }
    }
    double *o = L.Frec + (size_t)f * kFaceRec;
    // without the flux only S r (in the second 32-B chunk) is read back: the first chunk is not written
    if (FLUX)
        asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(o), "d"(out[0]), "d"(out[1]), "d"(out[2]), "d"(out[3])
                     : "memory");
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(o + 4), "d"(out[4]), "d"(out[5]), "d"(out[6]),
                 "d"(out[7])
                 : "memory");
}

// ---------------------------------------------------------------------------
// Cell gather (a6, a7, a9, a10, a16): per cell over its face slots.
// ---------------------------------------------------------------------------
// FL >= 0: the flag set as a compile-time constant (the V-cycle's fixed
// combinations: dead paths and their registers drop out); FL = -1: a.flags
template <int D, int FL>
__global__ void __launch_bounds__(256) k_gather(DevLevel L, GArgs a)
{
    const int flags = FL >= 0 ? FL : a.flags;
    pdl_launch_dependents();
    constexpr int NV = D + 2;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;   // gather position (ginfo.z: the cell)
    double R[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) R[q] = 0.0;
    // static slot data before the PDL wait (overlaps the predecessor's tail), face records after it
    int4 gi = make_int4(0, 0, 0, 0);
    if (t < L.n) gi = __ldg(L.ginfo + t);
    const int i = gi.z;
    // the first face id (static) before the wait as well; each next one a slot ahead (one round trip per slot)
    int sfn = (t < L.n && (gi.y & 0xffff) > 0) ? __ldg(L.gface + gi.x) : 0;
    pdl_wait();
    // the cell's one per-cell input of the epilogue (W for G_COPY_W, Rs for G_SET_F, F for G_ADD_F, the
    // explicit state for G_EXPLICIT) is loaded before the slot loop: its latency hides under the gathers,
    // and the epilogue's stores no longer wait on loads the compiler cannot hoist above them (aliasing)
    const int pk = (flags & G_COPY_W) ? G_COPY_W : (flags & G_SET_F) ? G_SET_F
                 : ((flags & G_WRITE_RT) && (flags & G_ADD_F)) ? G_ADD_F : (flags & G_EXPLICIT) ? G_EXPLICIT : 0;
    double pre[NV];
    if (t < L.n && pk) {
        const double *src = pk == G_COPY_W ? L.W : pk == G_SET_F ? L.Rs : pk == G_ADD_F ? L.F : a.Wexp;
        ld_rec<NV>(src, i, pre);
    }
    if (t < L.n) {
        // (gather base, all slots | interior slots << 16, cell, 0): one 16-byte load
        const int gb = gi.x, nt = gi.y & 0xffff;
        double sig = 0.0, al = 1.0;
        // coarse prepare: the restricted alpha is needed after the loop -- requested now
        const double a0 = ((flags & G_PREPARE) && !(flags & (G_BETA | G_ALPHA))) ? L.alpha[i] : 1.0;
        for (int s = 0; s < nt; ++s) {
            const int sf = sfn;
            if (s + 1 < nt) sfn = __ldg(L.gface + gb + kChunk * (s + 1));
            const int f = (sf > 0 ? sf : -sf) - 1;
            const double *fr = L.Frec + (size_t)f * kFaceRec;
            double c1[4];
            ld4na(fr + 4, c1);   // 3D: SF4, Sr, alpha^M, 0   2D: Sr, alpha^M, 0, 0 (no L1 allocation: the other
                                 // cell of the face reads the record much later, from L2)
            const double srf = c1[FR<D>::SR - 4];
            sig += srf;
            if (flags & G_FLUX) {
                double c0[4];
                ld4na(fr, c0);
                const double sg = sf > 0 ? 1.0 : -1.0;
#pragma unroll
                for (int q = 0; q < 4; ++q) R[q] += sg * c0[q];
                if (D == 3) R[NV - 1] += sg * c1[0];
                al *= c1[FR<D>::AM - 4];
            }
        }
        if (flags & G_ALPHA) L.alpha[i] = al;
        if (flags & G_SIGMA) L.sigma[i] = sig;
        if (flags & G_PREPARE) {
            const double ai = (flags & G_BETA) ? a.beta : ((flags & G_ALPHA) ? al : a0);
            // D = alpha (V/Dt_imp + Sigma/2) + (1 - alpha) V/Dt_exp (O6, A2, A3); c = alpha / (2 D)
            const double Dg = ai * (sig / a.cfl_imp + 0.5 * sig) + (1.0 - ai) * (sig / a.cfl_exp);
            const double iD = 1.0 / Dg;
            const double dc[2] = {iD, 0.5 * ai * iD};
            st2(L.dc + 2 * (size_t)i, dc);
        }
        const size_t o = (size_t)i * NV;
        if (flags & G_COPY_W) st_state<D>(L.wlin, (size_t)L.n_loc, i, pre);
        if (flags & G_SET_F) {
            if (pk == G_SET_F) {
                double v[NV];
#pragma unroll
                for (int q = 0; q < NV; ++q) v[q] = pre[q] - R[q];
                st_rec<NV>(L.F, i, v);
            } else {
#pragma unroll
                for (int q = 0; q < NV; ++q) L.F[o + q] = L.Rs[o + q] - R[q];
            }
        }
        if (flags & G_WRITE_RT) {
            if (flags & G_ADD_F) {
                if (pk == G_ADD_F) {
                    double v[NV];
#pragma unroll
                    for (int q = 0; q < NV; ++q) v[q] = R[q] + pre[q];
                    st_rec<NV>(L.Rt, i, v);
                } else {
#pragma unroll
                    for (int q = 0; q < NV; ++q) L.Rt[o + q] = R[q] + L.F[o + q];
                }
            } else {
                st_rec<NV>(L.Rt, i, R);
            }
        }
        if (flags & G_EXPLICIT) {
            const double c = a.cfl_exp / sig;
            if (pk == G_EXPLICIT) {
                double v[NV];
#pragma unroll
                for (int q = 0; q < NV; ++q) v[q] = pre[q] - c * R[q];
                st_rec<NV>(a.Wexp, i, v);
            } else {
#pragma unroll
                for (int q = 0; q < NV; ++q) a.Wexp[o + q] = a.Wexp[o + q] - c * R[q];
            }
        }
    }
    if (flags & G_NORM) {
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
            a.partial[(size_t)blockIdx.x * NV + threadIdx.x] = v;
        }
    }
}

// deterministic reduction of one domain's norm partials -> sumsq[q]: 1024
// threads, each sums a fixed strided subset of the blocks for all nv
// components at once, then a fixed shuffle + shared-memory tree (the same
// order on every run)
// fin (one domain, one rank: nothing to combine): also writes the history
// entry -- sqrt of the same sums, the bits k_norm_hist would write
__global__ void __launch_bounds__(1024) k_norm_sum(const double *__restrict__ partial, int nblocks, int nv,
                                                   double *sumsq, double *hist, int hist_cap, int *flags, int fin)
{
    pdl_enter();
    __shared__ double sh[32][5];
    double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int b = threadIdx.x; b < nblocks; b += 1024)
        for (int q = 0; q < nv; ++q) v[q] += partial[(size_t)b * nv + q];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int q = 0; q < nv; ++q) {
        for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_down_sync(0xffffffffu, v[q], o);
        if (lane == 0) sh[wid][q] = v[q];
    }
    __syncthreads();
    if (wid == 0) {
        const int idx = fin ? flags[0] : 0;
        for (int q = 0; q < nv; ++q) {
            double t = sh[lane][q];
            for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
            if (lane == 0) {
                sumsq[q] = t;
                if (fin) {
                    const double v = sqrt(t);
                    if (idx < hist_cap) hist[(size_t)idx * nv + q] = v;
                    if (!isfinite(v)) flags[1] = 1;
                }
            }
        }
        if (fin && lane == 0) flags[0] = idx + 1;
    }
}

// domains' sums (in domain order; already all-reduced across ranks) -> hist[counter][q]
__global__ void k_norm_hist(const double *__restrict__ sumsq, int ndom, int nv, double *hist, int hist_cap,
                            int *flags)
{
    pdl_enter();
    if (threadIdx.x != 0) return;
    const int idx = flags[0];
    for (int q = 0; q < nv; ++q) {
        double s = 0.0;
        for (int d = 0; d < ndom; ++d) s += sumsq[(size_t)d * nv + q];
        const double v = sqrt(s);
        if (idx < hist_cap) hist[(size_t)idx * nv + q] = v;
        if (!isfinite(v)) flags[1] = 1;
    }
    flags[0] = idx + 1;
}

// ---------------------------------------------------------------------------
// Halo exchange helpers (a13): pack owned cells' values, unpack into ghosts.
// Element k of a buffer holds ncomp doubles of cell idx[k]; src/dst are cell
// arrays with the given stride/offset (W', W_lin or W).  dst2 (nullable)
// receives a second copy with the same layout (ghost W' = W_lin).
// ---------------------------------------------------------------------------
// element q of cell c of an array: AoS (stride, offset) when split == 0, else
// a 3D split state array of `split` cells ([split][4] then [split], Wp<3>)
__device__ __forceinline__ size_t elem_at(size_t c, int q, int stride, int offset, int split)
{
    if (split) return q < 4 ? 4 * c + q : 4 * (size_t)split + c;
    return c * stride + offset + q;
}
__global__ void k_pack(int count, const int *__restrict__ idx, const double *__restrict__ src, int stride,
                       int offset, int ncomp, double *__restrict__ buf, int split)
{
    pdl_enter();
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= count) return;
    const size_t c = (size_t)idx[k];
    for (int q = 0; q < ncomp; ++q) buf[(size_t)k * ncomp + q] = src[elem_at(c, q, stride, offset, split)];
}
__global__ void k_unpack(int count, const int *__restrict__ idx, const double *__restrict__ buf, double *dst,
                         int stride, int offset, int ncomp, double *dst2, int split)
{
    pdl_enter();
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= count) return;
    const size_t c = (size_t)idx[k];
    for (int q = 0; q < ncomp; ++q) {
        const double v = buf[(size_t)k * ncomp + q];
        const size_t o = elem_at(c, q, stride, offset, split);
        dst[o] = v;
        if (dst2) dst2[o] = v;
    }
}


// ghost records from the (current) ghost state: W_lin = W' = W
template <int D>
__global__ void k_ghost_wlin(int n, int n_loc, const double *__restrict__ W, double *wlin, double *wp)
{
    pdl_enter();
    const int g = n + blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n_loc) return;
    double w[D + 2];
#pragma unroll
    for (int q = 0; q < D + 2; ++q) w[q] = W[(size_t)g * (D + 2) + q];
    st_state<D>(wlin, n_loc, g, w);
    st_state<D>(wp, n_loc, g, w);
}
// ghost states after a smoothing step: W = W' (already exchanged)
template <int D>
__global__ void k_ghost_w(int n, int n_loc, const double *__restrict__ wp, double *W)
{
    pdl_enter();
    const int g = n + blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n_loc) return;
    double w[D + 2];
    ld_state<D>(wp, n_loc, g, w);
#pragma unroll
    for (int q = 0; q < D + 2; ++q) W[(size_t)g * (D + 2) + q] = w[q];
}

// ---------------------------------------------------------------------------
// MC-LU-SGS sweep over one color block (a11 / a12): Eq.(gpu-forward-
// relaxation) / Eq.(gpu-backward-relaxation) P:536-551 with reading A7
// (every half-sweep reads all neighbours' current increments),
//   dW_i = -( Rt_i + alpha_i/2 sum_j [T(W_j+dW_j; A) - T(W_j; A) - S r dW_j] ) / D_i,
// A = sigma S n outward from i (the Euler flux is linear in its normal,
// S T(W; n) = T(W; A)), evaluated in the W' formulation (DESIGN.md §6,
// reading B4).  With W'_j = W_j + dW_j the W-only part
// P_i = sum_j [T(W_j; A) - S r W_j] is fixed during a smoothing step, so
//   W'_i = X_i - c_i sum_j [T(W'_j; A) - S r W'_j],
//   X_i  = W_i - Rt_i / D_i + c_i P_i,   c_i = alpha_i / (2 D_i):
// a neighbour contributes ONE flux evaluation of ONE state (two 256-bit loads
// in 3D, one in 2D) instead of two evaluations of (W, dW).  The first forward
// half-sweep of a step (FF) evaluates P_i on the way -- every neighbour's
// W_lin -- and stores X_i; its later-color owned neighbours still hold
// W' = W_lin, so only the lower-color (and ghost) neighbours contribute a
// difference [T(W') - S r W'] - [T(W) - S r W], read from W' and W_lin.
// Same-color cells never neighbour each other, so a color launch reads no
// state it writes (non-coherent loads are safe).
// LPC lanes per cell: each lane gathers its slots' neighbours (one dependent
// index -> record round trip), partial sums are combined with warp shuffles.
// ---------------------------------------------------------------------------
// t = T(w; A) - Sr w  (3D: 1 division, 27 FMA-class operations)
template <int D>
__device__ __forceinline__ void flux_rw(const double *w, const double *A, double Sr, double gm1, double *t)
{
    const double ir = 1.0 / w[0];
    double mA = 0.0, m2 = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        mA += w[1 + k] * A[k];
        m2 += w[1 + k] * w[1 + k];
    }
    const double p = gm1 * (w[D + 1] - 0.5 * m2 * ir);
    const double U = mA * ir;
    t[0] = mA - Sr * w[0];
#pragma unroll
    for (int k = 0; k < D; ++k) t[1 + k] = (w[1 + k] * U + p * A[k]) - Sr * w[1 + k];
    t[D + 1] = (w[D + 1] + p) * U - Sr * w[D + 1];
}

struct SweepArgs {
    int cbeg, cend;            // cells [cbeg, cend) of one color block (or its boundary / interior part)
    int lo, n_own;             // FF: owned neighbours j < lo are of earlier colors; j >= n_own are ghosts
    int n_loc;                 // cells of the state arrays (owned + ghosts)
    double gm1;
    const int2 *sinfo;         // [n] (first slot entry, interior slots)
    const int *sJe;            // [ns] neighbour
    const double *sRe;         // [ns][4] (A outward | S r)
    double *wp;                // W' (state array of n_loc cells, Wp<D> layout)
    double *xr;                // [n][kXr] (X, c)
    const double *wlin;        // W_lin (same layout)     (FF)
    const double *rhs;         // [n][nv] right-hand side Rt (FF)
    const double *dc;          // [n][2] (1/D, c)          (FF)
    double *Wout;              // [n][nv] or null: W = W' (last backward half-sweep)
    int rev;                   // 1: visit the cells from the end of the block (order only)
};

// Fused halo (gmg_options.p2p): the sweep that computes a boundary cell's W'
// also stores it straight into the ghost record of every rank (domain) that
// ghosts the cell, over peer memory (NVLink P2P between GPUs; plain device
// memory between the domains of one process).  Ordering between phases:
// every rank counts its completed color phases (ctl[0]); the last block of a
// sweep launch fences the stores system-wide and publishes the new count
// into each peer's flags[my rank] (st.release.sys); the next launch waits
// until every peer's count has reached its own (ld.acquire.sys) -- so a peer
// never reads a ghost before its phase's values landed, and never overwrites
// one that is still being read (each side waits for the other).
struct P2PArgs {
    const int *off, *k, *g;      // per owned cell: remote targets (peer slot, ghost local index), CSR
    double *const *peer_wp;      // [peer slot] the peer's W' array on this level
    const int *peer_nloc;        // [peer slot] the peer's cells (owned + ghosts) on this level
    int np;                      // peers on this level (0: count phases only)
    const int *wait_rank;        // [np] their ranks
    int *const *sig;             // [np] &peer.flags[my rank]
    const int *flags;            // [nranks] phase counts published by the peers
    int *ctl;                    // [0] phases completed, [1] blocks done, [2] wait timeout
};

template <int D, bool P2P>
__device__ __forceinline__ void p2p_store(const P2PArgs &p, int i, const double *w)
{
    if constexpr (P2P) {
        for (int m = p.off[i]; m < p.off[i + 1]; ++m) {
            double *r = p.peer_wp[p.k[m]];
            const size_t g = (size_t)p.g[m], nl = (size_t)p.peer_nloc[p.k[m]];
#pragma unroll
            for (int q = 0; q < 4; ++q) r[4 * g + q] = w[q];
            if constexpr (D == 3) r[4 * nl + g] = w[4];
        }
    }
}

template <bool CG, bool NA = false>
__device__ __forceinline__ void ld2x(const double *p, double *v)
{
    if constexpr (CG) ld2cg(p, v);
    else if constexpr (NA) ld2na(p, v);
    else ld2nc(p, v);
}

// the cells [cbeg, cend) x LPC lanes, grid-stride from thread gt0 with nthr
// threads (a launch sized to exactly one resident wave has no partial last
// wave), ascending or (a.rev, backward half-sweeps) descending; PDL: the slot range and first neighbour index (static during a
// smoothing step) are loaded before griddepcontrol.wait, so they overlap the
// previous phase's tail, and the records after it
// FF: 0 = a plain phase, 1 = a first-forward phase, 2 = the first-forward
// phase of the first color with no ghosts (no earlier-color neighbour: no W'
// gathers, W' = W - Rt/D)
template <int D, int LPC, int FF, bool CG, bool P2P, int WO = -1>
__device__ __forceinline__ void sweep_cells(const SweepArgs &a, const P2PArgs &p, int gt0, int nthr, bool pdl)
{
    constexpr int NV = D + 2;
    const size_t nl = (size_t)a.n_loc;
    const int total = (a.cend - a.cbeg) * LPC;
    const int rounds = (total + nthr - 1) / nthr;
    for (int r = 0; r < rounds; ++r) {
        const int g = gt0 + r * nthr;
        const int sub = g % LPC;
        const bool valid = g / LPC < a.cend - a.cbeg;
        // rev: the block from its end (backward half-sweeps; cells of one color are independent)
        const int i = a.rev ? a.cend - 1 - g / LPC : a.cbeg + g / LPC;
        double acc[NV], accP[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) { acc[q] = 0.0; accP[q] = 0.0; }
        if (valid) {
            const int2 sd = __ldg(a.sinfo + i);     // (first slot, degree) in one 8-byte load
            const int e1 = sd.x + sd.y;
            int e = sd.x + sub;
            int j = e < e1 ? __ldg(a.sJe + e) : 0;
            if (pdl && r == 0) pdl_wait();
            for (; e < e1; e += LPC) {
                const int jn = e + LPC < e1 ? __ldg(a.sJe + e + LPC) : 0;
                double sr[4];
                ld4na(a.sRe + (size_t)e * kSlotRec, sr);   // read once: not allocated in L1
                if constexpr (FF) {
                    // both states of an earlier-color neighbour requested before either flux (one round trip)
                    const bool upd = FF == 1 && (j < a.lo || j >= a.n_own);
                    double wl[NV], w1[NV], t0[NV];
                    ld_state<D, CG>(a.wlin, nl, j, wl);
                    if (upd) ld_state<D, CG>(a.wp, nl, j, w1);
                    flux_rw<D>(wl, sr, sr[D], a.gm1, t0);
#pragma unroll
                    for (int q = 0; q < NV; ++q) accP[q] += t0[q];
                    if (upd) {
                        double t1[NV];
                        flux_rw<D>(w1, sr, sr[D], a.gm1, t1);
#pragma unroll
                        for (int q = 0; q < NV; ++q) acc[q] += t1[q] - t0[q];
                    }
                } else {
                    double w1[NV], t1[NV];
                    ld_state<D, CG, true>(a.wp, nl, j, w1);
                    flux_rw<D>(w1, sr, sr[D], a.gm1, t1);
#pragma unroll
                    for (int q = 0; q < NV; ++q) acc[q] += t1[q];
                }
                j = jn;
            }
        }
        if (LPC > 1) {
#pragma unroll
            for (int o = LPC / 2; o > 0; o >>= 1) {
#pragma unroll
                for (int q = 0; q < NV; ++q) {
                    acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
                    if constexpr (FF) accP[q] += __shfl_xor_sync(0xffffffffu, accP[q], o);
                }
            }
        }
        if (valid && sub == 0) {
            double wn[NV], x[kXr];
            if constexpr (FF) {
                double wl[NV], rr[NV], dd[2];
                ld_state<D, CG>(a.wlin, nl, i, wl);
#pragma unroll
                for (int q = 0; q < NV; ++q) rr[q] = CG ? __ldcg(a.rhs + (size_t)i * NV + q) : __ldcs(a.rhs + (size_t)i * NV + q);
                ld2x<CG>(a.dc + 2 * (size_t)i, dd);
                const double invD = dd[0], c = dd[1];
#pragma unroll
                for (int q = 0; q < NV; ++q) {
                    const double b = wl[q] - rr[q] * invD;   // W - Rt/D
                    x[q] = b + c * accP[q];                  // X = W - Rt/D + c P
                    wn[q] = b - c * acc[q];                  // W' = W - Rt/D - c sum_lower (...)
                }
                x[NV] = c;
                if constexpr (NV + 1 < kXr) x[NV + 1] = 0.0;
                double *xo = a.xr + (size_t)i * kXr;
                st2(xo, x);
                st2(xo + 2, x + 2);
                st2(xo + 4, x + 4);
            } else {
                const double *xi = a.xr + (size_t)i * kXr;
                ld2x<CG, true>(xi, x);
                ld2x<CG, true>(xi + 2, x + 2);
                ld2x<CG, true>(xi + 4, x + 4);
                const double c = x[NV];
#pragma unroll
                for (int q = 0; q < NV; ++q) wn[q] = x[q] - c * acc[q];
            }
            st_state<D>(a.wp, nl, i, wn);
            p2p_store<D, P2P>(p, i, wn);
            // WO: the W write of the last backward phase known at compile time (1 / 0), -1: a.Wout decides
            if (WO == 1 || (WO < 0 && a.Wout)) st_rec<NV>(a.Wout, i, wn);
        }
    }
    if (pdl) pdl_wait();   // threads without a cell: nothing may run past the predecessor
}

// the sweep launch: 128-thread blocks, 9 per SM (FF, with its second set of
// accumulators, and the first color's FF, without W' gathers: 7), grid = one
// resident wave
template <int D, int LPC, int FF, int WO>
__global__ void __launch_bounds__(128, FF ? 7 : 9) k_sweep(SweepArgs a)
{
    pdl_launch_dependents();                       // the next phase may start its static prologue now
    sweep_cells<D, LPC, FF, false, false, WO>(a, P2PArgs{}, blockIdx.x * blockDim.x + threadIdx.x,
                                              gridDim.x * blockDim.x, true);
}

__device__ __forceinline__ int ld_acquire_sys(const int *p)
{
    int v;
    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(int *p, int v)
{
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// the sweep with the fused halo (see P2PArgs).  Launched for every phase on
// every rank, also with no cells, so that all phase counts advance together.
template <int D, int LPC, bool FF>
__global__ void __launch_bounds__(256, FF ? 3 : 4) k_sweep_p2p(SweepArgs a, P2PArgs p)
{
    __shared__ int s_bad;
    if (threadIdx.x == 0) {
        s_bad = 0;
        const int target = *(volatile int *)p.ctl;       // phases this rank completed
        for (int t = 0; t < p.np && !s_bad; ++t) {
            for (int spin = 0; ld_acquire_sys(p.flags + p.wait_rank[t]) < target; ++spin) {
                if (spin > (1 << 24) || *(volatile int *)(p.ctl + 2)) { atomicExch(p.ctl + 2, 1); s_bad = 1; break; }
                __nanosleep(64);
            }
        }
    }
    __syncthreads();
    if (!s_bad)
        sweep_cells<D, LPC, FF, false, true>(a, p, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x, false);
    // publish: every block orders its peer stores before its arrival on the
    // done counter (gpu scope); the last block to arrive -- which has observed
    // all arrivals -- fences at system scope and releases the new phase count
    // to the peers, so by cumulativity every block's stores precede the flag
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        if (atomicAdd(p.ctl + 1, 1) == (int)gridDim.x - 1) {
            p.ctl[1] = 0;
            const int ph = p.ctl[0] + 1;
            p.ctl[0] = ph;
            __threadfence_system();
            for (int t = 0; t < p.np; ++t) st_release_sys(p.sig[t], ph);
        }
    }
}

// restriction to a coarse level (a8, A15): W0 into the coarse
// W_lin record, Res*, alpha = min over the children
template <int D>
__global__ void __launch_bounds__(256) k_restrict(DevLevel C, DevLevel Fn, const double *__restrict__ Wf,
                                                  const double *__restrict__ Rf)
{
    pdl_launch_dependents();
    constexpr int NV = D + 2;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= C.n) { pdl_wait(); return; }
    // static hierarchy data before the PDL wait, the states after it
    const int c = __ldg(C.gord + t);   // coarse cells in the Morton order across colors: the children's
                                       // records are read as one ordered stream per fine color block
    const int k0 = __ldg(C.child + c), k1 = __ldg(C.child + C.n + c);
    const double V0 = __ldg(Fn.vol + k0);
    const double V1 = k1 >= 0 ? __ldg(Fn.vol + k1) : 0.0;
    const double vc = __ldg(C.vol + c);
    pdl_wait();
    double w[NV], r[NV], wk[NV], rk[NV];
    double a = Fn.alpha[k0];
    ld_rec<NV, true>(Wf, k0, wk);
    ld_rec<NV, true>(Rf, k0, rk);
#pragma unroll
    for (int q = 0; q < NV; ++q) { w[q] = V0 * wk[q]; r[q] = rk[q]; }
    if (k1 >= 0) {
        ld_rec<NV, true>(Wf, k1, wk);
        ld_rec<NV, true>(Rf, k1, rk);
#pragma unroll
        for (int q = 0; q < NV; ++q) { w[q] = w[q] + V1 * wk[q]; r[q] = r[q] + rk[q]; }
        a = fmin(a, Fn.alpha[k1]);
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) w[q] = w[q] / vc;
    st_rec<NV>(C.Rs, c, r);
    st_state<D>(C.wlin, (size_t)C.n_loc, c, w);
    C.alpha[c] = a;
}

// DF-limited prolongation, both levels fused (a15, A13, A14):
//   W_0 += alpha_0 ((W_1 - W0_1) + alpha_1 (W_2 - W0_2)[parent_1])[parent_0]
template <int D>
__global__ void __launch_bounds__(256) k_prolong(DevLevel F0, DevLevel C1, DevLevel C2, int nl)
{
    pdl_launch_dependents();
    constexpr int NV = D + 2;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= F0.n) { pdl_wait(); return; }
    // static hierarchy data before the PDL wait, the states after it
    const int i = __ldg(F0.gord + t);   // fine cells in the Morton order across colors (see k_restrict)
    const int p = __ldg(F0.parent + i);
    const int pp = nl >= 3 ? __ldg(C1.parent + p) : 0;
    pdl_wait();
    double corr[NV], w0[NV], wc[NV];
    ld_state<D>(C1.wlin, (size_t)C1.n_loc, p, w0);
    ld_rec<NV, true>(C1.W, p, wc);
#pragma unroll
    for (int q = 0; q < NV; ++q) corr[q] = wc[q] - w0[q];
    if (nl >= 3) {
        const double a1 = C1.alpha[p];
        ld_state<D>(C2.wlin, (size_t)C2.n_loc, pp, w0);
        ld_rec<NV, true>(C2.W, pp, wc);
#pragma unroll
        for (int q = 0; q < NV; ++q) corr[q] += a1 * (wc[q] - w0[q]);
    }
    const double a0 = F0.alpha[i];
    double wf[NV];
    ld_rec<NV>(F0.W, i, wf);
#pragma unroll
    for (int q = 0; q < NV; ++q) wf[q] += a0 * corr[q];
    st_rec<NV>(F0.W, i, wf);
}

// ---------------------------------------------------------------------------
// natural SoA [ncomp][N]  <->  local AoS (stride, offset), n local cells
__global__ void k_to_internal(int n, int N, int ncomp, const int *__restrict__ perm, const double *__restrict__ src,
                              double *__restrict__ dst, int stride, int offset)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int nat = perm[i];
    for (int q = 0; q < ncomp; ++q) dst[(size_t)i * stride + offset + q] = src[(size_t)q * N + nat];
}
__global__ void k_to_natural(int n, int N, int ncomp, const int *__restrict__ perm, const double *__restrict__ src,
                             double *__restrict__ dst, int stride, int offset)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int nat = perm[i];
    for (int q = 0; q < ncomp; ++q) dst[(size_t)q * N + nat] = src[(size_t)i * stride + offset + q];
}
// a state array (Wp layout, nloc cells) minus another (nullable) over n owned cells -> natural SoA [ncomp][N]
// (W0 = W_lin, dW = W' - W_lin; gmg_get_level_field, gmg_smooth)
__global__ void k_state_to_natural(int n, int N, int ncomp, const int *__restrict__ perm, const double *__restrict__ a,
                                   const double *__restrict__ b, int nloc, double *__restrict__ dst)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int nat = perm[i];
    const int split = ncomp == 5 ? nloc : 0;
    for (int q = 0; q < ncomp; ++q) {
        const size_t o = elem_at((size_t)i, q, 4, 0, split);
        dst[(size_t)q * N + nat] = b ? a[o] - b[o] : a[o];
    }
}
// owned-compact [ncomp][n] (SoA, local owned order) <-> AoS [n][ncomp]
__global__ void k_soa_to_aos(int n, int ncomp, const double *__restrict__ src, double *__restrict__ dst)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int q = 0; q < ncomp; ++q) dst[(size_t)i * ncomp + q] = src[(size_t)q * n + i];
}
__global__ void k_aos_to_soa(int n, int ncomp, const double *__restrict__ src, double *__restrict__ dst)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int q = 0; q < ncomp; ++q) dst[(size_t)q * n + i] = src[(size_t)i * ncomp + q];
}
__global__ void k_fill(int n, double *p, double v)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

}  // namespace gmg
