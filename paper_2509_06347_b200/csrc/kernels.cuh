// kernels.cuh -- sm_100a device kernels of libgmg (FP64, no tensor cores:
// the per-cell implicit "block" is a scalar times identity).
//
// Every kernel is HBM/latency bound gather-streaming work; see DESIGN.md
// "Kernels and rooflines".  Cell arrays are AoS [n][nv] in color-contiguous
// internal order.  The sweep reads a per-cell 32-byte aligned record
// Rec<D> = (W_lin | dW | 1/D | alpha/2), 96 bytes, with three 256-bit loads
// per neighbour, and per-slot 32-byte records (A outward | S r).  The sweep
// variants that were measured and lost, and the test-only P2P concurrency
// emulation, live in kernels_tried.cuh.
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
// state is read with a stride (NV for W, Rec<D>::STRIDE for the record).
// Output: one 64-byte record per face, Frec = (S F[nv] | S r | alpha^M | 0..),
// written with two 256-bit stores.
// ---------------------------------------------------------------------------
constexpr int kFaceRec = 8;
template <int D> struct FR { static constexpr int SR = D + 2, AM = D + 3; };

// PREP: also write the sweep slot records (A outward | S r) of the face's
// cells -- whole 32-byte records, so no partial-sector update (the gather
// used to patch S r into each slot)
template <int D, bool FLUX, int STRIDE, bool DF, bool PREP>
__global__ void __launch_bounds__(256, DF ? 3 : 4) k_face(DevLevel L, const double *__restrict__ Wsrc, Phys ph, BCs bc)
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
    pdl_wait();
    const double iS = rsqrt(S2), S = S2 * iS;
    double n[D];
#pragma unroll
    for (int k = 0; k < D; ++k) n[k] = A[k] * iS;
    double wl[NV], wr[NV];
    ld_vec<NV>(Wsrc + (size_t)l * STRIDE, wl);
    if (r >= 0) ld_vec<NV>(Wsrc + (size_t)r * STRIDE, wr);
    else ghost<D>(bc.kind[-r - 1], wl, bc, n, wr);

    double out[kFaceRec];
#pragma unroll
    for (int q = 0; q < kFaceRec; ++q) out[q] = 0.0;
    // spectral radius of the conservative average (O6, reading A5)
    {
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
        const int M = L.fM[f];
        for (int g = 0; g < M; ++g) aM *= af;
        out[FR<D>::AM] = aM;
    }
    if (PREP) {
        const int2 es = __ldg(L.fslot + f);
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
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(o), "d"(out[0]), "d"(out[1]), "d"(out[2]), "d"(out[3])
                 : "memory");
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(o + 4), "d"(out[4]), "d"(out[5]), "d"(out[6]),
                 "d"(out[7])
                 : "memory");
}

// ---------------------------------------------------------------------------
// Cell gather (a6, a7, a9, a10, a16): per cell over its face slots.
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256) k_gather(DevLevel L, GArgs a)
{
    pdl_launch_dependents();
    constexpr int NV = D + 2;
    using RC = Rec<D>;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double R[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) R[q] = 0.0;
    // static slot data before the PDL wait (overlaps the predecessor's tail), face records after it
    int4 gi = make_int4(0, 0, 0, 0);
    if (i < L.n) gi = __ldg(L.ginfo + i);
    pdl_wait();
    // the cell's one per-cell input of the epilogue (W for G_COPY_W, Rs for G_SET_F, F for G_ADD_F, the
    // explicit state for G_EXPLICIT) is loaded before the slot loop: its latency hides under the gathers,
    // and the epilogue's stores no longer wait on loads the compiler cannot hoist above them (aliasing)
    const int pk = (a.flags & G_COPY_W) ? G_COPY_W : (a.flags & G_SET_F) ? G_SET_F
                 : ((a.flags & G_WRITE_RT) && (a.flags & G_ADD_F)) ? G_ADD_F : (a.flags & G_EXPLICIT) ? G_EXPLICIT : 0;
    double pre[NV];
    if (i < L.n && pk) {
        const double *src = pk == G_COPY_W ? L.W : pk == G_SET_F ? L.Rs : pk == G_ADD_F ? L.F : a.Wexp;
#pragma unroll
        for (int q = 0; q < NV; ++q) pre[q] = src[(size_t)i * NV + q];
    }
    if (i < L.n) {
        // (gather base, all slots | interior slots << 16, sweep slot 0, sweep stride): one 16-byte load
        const int gb = gi.x, nt = gi.y & 0xffff;
        double sig = 0.0, al = 1.0;
        for (int s = 0; s < nt; ++s) {
            const int sf = __ldg(L.gface + gb + kChunk * s);
            const int f = (sf > 0 ? sf : -sf) - 1;
            const double *fr = L.Frec + (size_t)f * kFaceRec;
            double c1[4];
            ld4nc(fr + 4, c1);                 // 3D: SF4, Sr, alpha^M, 0   2D: Sr, alpha^M, 0, 0
            const double srf = c1[FR<D>::SR - 4];
            sig += srf;
            if (a.flags & G_FLUX) {
                double c0[4];
                ld4nc(fr, c0);
                const double sg = sf > 0 ? 1.0 : -1.0;
#pragma unroll
                for (int q = 0; q < 4; ++q) R[q] += sg * c0[q];
                if (D == 3) R[NV - 1] += sg * c1[0];
                al *= c1[FR<D>::AM - 4];
            }
        }
        if (a.flags & G_ALPHA) L.alpha[i] = al;
        if (a.flags & G_SIGMA) L.sigma[i] = sig;
        double *rc = L.rec + (size_t)i * RC::STRIDE;
        if (a.flags & G_PREPARE) {
            const double ai = (a.flags & G_BETA) ? a.beta : ((a.flags & G_ALPHA) ? al : L.alpha[i]);
            // D = alpha (V/Dt_imp + Sigma/2) + (1 - alpha) V/Dt_exp (O6, A2, A3)
            const double Dg = ai * (sig / a.cfl_imp + 0.5 * sig) + (1.0 - ai) * (sig / a.cfl_exp);
            rc[RC::INVD] = 1.0 / Dg;
            rc[RC::HA] = 0.5 * ai;
        }
        if (a.flags & G_ZERO_DW) {
#pragma unroll
            for (int q = 0; q < NV; ++q) rc[RC::DW + q] = 0.0;
        }
        const size_t o = (size_t)i * NV;
        if (a.flags & G_COPY_W) {
#pragma unroll
            for (int q = 0; q < NV; ++q) rc[RC::W + q] = pre[q];
        }
        if (a.flags & G_SET_F) {
            if (pk == G_SET_F) {
#pragma unroll
                for (int q = 0; q < NV; ++q) L.F[o + q] = pre[q] - R[q];
            } else {
#pragma unroll
                for (int q = 0; q < NV; ++q) L.F[o + q] = L.Rs[o + q] - R[q];
            }
        }
        if (a.flags & G_WRITE_RT) {
            if (a.flags & G_ADD_F) {
                if (pk == G_ADD_F) {
#pragma unroll
                    for (int q = 0; q < NV; ++q) L.Rt[o + q] = R[q] + pre[q];
                } else {
#pragma unroll
                    for (int q = 0; q < NV; ++q) L.Rt[o + q] = R[q] + L.F[o + q];
                }
            } else {
#pragma unroll
                for (int q = 0; q < NV; ++q) L.Rt[o + q] = R[q];
            }
        }
        if (a.flags & G_EXPLICIT) {
            const double c = a.cfl_exp / sig;
            if (pk == G_EXPLICIT) {
#pragma unroll
                for (int q = 0; q < NV; ++q) a.Wexp[o + q] = pre[q] - c * R[q];
            } else {
#pragma unroll
                for (int q = 0; q < NV; ++q) a.Wexp[o + q] = a.Wexp[o + q] - c * R[q];
            }
        }
    }
    if (a.flags & G_NORM) {
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

// deterministic reduction of one domain's norm partials -> sumsq[q]
__global__ void __launch_bounds__(256) k_norm_sum(const double *__restrict__ partial, int nblocks, int nv,
                                                  double *sumsq)
{
    pdl_enter();
    __shared__ double sh[256];
    for (int q = 0; q < nv; ++q) {
        double s = 0.0;
        for (int b = threadIdx.x; b < nblocks; b += 256) s += partial[(size_t)b * nv + q];
        sh[threadIdx.x] = s;
        __syncthreads();
        for (int w = 128; w > 0; w >>= 1) {
            if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
            __syncthreads();
        }
        if (threadIdx.x == 0) sumsq[q] = sh[0];
        __syncthreads();
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
// arrays with the given stride/offset (record dW, record W_lin, or W).
// ---------------------------------------------------------------------------
__global__ void k_pack(int count, const int *__restrict__ idx, const double *__restrict__ src, int stride,
                       int offset, int ncomp, double *__restrict__ buf)
{
    pdl_enter();
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= count) return;
    const double *s = src + (size_t)idx[k] * stride + offset;
    for (int q = 0; q < ncomp; ++q) buf[(size_t)k * ncomp + q] = s[q];
}
__global__ void k_unpack(int count, const int *__restrict__ idx, const double *__restrict__ buf, double *dst,
                         int stride, int offset, int ncomp, int zero_at, int nzero)
{
    pdl_enter();
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= count) return;
    double *d = dst + (size_t)idx[k] * stride;
    for (int q = 0; q < ncomp; ++q) d[offset + q] = buf[(size_t)k * ncomp + q];
    for (int q = 0; q < nzero; ++q) d[zero_at + q] = 0.0;
}

// ghost records from the (current) ghost state: W_lin = W, dW = 0
template <int D>
__global__ void k_ghost_wlin(int n, int n_loc, const double *__restrict__ W, double *rec)
{
    pdl_enter();
    using RC = Rec<D>;
    const int g = n + blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n_loc) return;
#pragma unroll
    for (int q = 0; q < D + 2; ++q) {
        rec[(size_t)g * RC::STRIDE + RC::W + q] = W[(size_t)g * (D + 2) + q];
        rec[(size_t)g * RC::STRIDE + RC::DW + q] = 0.0;
    }
}
// ghost states after a smoothing step: W = W_lin + dW (both already exchanged)
template <int D>
__global__ void k_ghost_w(int n, int n_loc, const double *__restrict__ rec, double *W)
{
    pdl_enter();
    using RC = Rec<D>;
    const int g = n + blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n_loc) return;
#pragma unroll
    for (int q = 0; q < D + 2; ++q)
        W[(size_t)g * (D + 2) + q] = rec[(size_t)g * RC::STRIDE + RC::W + q] + rec[(size_t)g * RC::STRIDE + RC::DW + q];
}

// ---------------------------------------------------------------------------
// MC-LU-SGS sweep over one color block (a11 / a12), reading all neighbours'
// current increments (reading A7):
//   dW_i = -( Rt_i + alpha_i/2 sum_j [T(W_j+dW_j; A) - T(W_j; A) - S r dW_j] ) / D_i
// with A = sigma S n (the Euler flux is linear in its normal, S T(W;n) = T(W;A)).
// LPC lanes per cell: each lane gathers its slots' neighbours (one dependent
// index->record round trip), partial sums are combined with warp shuffles.
// Same-color cells never neighbour each other, so the in-place dW update is
// race free and neighbours' dW may be read through the non-coherent path.
// ---------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ void flux_diff(const double *w, const double *dw, const double *A, double gm1,
                                          double Sr, double *acc)
{
    const double r0 = w[0], r1 = w[0] + dw[0];
    const double i0 = 1.0 / r0, i1 = 1.0 / r1;
    double mA0 = 0.0, mA1 = 0.0, m20 = 0.0, m21 = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const double a0 = w[1 + k], a1 = w[1 + k] + dw[1 + k];
        mA0 += a0 * A[k];
        mA1 += a1 * A[k];
        m20 += a0 * a0;
        m21 += a1 * a1;
    }
    const double E0 = w[D + 1], E1 = w[D + 1] + dw[D + 1];
    const double p0 = gm1 * (E0 - 0.5 * m20 * i0), p1 = gm1 * (E1 - 0.5 * m21 * i1);
    const double U0 = mA0 * i0, U1 = mA1 * i1;
    acc[0] += (mA1 - mA0) - Sr * dw[0];
#pragma unroll
    for (int k = 0; k < D; ++k)
        acc[1 + k] += ((w[1 + k] + dw[1 + k]) * U1 + p1 * A[k]) - (w[1 + k] * U0 + p0 * A[k]) - Sr * dw[1 + k];
    acc[D + 1] += (E1 + p1) * U1 - (E0 + p0) * U0 - Sr * dw[D + 1];
}

struct SweepArgs {
    int cbeg, cend;            // color block [cbeg, cend) of owned cells
    double gm1;
    double *rec;               // [n_loc][Rec::STRIDE]
    const int *ecell;          // [n] first slot entry of each cell
    const uint8_t *deg;        // [n] interior slots of each cell
    const int2 *sinfo;         // [n] (first slot entry, interior slots) packed
    const int *sJe;            // [ns] neighbour
    const double *sRe;         // [ns][4] (A outward | S r)
    const double *rhs;         // [n][nv]
    double *Wout;              // [n][nv] or null: W = W_lin + dW (last backward half-sweep)
    int zlo, zhi;              // neighbours j in [zlo, zhi) still hold dW = +0 exactly (first
                               // forward half-sweep, later colors): their term is +0, skipped
};

// neighbour record -> (W_lin, dW)
template <int D>
__device__ __forceinline__ void ld_neighbour(const double *rj, double *w, double *dw)
{
    if constexpr (D == 3) {
        double c0[4], c1[4], c2[4];
        ld4nc(rj, c0);
        ld4nc(rj + 4, c1);
        ld4nc(rj + 8, c2);
        w[0] = c0[0]; w[1] = c0[1]; w[2] = c0[2]; w[3] = c0[3]; w[4] = c1[0];
        dw[0] = c1[3]; dw[1] = c2[0]; dw[2] = c2[1]; dw[3] = c2[2]; dw[4] = c2[3];
    } else {
        ld4nc(rj, w);
        ld4nc(rj + 4, dw);
    }
}

// own-cell epilogue: dW_i = -(rhs_i + alpha_i/2 acc) / D_i into the record,
// and W = W_lin + dW on the last backward half-sweep
template <int D>
__device__ __forceinline__ void sweep_finish(const SweepArgs &a, int i, const double *acc)
{
    constexpr int NV = D + 2;
    using RC = Rec<D>;
    double *ri = a.rec + (size_t)i * RC::STRIDE;
    const size_t o = (size_t)i * NV;
    double r[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) r[q] = __ldcs(a.rhs + o + q);
    if constexpr (D == 3) {
        double c1[4];
        ld4nc(ri + 4, c1);                          // W4, 1/D, alpha/2, dW0
        const double invD = c1[1], ha = c1[2];
        double d[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) d[q] = -(r[q] + ha * acc[q]) * invD;
        ri[RC::DW] = d[0];                          // dW0 alone: a partial-sector write
        const double c2[4] = {d[1], d[2], d[3], d[4]};
        st4(ri + 8, c2);
        if (a.Wout) {
            double c0[4];
            ld4nc(ri, c0);
            a.Wout[o + 0] = c0[0] + d[0];
            a.Wout[o + 1] = c0[1] + d[1];
            a.Wout[o + 2] = c0[2] + d[2];
            a.Wout[o + 3] = c0[3] + d[3];
            a.Wout[o + 4] = c1[0] + d[4];
        }
    } else {
        double c2[4];
        ld4nc(ri + 8, c2);                          // 1/D, alpha/2, -, -
        const double invD = c2[0], ha = c2[1];
        double d[4];
#pragma unroll
        for (int q = 0; q < NV; ++q) d[q] = -(r[q] + ha * acc[q]) * invD;
        st4(ri + 4, d);
        if (a.Wout) {
            double c0[4];
            ld4nc(ri, c0);
#pragma unroll
            for (int q = 0; q < NV; ++q) a.Wout[o + q] = c0[q] + d[q];
        }
    }
}

// sweep variants (template bits, GMG_SWEEPV; default 3, measured DESIGN.md §6):
//  1 = dW0 written inside the whole 32-B chunk (W4 1/D alpha/2 | dW0), no partial sector
//  2 = neighbour index of the next slot loaded one iteration ahead
//  4 = own record tail + rhs prefetched to L1 before the slot loop
// Fused halo (GMG_P2P): the sweep that computes a boundary cell's increment
// also stores it straight into the ghost record of every rank (domain) that
// ghosts the cell, over peer memory (NVLink P2P between GPUs; plain device
// memory between the domains of one process).  Ordering between phases:
// every rank counts its completed color phases (ctl[0]); the last block of a
// sweep launch fences the increments system-wide and publishes the new count
// into each peer's flags[my rank] (st.release.sys); the next launch waits
// until every peer's count has reached its own (ld.acquire.sys) -- so a peer
// never reads a ghost before its phase's increments landed, and never
// overwrites one that is still being read (each side waits for the other).
struct P2PArgs {
    const int *off, *k, *g;      // per owned cell: remote targets (peer slot, ghost local index), CSR
    double *const *peer_rec;     // [peer slot] the peer's record array on this level
    int np;                      // peers on this level (0: count phases only)
    const int *wait_rank;        // [np] their ranks
    int *const *sig;             // [np] &peer.flags[my rank]
    const int *flags;            // [nranks] phase counts published by the peers
    int *ctl;                    // [0] phases completed, [1] blocks done, [2] wait timeout
};

template <int D, bool P2P = false>
__device__ __forceinline__ void p2p_store(const P2PArgs &p, int i, const double *d)
{
    if constexpr (P2P) {
        for (int m = p.off[i]; m < p.off[i + 1]; ++m) {
            double *r = p.peer_rec[p.k[m]] + (size_t)p.g[m] * Rec<D>::STRIDE + Rec<D>::DW;
#pragma unroll
            for (int q = 0; q < D + 2; ++q) r[q] = d[q];
        }
    }
}

template <int D, bool P2P = false, bool CS = true>
__device__ __forceinline__ void sweep_finish_full(const SweepArgs &a, int i, const double *acc,
                                                  const P2PArgs &p = P2PArgs{})
{
    constexpr int NV = D + 2;
    double *ri = a.rec + (size_t)i * Rec<D>::STRIDE;
    const size_t o = (size_t)i * NV;
    double r[NV], c1[4], c2[4];
#pragma unroll
    for (int q = 0; q < NV; ++q) r[q] = CS ? __ldcs(a.rhs + o + q) : __ldg(a.rhs + o + q);
    if constexpr (D == 3) ld4nc(ri + 4, c1);       // W4, 1/D, alpha/2, dW0
    else ld4nc(ri + 8, c2);                         // 1/D, alpha/2, -, -
    if constexpr (D == 3) {
        const double invD = c1[1], ha = c1[2];
        double d[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) d[q] = -(r[q] + ha * acc[q]) * invD;
        const double w1[4] = {c1[0], c1[1], c1[2], d[0]};
        st4(ri + 4, w1);
        const double w2[4] = {d[1], d[2], d[3], d[4]};
        st4(ri + 8, w2);
        p2p_store<D, P2P>(p, i, d);
        if (a.Wout) {
            double c0[4];
            ld4nc(ri, c0);
            a.Wout[o + 0] = c0[0] + d[0];
            a.Wout[o + 1] = c0[1] + d[1];
            a.Wout[o + 2] = c0[2] + d[2];
            a.Wout[o + 3] = c0[3] + d[3];
            a.Wout[o + 4] = c1[0] + d[4];
        }
    } else {
        const double invD = c2[0], ha = c2[1];
        double d[4];
#pragma unroll
        for (int q = 0; q < NV; ++q) d[q] = -(r[q] + ha * acc[q]) * invD;
        st4(ri + 4, d);
        p2p_store<D, P2P>(p, i, d);
        if (a.Wout) {
            double c0[4];
            ld4nc(ri, c0);
#pragma unroll
            for (int q = 0; q < NV; ++q) a.Wout[o + q] = c0[q] + d[q];
        }
    }
}

template <int D, int LPC, int VAR, bool P2P>
__device__ __forceinline__ void sweep_body(const SweepArgs &a, const P2PArgs &p)
{
    constexpr int NV = D + 2;
    using RC = Rec<D>;
    // grid-stride over the color's cells: a launch sized to exactly the
    // resident waves has no partial last wave (the block count of a color is
    // rarely a multiple of SMs x resident blocks)
    const int total = (a.cend - a.cbeg) * LPC;
    const int stride = gridDim.x * blockDim.x;
    const int rounds = (total + stride - 1) / stride;
    for (int r = 0; r < rounds; ++r) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x + r * stride;
    const int i = a.cbeg + g / LPC;
    const int sub = g % LPC;
    const bool valid = i < a.cend;
    double acc[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) acc[q] = 0.0;
    if (valid) {
        // per-cell contiguous slots (CSR): [ecell[i], ecell[i] + deg[i]); the
        // two index loads are independent.  (Measured against ELL and
        // chunked-ELL layouts: CSR wins on the coarse levels, where the degree
        // spread is wide -- DESIGN.md §6.)
        // (first slot, degree) in ONE 8-byte load: separate loads were
        // serialised by the compiler (degree test before the offset load)
        const int2 sd = __ldg(a.sinfo + i);
        if constexpr ((VAR & 4) != 0) {
            if (sub == 0) {   // own record tail + rhs towards L1 while the gathers run
                const double *ri = a.rec + (size_t)i * RC::STRIDE;
                asm volatile("prefetch.global.L1 [%0];" ::"l"(ri + 4));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(a.rhs + (size_t)i * NV));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(a.rhs + (size_t)i * NV + NV - 1));
            }
        }
        const int e0 = sd.x, e1 = sd.x + sd.y;
        if constexpr ((VAR & 8) != 0) {
            // PDL prologue: the slot indices are static during a smoothing step, so the cell's slot range
            // and first neighbour index are loaded before griddepcontrol.wait -- they overlap the previous
            // phase's tail; slot records and neighbour records (previous phases' increments) after it
            int e = e0 + sub;
            int j = e < e1 ? __ldg(a.sJe + e) : 0;
            if (r == 0) pdl_wait();
            for (; e < e1; e += LPC) {
                const int jn = e + LPC < e1 ? __ldg(a.sJe + e + LPC) : 0;
                if (j >= a.zlo && j < a.zhi) { j = jn; continue; }
                double sr[4];
                if constexpr ((VAR & 32) != 0) ld4nc(a.sRe + (size_t)e * kSlotRec, sr);   // L2-resident
                else ld4cs(a.sRe + (size_t)e * kSlotRec, sr);
                double w[NV], dw[NV];
                ld_neighbour<D>(a.rec + (size_t)j * RC::STRIDE, w, dw);
                flux_diff<D>(w, dw, sr, a.gm1, sr[D], acc);
                j = jn;
            }
        } else if constexpr ((VAR & 2) != 0) {
            int e = e0 + sub;
            int j = e < e1 ? __ldg(a.sJe + e) : 0;
            for (; e < e1; e += LPC) {
                const int jn = e + LPC < e1 ? __ldg(a.sJe + e + LPC) : 0;
                if (j >= a.zlo && j < a.zhi) { j = jn; continue; }
                double sr[4];
                ld4cs(a.sRe + (size_t)e * kSlotRec, sr);
                double w[NV], dw[NV];
                ld_neighbour<D>(a.rec + (size_t)j * RC::STRIDE, w, dw);
                flux_diff<D>(w, dw, sr, a.gm1, sr[D], acc);
                j = jn;
            }
        } else {
            for (int e = e0 + sub; e < e1; e += LPC) {
                const int j = __ldg(a.sJe + e);
                if (j >= a.zlo && j < a.zhi) continue;
                double sr[4];
                ld4cs(a.sRe + (size_t)e * kSlotRec, sr);
                double w[NV], dw[NV];
                ld_neighbour<D>(a.rec + (size_t)j * RC::STRIDE, w, dw);
                flux_diff<D>(w, dw, sr, a.gm1, sr[D], acc);
            }
        }
    }
    if (LPC > 1) {
#pragma unroll
        for (int o = LPC / 2; o > 0; o >>= 1) {
#pragma unroll
            for (int q = 0; q < NV; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
        }
    }
    if (valid && sub == 0) {
        if constexpr ((VAR & 1) != 0 || P2P) sweep_finish_full<D, P2P, (VAR & 32) == 0>(a, i, acc, p);
        else sweep_finish<D>(a, i, acc);
    }
    }
    if constexpr ((VAR & 8) != 0) pdl_wait();   // threads without a cell: nothing may run past the predecessor
}

// (VAR bit 16) the same sweep software-pipelined across grid-stride rounds: a
// launch sized to one resident wave runs each thread over several cells, one
// after the other, and every cell is a chain of dependent round trips
// ((first slot, degree) -> neighbour index -> records -> epilogue).  The next
// round's (first slot, degree) is loaded when a round starts and its first
// neighbour index before the round's epilogue, so a later round starts with
// its record loads; round 0's indices are loaded before griddepcontrol.wait.
template <int D, int LPC>
__device__ __forceinline__ void sweep_body_pipe(const SweepArgs &a)
{
    constexpr int NV = D + 2;
    using RC = Rec<D>;
    const int stride = gridDim.x * blockDim.x;            // a multiple of LPC: sub is fixed per thread
    const int g0 = blockIdx.x * blockDim.x + threadIdx.x;
    const int sub = g0 % LPC;
    const int cstep = stride / LPC;
    int i = a.cbeg + g0 / LPC;
    int2 sd = make_int2(0, 0);
    int jf = 0;
    if (i < a.cend) {
        sd = __ldg(a.sinfo + i);
        jf = sub < sd.y ? __ldg(a.sJe + sd.x + sub) : 0;
    }
    pdl_wait();
    const int total = (a.cend - a.cbeg) * LPC;
    const int rounds = (total + stride - 1) / stride;
    for (int r = 0; r < rounds; ++r, i += cstep) {
        const bool valid = i < a.cend;
        const int in = i + cstep;
        int2 sdn = make_int2(0, 0);
        if (in < a.cend) sdn = __ldg(a.sinfo + in);
        double acc[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) acc[q] = 0.0;
        if (valid) {
            const int e1 = sd.x + sd.y;
            int j = jf;
            for (int e = sd.x + sub; e < e1; e += LPC) {
                const int jn = e + LPC < e1 ? __ldg(a.sJe + e + LPC) : 0;
                if (j >= a.zlo && j < a.zhi) { j = jn; continue; }
                double sr[4];
                ld4cs(a.sRe + (size_t)e * kSlotRec, sr);
                double w[NV], dw[NV];
                ld_neighbour<D>(a.rec + (size_t)j * RC::STRIDE, w, dw);
                flux_diff<D>(w, dw, sr, a.gm1, sr[D], acc);
                j = jn;
            }
        }
        jf = (in < a.cend && sub < sdn.y) ? __ldg(a.sJe + sdn.x + sub) : 0;
        sd = sdn;
        if (LPC > 1) {
#pragma unroll
            for (int o = LPC / 2; o > 0; o >>= 1) {
#pragma unroll
                for (int q = 0; q < NV; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
            }
        }
        if (valid && sub == 0) sweep_finish_full<D, false>(a, i, acc);
    }
}

template <int D, int LPC, int MINB, int VAR = 3>
__global__ void __launch_bounds__(256, MINB) k_sweep(SweepArgs a)
{
    pdl_enter();
    sweep_body<D, LPC, VAR, false>(a, P2PArgs{});
}

// the default sweep launch: 128-thread blocks, 8 per SM (GMG_SWEEP_BS=256 -> k_sweep)
template <int D, int LPC, int VAR = 3 | 8, int MINB = 8>
__global__ void __launch_bounds__(128, MINB) k_sweep128(SweepArgs a)
{
    pdl_launch_dependents();                       // the next phase may start its static prologue now
    if constexpr ((VAR & 16) != 0) sweep_body_pipe<D, LPC>(a);
    else sweep_body<D, LPC, VAR, false>(a, P2PArgs{});
}

// 64-thread blocks, 16 per SM (GMG_SWEEP_BS=64): finer-grained block
// scheduling for the partial last round of a grid-stride color launch
template <int D, int LPC>
__global__ void __launch_bounds__(64, 16) k_sweep64(SweepArgs a)
{
    pdl_launch_dependents();
    sweep_body<D, LPC, 3 | 8, false>(a, P2PArgs{});
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
template <int D, int LPC>
__global__ void __launch_bounds__(256, 4) k_sweep_p2p(SweepArgs a, P2PArgs p)
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
    if (!s_bad) sweep_body<D, LPC, 3, true>(a, p);
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

// restriction to a coarse level (a8, A15) into the coarse record's
// W_lin, plus dW = 0 for its sweeps
template <int D>
__global__ void __launch_bounds__(256) k_restrict(DevLevel C, DevLevel Fn, const double *__restrict__ Wf,
                                                  const double *__restrict__ Rf)
{
    pdl_enter();
    constexpr int NV = D + 2;
    using RC = Rec<D>;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C.n) return;
    const int k0 = C.child[c], k1 = C.child[C.n + c];
    const double V0 = Fn.vol[k0];
    double w[NV], r[NV];
    double a = Fn.alpha[k0];
#pragma unroll
    for (int q = 0; q < NV; ++q) { w[q] = V0 * Wf[(size_t)k0 * NV + q]; r[q] = Rf[(size_t)k0 * NV + q]; }
    if (k1 >= 0) {
        const double V1 = Fn.vol[k1];
#pragma unroll
        for (int q = 0; q < NV; ++q) { w[q] = w[q] + V1 * Wf[(size_t)k1 * NV + q]; r[q] = r[q] + Rf[(size_t)k1 * NV + q]; }
        a = fmin(a, Fn.alpha[k1]);
    }
    const double vc = C.vol[c];
    double *rc = C.rec + (size_t)c * RC::STRIDE;
    const size_t o = (size_t)c * NV;
#pragma unroll
    for (int q = 0; q < NV; ++q) { w[q] = w[q] / vc; C.Rs[o + q] = r[q]; }
    // whole 32-byte chunks (no partial-sector writes): W_lin, dW = 0; the 3D
    // record's 1/D and alpha/2 slots are zeroed too -- the next prepare sets them
    if constexpr (D == 3) {
        const double c0[4] = {w[0], w[1], w[2], w[3]}, c1[4] = {w[4], 0.0, 0.0, 0.0}, c2[4] = {0.0, 0.0, 0.0, 0.0};
        st4(rc, c0);
        st4(rc + 4, c1);
        st4(rc + 8, c2);
    } else {
        const double c1[4] = {0.0, 0.0, 0.0, 0.0};
        st4(rc, w);
        st4(rc + 4, c1);
    }
    C.alpha[c] = a;
}

// DF-limited prolongation, both levels fused (a15, A13, A14):
//   W_0 += alpha_0 (dW_1 + alpha_1 dW_2[parent_1])[parent_0]
template <int D>
__global__ void __launch_bounds__(256) k_prolong(DevLevel F0, DevLevel C1, DevLevel C2, int nl)
{
    pdl_enter();
    constexpr int NV = D + 2;
    using RC = Rec<D>;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= F0.n) return;
    const int p = F0.parent[i];
    double corr[NV];
    const double *r1 = C1.rec + (size_t)p * RC::STRIDE + RC::DW;
#pragma unroll
    for (int q = 0; q < NV; ++q) corr[q] = r1[q];
    if (nl >= 3) {
        const int pp = C1.parent[p];
        const double a1 = C1.alpha[p];
        const double *r2 = C2.rec + (size_t)pp * RC::STRIDE + RC::DW;
#pragma unroll
        for (int q = 0; q < NV; ++q) corr[q] += a1 * r2[q];
    }
    const double a0 = F0.alpha[i];
#pragma unroll
    for (int q = 0; q < NV; ++q) F0.W[(size_t)i * NV + q] += a0 * corr[q];
}

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
