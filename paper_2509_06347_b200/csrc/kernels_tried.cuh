// kernels_tried.cuh -- sweep variants that were measured and lost against the
// per-color k_sweep (DESIGN.md §6 table), kept runnable behind their opt-in
// switches, and the test-only concurrency emulation of the fused P2P halo.
// Included by api.cu after kernels.cuh (uses its types and helpers).
#pragma once
#include "kernels.cuh"

namespace gmg {
// ---------------------------------------------------------------------------
// Dependency-driven sweep (single domain, GMG_FLOW): ONE persistent launch runs
// every color phase of a smoothing step.  The cells are grouped into spatial
// chunks; chunk x may run phase p once every neighbouring chunk has finished
// phase p-1 (prog[y] >= p).  A chunk's cells of color(p) read only cells of
// other colors, which by then hold exactly the increments of phases < p (a
// neighbour cannot start phase p+1 before x has published p+1), so the result
// is Algorithm 2's, without a grid-wide barrier (kernel boundary) between
// phases.  Requires all CTAs resident (cooperative launch).  Records written
// inside the launch are read with L2-coherent loads (.cg); progress is
// published with st.release.gpu after a CTA barrier and observed with
// ld.acquire.gpu.  A bounded wait reports a timeout in *err instead of hanging.
// ---------------------------------------------------------------------------
constexpr int kFlowMaxPh = 320;
struct FlowArgs {
    int nph, K, n_own;
    const int *seg, *cnoff, *cnidx;
    int *prog, *err;
    unsigned short ph[kFlowMaxPh];   // color | last << 8 (write W) | first-forward << 9 (skip +0 terms)
};

__device__ __forceinline__ void ld4cg(const double *p, double *v)
{
    asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}
__device__ __forceinline__ int ld_acquire(const int *p)
{
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int *p, int v)
{
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int D>
__global__ void __launch_bounds__(256, 4) k_sweep_flow(SweepArgs a, FlowArgs f)
{
    constexpr int NV = D + 2;
    using RC = Rec<D>;
    __shared__ int s_bad;
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    for (int p = 0; p < f.nph; ++p) {
        const int code = f.ph[p];
        const int c = code & 255;
        double *Wout = (code >> 8 & 1) ? a.Wout : nullptr;
        const int *sg = f.seg + (size_t)c * (f.K + 1);
        const int zlo = (code >> 9 & 1) ? sg[f.K] : 0, zhi = (code >> 9 & 1) ? f.n_own : 0;
        for (int x = blockIdx.x; x < f.K; x += gridDim.x) {
            const int s0 = sg[x], s1 = sg[x + 1];
            if (s1 > s0) {
                if (p > 0) {
                    for (int t = f.cnoff[x] + threadIdx.x; t < f.cnoff[x + 1]; t += blockDim.x) {
                        const int y = f.cnidx[t];
                        for (int spin = 0; ld_acquire(f.prog + y) < p; ++spin) {
                            if (spin > (1 << 22) || *(volatile int *)f.err) {
                                atomicExch(f.err, 1);
                                s_bad = 1;
                                break;
                            }
                            __nanosleep(64);
                        }
                    }
                    __syncthreads();
                    if (s_bad) return;
                }
                // lanes per cell: fill the CTA with the segment's cells
                const int ncell = s1 - s0;
                int L = 2;
                while (L < 16 && ncell * L * 2 <= (int)blockDim.x) L *= 2;
                const int cpi = blockDim.x / L;
                for (int base = s0; base < s1; base += cpi) {
                    const int i = base + threadIdx.x / L, sub = threadIdx.x % L;
                    const bool valid = i < s1;
                    double acc[NV];
#pragma unroll
                    for (int q = 0; q < NV; ++q) acc[q] = 0.0;
                    if (valid) {
                        const int2 sd = __ldg(a.sinfo + i);
                        const int e1 = sd.x + sd.y;
                        for (int e = sd.x + sub; e < e1; e += L) {
                            const int j = __ldg(a.sJe + e);
                            if (j >= zlo && j < zhi) continue;
                            double sr[4];
                            ld4cs(a.sRe + (size_t)e * kSlotRec, sr);
                            const double *rj = a.rec + (size_t)j * RC::STRIDE;
                            double w[NV], dw[NV];
                            if constexpr (D == 3) {
                                double c0[4], c1[4], c2[4];
                                ld4cg(rj, c0);
                                ld4cg(rj + 4, c1);
                                ld4cg(rj + 8, c2);
                                w[0] = c0[0]; w[1] = c0[1]; w[2] = c0[2]; w[3] = c0[3]; w[4] = c1[0];
                                dw[0] = c1[3]; dw[1] = c2[0]; dw[2] = c2[1]; dw[3] = c2[2]; dw[4] = c2[3];
                            } else {
                                ld4cg(rj, w);
                                ld4cg(rj + 4, dw);
                            }
                            flux_diff<D>(w, dw, sr, a.gm1, sr[D], acc);
                        }
                    }
                    for (int o = L / 2; o > 0; o >>= 1) {
#pragma unroll
                        for (int q = 0; q < NV; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
                    }
                    if (valid && sub == 0) {
                        double *ri = a.rec + (size_t)i * RC::STRIDE;
                        const size_t o = (size_t)i * NV;
                        double r[NV], c1[4], c2[4];
#pragma unroll
                        for (int q = 0; q < NV; ++q) r[q] = __ldcs(a.rhs + o + q);
                        ld4cg(ri + 4, c1);
                        ld4cg(ri + 8, c2);
                        if constexpr (D == 3) {
                            const double invD = c1[1], ha = c1[2];
                            double d[NV];
#pragma unroll
                            for (int q = 0; q < NV; ++q) d[q] = -(r[q] + ha * acc[q]) * invD;
                            const double w1[4] = {c1[0], c1[1], c1[2], d[0]};
                            st4(ri + 4, w1);
                            const double w2[4] = {d[1], d[2], d[3], d[4]};
                            st4(ri + 8, w2);
                            if (Wout) {
                                double c0[4];
                                ld4cg(ri, c0);
                                Wout[o + 0] = c0[0] + d[0];
                                Wout[o + 1] = c0[1] + d[1];
                                Wout[o + 2] = c0[2] + d[2];
                                Wout[o + 3] = c0[3] + d[3];
                                Wout[o + 4] = c1[0] + d[4];
                            }
                        } else {
                            const double invD = c2[0], ha = c2[1];
                            double d[4];
#pragma unroll
                            for (int q = 0; q < NV; ++q) d[q] = -(r[q] + ha * acc[q]) * invD;
                            st4(ri + 4, d);
                            if (Wout) {
                                double c0[4];
                                ld4cg(ri, c0);
#pragma unroll
                                for (int q = 0; q < NV; ++q) Wout[o + q] = c0[q] + d[q];
                            }
                        }
                    }
                }
                __syncthreads();   // every write of the segment before the release below
            }
            if (threadIdx.x == 0) st_release(f.prog + x, p + 1);
        }
    }
}

// warp-granular variant (GMG_FLOW=2): every WARP owns chunks and runs their
// phases; no CTA barrier -- lanes wait with a warp vote, __syncwarp orders the
// warp's record writes before lane 0's release
template <int D>
__global__ void __launch_bounds__(256, 4) k_sweep_flow_w(SweepArgs a, FlowArgs f)
{
    constexpr int NV = D + 2;
    using RC = Rec<D>;
    const int lane = threadIdx.x & 31;
    const int worker = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int nworker = gridDim.x * (blockDim.x >> 5);
    for (int p = 0; p < f.nph; ++p) {
        const int code = f.ph[p];
        const int c = code & 255;
        double *Wout = (code >> 8 & 1) ? a.Wout : nullptr;
        const int *sg = f.seg + (size_t)c * (f.K + 1);
        const int zlo = (code >> 9 & 1) ? sg[f.K] : 0, zhi = (code >> 9 & 1) ? f.n_own : 0;
        for (int x = worker; x < f.K; x += nworker) {
            const int s0 = sg[x], s1 = sg[x + 1];
            if (s1 > s0) {
                if (p > 0) {
                    bool bad = false;
                    for (int t = f.cnoff[x] + lane; t < f.cnoff[x + 1]; t += 32) {
                        const int y = f.cnidx[t];
                        for (int spin = 0; ld_acquire(f.prog + y) < p; ++spin) {
                            if (spin > (1 << 22) || *(volatile int *)f.err) { atomicExch(f.err, 1); bad = true; break; }
                            __nanosleep(32);
                        }
                    }
                    if (__any_sync(0xffffffffu, bad)) return;
                }
                const int ncell = s1 - s0;
                int L = 2;
                while (L < 16 && ncell * L * 2 <= 32) L *= 2;
                const int cpi = 32 / L;
                for (int base = s0; base < s1; base += cpi) {
                    const int i = base + lane / L, sub = lane % L;
                    const bool valid = i < s1;
                    double acc[NV];
#pragma unroll
                    for (int q = 0; q < NV; ++q) acc[q] = 0.0;
                    if (valid) {
                        const int2 sd = __ldg(a.sinfo + i);
                        const int e1 = sd.x + sd.y;
                        for (int e = sd.x + sub; e < e1; e += L) {
                            const int j = __ldg(a.sJe + e);
                            if (j >= zlo && j < zhi) continue;
                            double sr[4];
                            ld4cs(a.sRe + (size_t)e * kSlotRec, sr);
                            const double *rj = a.rec + (size_t)j * RC::STRIDE;
                            double w[NV], dw[NV];
                            if constexpr (D == 3) {
                                double c0[4], c1[4], c2[4];
                                ld4cg(rj, c0);
                                ld4cg(rj + 4, c1);
                                ld4cg(rj + 8, c2);
                                w[0] = c0[0]; w[1] = c0[1]; w[2] = c0[2]; w[3] = c0[3]; w[4] = c1[0];
                                dw[0] = c1[3]; dw[1] = c2[0]; dw[2] = c2[1]; dw[3] = c2[2]; dw[4] = c2[3];
                            } else {
                                ld4cg(rj, w);
                                ld4cg(rj + 4, dw);
                            }
                            flux_diff<D>(w, dw, sr, a.gm1, sr[D], acc);
                        }
                    }
                    for (int o = L / 2; o > 0; o >>= 1) {
#pragma unroll
                        for (int q = 0; q < NV; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
                    }
                    if (valid && sub == 0) {
                        double *ri = a.rec + (size_t)i * RC::STRIDE;
                        const size_t o = (size_t)i * NV;
                        double r[NV], c1[4], c2[4];
#pragma unroll
                        for (int q = 0; q < NV; ++q) r[q] = __ldcs(a.rhs + o + q);
                        ld4cg(ri + 4, c1);
                        ld4cg(ri + 8, c2);
                        if constexpr (D == 3) {
                            const double invD = c1[1], ha = c1[2];
                            double d[NV];
#pragma unroll
                            for (int q = 0; q < NV; ++q) d[q] = -(r[q] + ha * acc[q]) * invD;
                            const double w1[4] = {c1[0], c1[1], c1[2], d[0]};
                            st4(ri + 4, w1);
                            const double w2[4] = {d[1], d[2], d[3], d[4]};
                            st4(ri + 8, w2);
                            if (Wout) {
                                double c0[4];
                                ld4cg(ri, c0);
                                Wout[o + 0] = c0[0] + d[0];
                                Wout[o + 1] = c0[1] + d[1];
                                Wout[o + 2] = c0[2] + d[2];
                                Wout[o + 3] = c0[3] + d[3];
                                Wout[o + 4] = c1[0] + d[4];
                            }
                        } else {
                            const double invD = c2[0], ha = c2[1];
                            double d[4];
#pragma unroll
                            for (int q = 0; q < NV; ++q) d[q] = -(r[q] + ha * acc[q]) * invD;
                            st4(ri + 4, d);
                            if (Wout) {
                                double c0[4];
                                ld4cg(ri, c0);
#pragma unroll
                                for (int q = 0; q < NV; ++q) Wout[o + q] = c0[q] + d[q];
                            }
                        }
                    }
                }
                __syncwarp();
            }
            if (lane == 0) st_release(f.prog + x, p + 1);
        }
    }
}

// ---------------------------------------------------------------------------
// Tail sweep: consecutive TINY color phases of a smoothing step (e.g. the last
// colors of a forward pass and the first ones of the next backward pass) run
// in ONE single-CTA launch, one phase after the other with a block barrier in
// between -- the color order of Algorithm 2 is kept, only the launches are
// merged.  Neighbour increments written by an earlier phase of the same launch
// are read with coherent loads.  Single-domain runs only (a partitioned run
// exchanges increments after every color).
// ---------------------------------------------------------------------------
constexpr int kTailMaxPh = 12;
constexpr int kTailT = 1024;
struct TailArgs {
    int nph;
    int cbeg[kTailMaxPh], cend[kTailMaxPh], wout[kTailMaxPh];
    SweepArgs a;                // rec, ecell, deg, sJe, sRe, rhs, Wout, gm1 (cbeg/cend unused)
};

// Cooperative tail (opt-in, GMG_TAILC=1; measured slower): a run of
// consecutive SMALL color phases (each fits one resident wave at >= 2 lanes
// per cell) runs in ONE launch over the whole resident grid, phases separated
// by a grid barrier instead of kernel boundaries.  Records written by an
// earlier phase of the launch are read L2-coherent (.cg).
__device__ __forceinline__ void grid_barrier(int *bar)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        const int g = ld_acquire(bar + 1);
        __threadfence();
        if (atomicAdd(bar, 1) == (int)gridDim.x - 1) {
            bar[0] = 0;
            st_release(bar + 1, g + 1);
        } else {
            while (ld_acquire(bar + 1) == g) __nanosleep(32);
        }
    }
    __syncthreads();
}

template <int D>
__global__ void __launch_bounds__(256, 4) k_sweep_tailc(TailArgs t, int *bar)
{
    constexpr int NV = D + 2;
    using RC = Rec<D>;
    const SweepArgs &a = t.a;
    const int nthr = gridDim.x * blockDim.x, gtid = blockIdx.x * blockDim.x + threadIdx.x;
    for (int ph = 0; ph < t.nph; ++ph) {
        const int b0 = t.cbeg[ph], b1 = t.cend[ph], cells = b1 - b0;
        double *Wout = t.wout[ph] ? a.Wout : nullptr;
        int L = 2;
        while (L < 16 && cells * L * 2 <= nthr) L *= 2;
        const int per = nthr / L;
        const int rounds = (cells + per - 1) / per;
        for (int r = 0; r < rounds; ++r) {
            const int i = b0 + r * per + gtid / L, sub = gtid % L;
            const bool valid = i < b1;
            double acc[NV];
#pragma unroll
            for (int q = 0; q < NV; ++q) acc[q] = 0.0;
            if (valid) {
                const int2 sd = __ldg(a.sinfo + i);
                const int e1 = sd.x + sd.y;
                for (int e = sd.x + sub; e < e1; e += L) {
                    const int j = __ldg(a.sJe + e);
                    double sr[4];
                    ld4cs(a.sRe + (size_t)e * kSlotRec, sr);
                    const double *rj = a.rec + (size_t)j * RC::STRIDE;
                    double w[NV], dw[NV];
                    if constexpr (D == 3) {
                        double c0[4], c1[4], c2[4];
                        ld4cg(rj, c0);
                        ld4cg(rj + 4, c1);
                        ld4cg(rj + 8, c2);
                        w[0] = c0[0]; w[1] = c0[1]; w[2] = c0[2]; w[3] = c0[3]; w[4] = c1[0];
                        dw[0] = c1[3]; dw[1] = c2[0]; dw[2] = c2[1]; dw[3] = c2[2]; dw[4] = c2[3];
                    } else {
                        ld4cg(rj, w);
                        ld4cg(rj + 4, dw);
                    }
                    flux_diff<D>(w, dw, sr, a.gm1, sr[D], acc);
                }
            }
            for (int o = L / 2; o > 0; o >>= 1) {
#pragma unroll
                for (int q = 0; q < NV; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
            }
            if (valid && sub == 0) {
                double *ri = a.rec + (size_t)i * RC::STRIDE;
                const size_t o = (size_t)i * NV;
                double rr[NV], c1[4], c2[4];
#pragma unroll
                for (int q = 0; q < NV; ++q) rr[q] = __ldcs(a.rhs + o + q);
                ld4cg(ri + 4, c1);
                ld4cg(ri + 8, c2);
                if constexpr (D == 3) {
                    const double invD = c1[1], ha = c1[2];
                    double d[NV];
#pragma unroll
                    for (int q = 0; q < NV; ++q) d[q] = -(rr[q] + ha * acc[q]) * invD;
                    const double w1[4] = {c1[0], c1[1], c1[2], d[0]};
                    st4(ri + 4, w1);
                    const double w2[4] = {d[1], d[2], d[3], d[4]};
                    st4(ri + 8, w2);
                    if (Wout) {
                        double c0[4];
                        ld4cg(ri, c0);
                        Wout[o + 0] = c0[0] + d[0];
                        Wout[o + 1] = c0[1] + d[1];
                        Wout[o + 2] = c0[2] + d[2];
                        Wout[o + 3] = c0[3] + d[3];
                        Wout[o + 4] = c1[0] + d[4];
                    }
                } else {
                    const double invD = c2[0], ha = c2[1];
                    double d[4];
#pragma unroll
                    for (int q = 0; q < NV; ++q) d[q] = -(rr[q] + ha * acc[q]) * invD;
                    st4(ri + 4, d);
                    if (Wout) {
                        double c0[4];
                        ld4cg(ri, c0);
#pragma unroll
                        for (int q = 0; q < NV; ++q) Wout[o + q] = c0[q] + d[q];
                    }
                }
            }
        }
        if (ph + 1 < t.nph) grid_barrier(bar);
    }
}

// ---------------------------------------------------------------------------
// Concurrency test of the fused P2P halo protocol on ONE GPU (test only,
// gmg_p2p_emulate_smooth): the guide-sanctioned way to run mutually waiting
// ranks on one device -- ONE cooperative launch, one group of blocks per
// domain ("rank"), all groups resident and running at the same time.  Each
// group runs its domain's smoothing step phase by phase with exactly the
// protocol of k_sweep_p2p: wait until every peer's phase count reached its
// own (acquire), sweep the color block storing boundary increments into the
// peers' ghost records, then publish the new count (release); a group-wide
// barrier stands in for the kernel boundaries of the production launches.
// ---------------------------------------------------------------------------
constexpr int kEmuMaxDom = 16, kEmuMaxCol = 24;
struct EmuDom {
    SweepArgs a;
    P2PArgs p;
    int blk[kEmuMaxCol + 1];
    int n_own, rank;
    int *bar;                      // [2] group barrier (count, generation)
};
struct EmuArgs {
    int ndom, nph, per_group;
    const EmuDom *dom;
    unsigned short ph[kFlowMaxPh];  // color | last << 8, 255 = empty synchronisation phase
};

__device__ __forceinline__ void group_barrier(int *bar, int nblocks)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        const int g = ld_acquire(bar + 1);
        __threadfence();
        if (atomicAdd(bar, 1) == nblocks - 1) {
            bar[0] = 0;
            st_release(bar + 1, g + 1);
        } else {
            while (ld_acquire(bar + 1) == g) __nanosleep(32);
        }
    }
    __syncthreads();
}

template <int D>
__global__ void __launch_bounds__(256, 4) k_p2p_emulate(EmuArgs e)
{
    constexpr int NV = D + 2;
    using RC = Rec<D>;
    const int grp = blockIdx.x / e.per_group, gb = blockIdx.x % e.per_group;
    if (grp >= e.ndom) return;
    const EmuDom &dm = e.dom[grp];
    const SweepArgs &a = dm.a;
    const P2PArgs &p = dm.p;
    const int nthr = e.per_group * blockDim.x, gtid = gb * blockDim.x + threadIdx.x;
    __shared__ int s_bad;
    for (int k = 0; k < e.nph; ++k) {
        // wait: every peer completed as many phases as this rank
        if (threadIdx.x == 0) {
            s_bad = 0;
            const int target = *(volatile int *)p.ctl;
            for (int t = 0; t < p.np && !s_bad; ++t)
                for (int spin = 0; ld_acquire(p.flags + p.wait_rank[t]) < target; ++spin) {
                    if (spin > (1 << 24)) { atomicExch(p.ctl + 2, 1); s_bad = 1; break; }
                    __nanosleep(64);
                }
        }
        __syncthreads();
        if (s_bad) return;
        const int code = e.ph[k];
        const int c = code & 255;
        if (c != 255) {
            double *Wout = (code >> 8 & 1) ? a.Wout : nullptr;
            const int b0 = dm.blk[c], b1 = dm.blk[c + 1];
            const int L = 2, per = nthr / L;
            const int rounds = (b1 - b0 + per - 1) / per;
            for (int r = 0; r < rounds; ++r) {
                const int i = b0 + r * per + gtid / L, sub = gtid % L;
                const bool valid = i < b1;
                double acc[NV];
#pragma unroll
                for (int q = 0; q < NV; ++q) acc[q] = 0.0;
                if (valid) {
                    const int2 sd = __ldg(a.sinfo + i);
                    for (int e2 = sd.x + sub; e2 < sd.x + sd.y; e2 += L) {
                        const int j = __ldg(a.sJe + e2);
                        double sr[4];
                        ld4cs(a.sRe + (size_t)e2 * kSlotRec, sr);
                        const double *rj = a.rec + (size_t)j * RC::STRIDE;
                        double w[NV], dw[NV];
                        if constexpr (D == 3) {
                            double c0[4], c1[4], c2[4];
                            ld4cg(rj, c0);
                            ld4cg(rj + 4, c1);
                            ld4cg(rj + 8, c2);
                            w[0] = c0[0]; w[1] = c0[1]; w[2] = c0[2]; w[3] = c0[3]; w[4] = c1[0];
                            dw[0] = c1[3]; dw[1] = c2[0]; dw[2] = c2[1]; dw[3] = c2[2]; dw[4] = c2[3];
                        } else {
                            ld4cg(rj, w);
                            ld4cg(rj + 4, dw);
                        }
                        flux_diff<D>(w, dw, sr, a.gm1, sr[D], acc);
                    }
                }
#pragma unroll
                for (int q = 0; q < NV; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], 1);
                if (valid && sub == 0) {
                    double *ri = a.rec + (size_t)i * RC::STRIDE;
                    const size_t o = (size_t)i * NV;
                    double rr[NV], c1[4], c2[4];
#pragma unroll
                    for (int q = 0; q < NV; ++q) rr[q] = __ldcs(a.rhs + o + q);
                    ld4cg(ri + 4, c1);
                    ld4cg(ri + 8, c2);
                    double d[NV];
                    if constexpr (D == 3) {
                        const double invD = c1[1], ha = c1[2];
#pragma unroll
                        for (int q = 0; q < NV; ++q) d[q] = -(rr[q] + ha * acc[q]) * invD;
                        const double w1[4] = {c1[0], c1[1], c1[2], d[0]};
                        st4(ri + 4, w1);
                        const double w2[4] = {d[1], d[2], d[3], d[4]};
                        st4(ri + 8, w2);
                        if (Wout) {
                            double c0[4];
                            ld4cg(ri, c0);
                            for (int q = 0; q < 4; ++q) Wout[o + q] = c0[q] + d[q];
                            Wout[o + 4] = c1[0] + d[4];
                        }
                    } else {
                        const double invD = c2[0], ha = c2[1];
#pragma unroll
                        for (int q = 0; q < NV; ++q) d[q] = -(rr[q] + ha * acc[q]) * invD;
                        st4(ri + 4, d);
                        if (Wout) {
                            double c0[4];
                            ld4cg(ri, c0);
                            for (int q = 0; q < NV; ++q) Wout[o + q] = c0[q] + d[q];
                        }
                    }
                    p2p_store<D, true>(p, i, d);
                }
            }
        }
        // the kernel boundary of the production launches: the group's stores, then the release
        __threadfence();
        group_barrier(dm.bar, e.per_group);
        if (gb == 0 && threadIdx.x == 0) {
            const int ph = p.ctl[0] + 1;
            p.ctl[0] = ph;
            __threadfence();
            for (int t = 0; t < p.np; ++t) st_release(p.sig[t], ph);
        }
        group_barrier(dm.bar, e.per_group);   // ctl[0] visible to the group before the next wait
    }
}

__device__ __forceinline__ void ld4(const double *p, double *v)
{
    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p) : "memory");
}

template <int D>
__global__ void __launch_bounds__(kTailT) k_sweep_tail(TailArgs t)
{
    pdl_enter();
    constexpr int NV = D + 2;
    using RC = Rec<D>;
    SweepArgs a = t.a;
    for (int p = 0; p < t.nph; ++p) {
        a.cbeg = t.cbeg[p];
        a.cend = t.cend[p];
        double *wout = t.wout[p] ? t.a.Wout : nullptr;
        a.Wout = wout;
        const int total = (a.cend - a.cbeg) * 2;
        for (int base = 0; base < total; base += kTailT) {
            const int g = base + threadIdx.x;
            const int i = a.cbeg + g / 2, sub = g & 1;
            const bool valid = g < total;
            double acc[NV];
#pragma unroll
            for (int q = 0; q < NV; ++q) acc[q] = 0.0;
            if (valid) {
                const int e0 = __ldg(a.ecell + i), e1 = e0 + __ldg(a.deg + i);
                for (int e = e0 + sub; e < e1; e += 2) {
                    const int j = __ldg(a.sJe + e);
                    double sr[4];
                    ld4cs(a.sRe + (size_t)e * kSlotRec, sr);
                    const double *rj = a.rec + (size_t)j * RC::STRIDE;
                    double w[NV], dw[NV];
                    if constexpr (D == 3) {
                        double c0[4], c1[4], c2[4];
                        ld4(rj, c0);
                        ld4(rj + 4, c1);
                        ld4(rj + 8, c2);
                        w[0] = c0[0]; w[1] = c0[1]; w[2] = c0[2]; w[3] = c0[3]; w[4] = c1[0];
                        dw[0] = c1[3]; dw[1] = c2[0]; dw[2] = c2[1]; dw[3] = c2[2]; dw[4] = c2[3];
                    } else {
                        ld4(rj, w);
                        ld4(rj + 4, dw);
                    }
                    flux_diff<D>(w, dw, sr, a.gm1, sr[D], acc);
                }
            }
#pragma unroll
            for (int q = 0; q < NV; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], 1);
            if (valid && sub == 0) sweep_finish<D>(a, i, acc);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Slot-parallel sweep: a block owns a run of whole cells of the color whose
// CSR slots fit in SP_T lanes; lane t gathers slot e_begin + t (one dependent
// index -> record round trip per lane, no per-cell serial slot loop), writes
// its flux-difference contribution to smem, then one thread per cell sums its
// contiguous slots and finishes the cell.  Groups: gcell[g] .. gcell[g+1].
// ---------------------------------------------------------------------------
constexpr int kSpT = 256;

template <int D>
__global__ void __launch_bounds__(kSpT) k_sweep_sp(SweepArgs a, const int *__restrict__ gcell)
{
    pdl_enter();
    constexpr int NV = D + 2;
    using RC = Rec<D>;
    __shared__ double part[kSpT][NV];
    const int c0 = __ldg(gcell + blockIdx.x), c1 = __ldg(gcell + blockIdx.x + 1);
    const int eb = __ldg(a.ecell + c0);
    const int ee = __ldg(a.ecell + c1 - 1) + __ldg(a.deg + c1 - 1);
    const int t = threadIdx.x;
    const int e = eb + t;
    if (e < ee) {
        double acc[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) acc[q] = 0.0;
        const int j = __ldg(a.sJe + e);
        double sr[4];
        ld4cs(a.sRe + (size_t)e * kSlotRec, sr);
        double w[NV], dw[NV];
        ld_neighbour<D>(a.rec + (size_t)j * RC::STRIDE, w, dw);
        flux_diff<D>(w, dw, sr, a.gm1, sr[D], acc);
#pragma unroll
        for (int q = 0; q < NV; ++q) part[t][q] = acc[q];
    }
    __syncthreads();
    const int i = c0 + t;
    if (i >= c1) return;
    double acc[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) acc[q] = 0.0;
    const int s0 = __ldg(a.ecell + i) - eb, s1 = s0 + __ldg(a.deg + i);
    for (int s = s0; s < s1; ++s) {
#pragma unroll
        for (int q = 0; q < NV; ++q) acc[q] += part[s][q];
    }
    sweep_finish<D>(a, i, acc);
}

// ---------------------------------------------------------------------------
// Warp-staged sweep: a warp owns 32 consecutive cells of the color; it
// cp.async's (LDGSTS, no registers held) every neighbour record (6 x 16 B)
// and slot record (2 x 16 B) of its cells' slots into its own smem slice,
// waits (no block barrier), then computes thread-per-cell from smem.  Memory
// parallelism = bytes staged per warp, independent of the register budget.
// smem slice per warp: max_slots x (kRecS + 4) doubles; records padded to
// 112 B so that 16-byte smem accesses of neighbouring slots spread over banks.
// ---------------------------------------------------------------------------
constexpr int kRecS = 14;   // staged record stride (doubles)

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}

template <int D, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_sweep_ws(SweepArgs a, int max_slots)
{
    pdl_enter();
    constexpr int NV = D + 2;
    using RC = Rec<D>;
    extern __shared__ __align__(16) double sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i0 = a.cbeg + (blockIdx.x * WARPS + warp) * 32;
    if (i0 >= a.cend) return;                         // whole warp: no block-level sync below
    const int i = i0 + lane;
    const bool valid = i < a.cend;
    const int last = min(i0 + 31, a.cend - 1);
    const int g0 = __ldg(a.ecell + i0);
    const int ns = __ldg(a.ecell + last) + __ldg(a.deg + last) - g0;
    double *recS = sm + (size_t)warp * max_slots * (kRecS + kSlotRec);
    double *slotS = recS + (size_t)max_slots * kRecS;
    for (int t = lane; t < ns * 2; t += 32) cp_async16(slotS + 2 * t, a.sRe + (size_t)g0 * kSlotRec + 2 * t);
    for (int t = lane; t < ns * 6; t += 32) {
        const int s = t / 6, p = t - 6 * s;
        const int j = __ldg(a.sJe + g0 + s);
        cp_async16(recS + (size_t)s * kRecS + 2 * p, a.rec + (size_t)j * RC::STRIDE + 2 * p);
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    if (!valid) return;
    double acc[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) acc[q] = 0.0;
    const int e0 = __ldg(a.ecell + i) - g0, e1 = e0 + __ldg(a.deg + i);
    for (int s = e0; s < e1; ++s) {
        const double *r = recS + (size_t)s * kRecS;
        const double *sr = slotS + (size_t)s * kSlotRec;
        double w[NV], dw[NV], A[D];
#pragma unroll
        for (int q = 0; q < NV; ++q) { w[q] = r[RC::W + q]; dw[q] = r[RC::DW + q]; }
#pragma unroll
        for (int k = 0; k < D; ++k) A[k] = sr[k];
        flux_diff<D>(w, dw, A, a.gm1, sr[D], acc);
    }
    sweep_finish<D>(a, i, acc);
}

// ---------------------------------------------------------------------------
// Pipelined persistent warp sweep: each warp walks 8-cell batches of the color
// (b = warp id, + total warps, ...) with a 2-stage smem ring: while it computes
// batch b from smem, the cp.async's of batch b+1 (neighbour records, slot
// records, the cells' rhs and own 1/D-alpha chunk) are in flight, and the
// slot indices of batch b+2 are being loaded into registers.  Compute is
// thread-per-slot, then one lane per cell sums its contiguous slot partials.
// ---------------------------------------------------------------------------
constexpr int kPB = 8;            // cells per batch
constexpr int kPW = 4;            // warps per block

struct PipeLayout {               // per-warp smem (doubles)
    int maxS;                     // max slots of a batch on this level
    __device__ __host__ int stage() const { return maxS * (kRecS + kSlotRec) + kPB * 5 + kPB * 4; }
    __device__ __host__ int warp() const { return 2 * stage() + ((maxS * 5 + 1) & ~1) + ((maxS + 1) / 2 + 1) / 2 * 2; }
};

template <int D>
__device__ __forceinline__ void pipe_issue(const SweepArgs &a, int c0, int c1, int s0, int ns, const int *jr,
                                           double *st, const PipeLayout &pl, int lane, int *jS)
{
    double *recS = st, *slotS = st + (size_t)pl.maxS * kRecS, *rhsS = slotS + (size_t)pl.maxS * kSlotRec;
    double *ownS = rhsS + kPB * 5;
    constexpr int NV = D + 2;
    using RC = Rec<D>;
    for (int t = lane; t < ns * 2; t += 32) cp_async16(slotS + 2 * t, a.sRe + (size_t)s0 * kSlotRec + 2 * t);
    // neighbour records: indices via smem, then consecutive lanes copy consecutive
    // 16-B pieces of the same record (5-6 records per warp instruction)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int s = lane + 32 * k;
        if (s < ns) jS[s] = jr[k];
    }
    __syncwarp();
    for (int t = lane; t < ns * 6; t += 32) {
        const int s = t / 6, p = t - 6 * s;
        cp_async16(recS + (size_t)s * kRecS + 2 * p, a.rec + (size_t)jS[s] * RC::STRIDE + 2 * p);
    }
    __syncwarp();
    // rhs (nv doubles per cell, 8-byte aligned only -> 8-byte copies) and the own 1/D, alpha/2 chunk
    const int nc = c1 - c0;
    for (int t = lane; t < nc * NV; t += 32) {
        const unsigned s = (unsigned)__cvta_generic_to_shared(rhsS + t);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(a.rhs + (size_t)c0 * NV + t) : "memory");
    }
    for (int t = lane; t < nc * 2; t += 32)
        cp_async16(ownS + 2 * t, a.rec + (size_t)(c0 + t / 2) * RC::STRIDE + RC::INVD - RC::INVD % 4 + 2 * (t & 1));
}

template <int D>
__global__ void __launch_bounds__(kPW * 32) k_sweep_pipe(SweepArgs a, PipeLayout pl)
{
    pdl_enter();
    constexpr int NV = D + 2;
    using RC = Rec<D>;
    extern __shared__ __align__(16) double sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *wbase = sm + (size_t)warp * pl.warp();
    double *part = wbase + 2 * (size_t)pl.stage();
    int *jS = reinterpret_cast<int *>(part + ((pl.maxS * 5 + 1) & ~1));
    const int ncell = a.cend - a.cbeg;
    const int nb = (ncell + kPB - 1) / kPB;
    const int W = gridDim.x * kPW;
    int b = blockIdx.x * kPW + warp;
    if (b >= nb) return;
    auto range = [&](int bb, int &c0, int &c1, int &s0, int &ns) {
        c0 = a.cbeg + bb * kPB;
        c1 = min(c0 + kPB, a.cend);
        s0 = __ldg(a.ecell + c0);
        ns = __ldg(a.ecell + c1 - 1) + __ldg(a.deg + c1 - 1) - s0;
    };
    auto load_idx = [&](int s0, int ns, int *jr) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int s = lane + 32 * k;
            jr[k] = s < ns ? __ldg(a.sJe + s0 + s) : 0;
        }
    };
    int c0, c1, s0, ns, jr[4];
    range(b, c0, c1, s0, ns);
    load_idx(s0, ns, jr);
    pipe_issue<D>(a, c0, c1, s0, ns, jr, wbase, pl, lane, jS);
    asm volatile("cp.async.commit_group;" ::: "memory");
    int stage = 0;
    while (true) {
        const int bn = b + W;
        int d0 = 0, d1 = 0, t0 = 0, tn = 0, jn[4] = {0, 0, 0, 0};
        if (bn < nb) { range(bn, d0, d1, t0, tn); load_idx(t0, tn, jn); }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        double *st = wbase + (size_t)stage * pl.stage();
        if (bn < nb) {
            pipe_issue<D>(a, d0, d1, t0, tn, jn, wbase + (size_t)(stage ^ 1) * pl.stage(), pl, lane, jS);
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        // compute batch b from stage: thread per slot
        const double *recS = st, *slotS = st + (size_t)pl.maxS * kRecS, *rhsS = slotS + (size_t)pl.maxS * kSlotRec;
        const double *ownS = rhsS + kPB * 5;
        for (int s = lane; s < ns; s += 32) {
            double acc[NV];
#pragma unroll
            for (int q = 0; q < NV; ++q) acc[q] = 0.0;
            const double *r = recS + (size_t)s * kRecS;
            const double *sr = slotS + (size_t)s * kSlotRec;
            double w[NV], dw[NV], A[D];
#pragma unroll
            for (int q = 0; q < NV; ++q) { w[q] = r[RC::W + q]; dw[q] = r[RC::DW + q]; }
#pragma unroll
            for (int k = 0; k < D; ++k) A[k] = sr[k];
            flux_diff<D>(w, dw, A, a.gm1, sr[D], acc);
#pragma unroll
            for (int q = 0; q < NV; ++q) part[s * 5 + q] = acc[q];
        }
        __syncwarp();
        if (lane < c1 - c0) {
            const int i = c0 + lane;
            const int e0 = __ldg(a.ecell + i) - s0, e1 = e0 + __ldg(a.deg + i);
            double acc[NV];
#pragma unroll
            for (int q = 0; q < NV; ++q) acc[q] = 0.0;
            for (int s = e0; s < e1; ++s) {
#pragma unroll
                for (int q = 0; q < NV; ++q) acc[q] += part[s * 5 + q];
            }
            const double *own = ownS + lane * 4;     // the 32-B chunk holding 1/D and alpha/2
            const double invD = own[RC::INVD % 4], ha = own[RC::HA % 4];
            double d[NV];
#pragma unroll
            for (int q = 0; q < NV; ++q) d[q] = -(rhsS[lane * NV + q] + ha * acc[q]) * invD;
            double *ri = a.rec + (size_t)i * RC::STRIDE;
#pragma unroll
            for (int q = 0; q < NV; ++q) ri[RC::DW + q] = d[q];
            if (a.Wout) {
#pragma unroll
                for (int q = 0; q < NV; ++q) a.Wout[(size_t)i * NV + q] = ri[RC::W + q] + d[q];
            }
        }
        __syncwarp();
        if (bn >= nb) break;
        b = bn; c0 = d0; c1 = d1; s0 = t0; ns = tn;
        stage ^= 1;
    }
}

}  // namespace gmg
