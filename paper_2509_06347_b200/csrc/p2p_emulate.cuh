// p2p_emulate.cuh -- concurrency test of the fused P2P halo protocol on ONE
// GPU (test only, gmg_p2p_emulate_smooth).  Included by api.cu after
// kernels.cuh (uses its types and the sweep body).
//
// The guide-sanctioned way to run mutually waiting ranks on one device: ONE
// cooperative launch, one group of blocks per domain ("rank"), all groups
// resident and running at the same time.  Each group runs its domain's
// smoothing step phase by phase with exactly the protocol of k_sweep_p2p:
// wait until every peer's phase count reached its own (acquire), sweep the
// color block storing boundary states into the peers' ghost records, then
// publish the new count (release); a group-wide barrier stands in for the
// kernel boundaries of the production launches.  Records written inside the
// launch are read L2-coherent (.cg).
#pragma once
#include "kernels.cuh"

namespace gmg {

constexpr int kEmuMaxDom = 16, kEmuMaxCol = 24, kEmuMaxPh = 320;
struct EmuDom {
    SweepArgs a;                   // cbeg / cend / lo set per phase
    P2PArgs p;
    int blk[kEmuMaxCol + 1];
    int rank;
    int *bar;                      // [2] group barrier (count, generation)
};
struct EmuArgs {
    int ndom, nph, per_group;
    const EmuDom *dom;
    unsigned short ph[kEmuMaxPh];  // color | last << 8 | first-forward << 9, 255 = empty synchronisation phase
};

__device__ __forceinline__ int ld_acquire_gpu(const int *p)
{
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int *p, int v)
{
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void group_barrier(int *bar, int nblocks)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        const int g = ld_acquire_gpu(bar + 1);
        __threadfence();
        if (atomicAdd(bar, 1) == nblocks - 1) {
            bar[0] = 0;
            st_release_gpu(bar + 1, g + 1);
        } else {
            while (ld_acquire_gpu(bar + 1) == g) __nanosleep(32);
        }
    }
    __syncthreads();
}

template <int D>
__global__ void __launch_bounds__(256, 3) k_p2p_emulate(EmuArgs e)
{
    const int grp = blockIdx.x / e.per_group, gb = blockIdx.x % e.per_group;
    if (grp >= e.ndom) return;
    const EmuDom &dm = e.dom[grp];
    const P2PArgs &p = dm.p;
    const int nthr = e.per_group * blockDim.x, gtid = gb * blockDim.x + threadIdx.x;
    __shared__ int s_bad;
    for (int k = 0; k < e.nph; ++k) {
        // wait: every peer completed as many phases as this rank
        if (threadIdx.x == 0) {
            s_bad = 0;
            const int target = *(volatile int *)p.ctl;
            for (int t = 0; t < p.np && !s_bad; ++t)
                for (int spin = 0; ld_acquire_gpu(p.flags + p.wait_rank[t]) < target; ++spin) {
                    if (spin > (1 << 24)) { atomicExch(p.ctl + 2, 1); s_bad = 1; break; }
                    __nanosleep(64);
                }
        }
        __syncthreads();
        if (s_bad) return;
        const int code = e.ph[k];
        const int c = code & 255;
        if (c != 255) {
            SweepArgs a = dm.a;
            a.cbeg = dm.blk[c];
            a.cend = dm.blk[c + 1];
            a.lo = dm.blk[c];
            if (!(code >> 8 & 1)) a.Wout = nullptr;
            if (code >> 9 & 1) sweep_cells<D, 2, true, true, true>(a, p, gtid, nthr, false);
            else sweep_cells<D, 2, false, true, true>(a, p, gtid, nthr, false);
        }
        // the kernel boundary of the production launches: the group's stores, then the release
        __threadfence();
        group_barrier(dm.bar, e.per_group);
        if (gb == 0 && threadIdx.x == 0) {
            const int ph = p.ctl[0] + 1;
            p.ctl[0] = ph;
            __threadfence();
            for (int t = 0; t < p.np; ++t) st_release_gpu(p.sig[t], ph);
        }
        group_barrier(dm.bar, e.per_group);   // ctl[0] visible to the group before the next wait
    }
}

}  // namespace gmg
