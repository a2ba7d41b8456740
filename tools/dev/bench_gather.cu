// DEV microbenchmark: neighbour-record gather through registers (LDG.256, as the sweep does) vs TMA
// tile::gather4 into shared memory.  Synthetic index stream with sweep-like locality: slot s of "cell"
// i reads record j = perm-local neighbour (i*ratio + jitter) of a second array.  Prints GB/s of
// gathered record bytes (64 B per slot) + slot records (32 B per slot, streamed).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ void ld4nc(const double *p, double *v)
{
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}
__device__ __forceinline__ void ld4cs(const double *p, double *v)
{
    asm volatile("ld.global.cs.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}

// A: one thread per slot, grid-stride, one wave
__global__ void __launch_bounds__(128, 8) k_ldg(int ns, const int *__restrict__ idx, const double *__restrict__ rec,
                                                const double *__restrict__ srec, double *out)
{
    double acc = 0.0;
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < ns; s += gridDim.x * blockDim.x) {
        const int j = __ldg(idx + s);
        double a[4], b[4], c[4];
        ld4cs(srec + (size_t)s * 4, c);
        ld4nc(rec + (size_t)j * 8, a);
        ld4nc(rec + (size_t)j * 8 + 4, b);
        acc += a[0] * c[0] + a[1] * c[1] + a[2] * c[2] + a[3] * c[3] + b[0];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *m, int cnt)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *m, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *m, uint32_t parity)
{
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(smem_u32(m)),
        "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_gather4(void *dst, const CUtensorMap *map, uint64_t *mbar, int r0, int r1, int r2, int r3)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(mbar)), "r"(0), "r"(r0),
        "r"(r1), "r"(r2), "r"(r3) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *mbar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(mbar)) : "memory");
}

// B: persistent CTAs; tile = T slots; 2-stage ring: warp 0 issues the loads of tile k+1 while all
// threads consume tile k from smem
template <int T>
__global__ void __launch_bounds__(256, 1) k_tma(int ns, const int *__restrict__ idx, const __grid_constant__ CUtensorMap map,
                                                const double *__restrict__ srec, double *out)
{
    extern __shared__ __align__(128) unsigned char sm[];
    double *rows = (double *)sm;                       // [2][T][8]
    double *sr = rows + 2 * T * 8;                     // [2][T][4]
    uint64_t *bar = (uint64_t *)(sr + 2 * T * 4);      // [2]
    const int ntile = (ns + T - 1) / T;
    if (threadIdx.x == 0) { mbar_init(bar, 1); mbar_init(bar + 1, 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    auto issue = [&](int tile, int st) {
        // warp 0: lane l issues gather4s for rows 4l.. of the tile
        const int s0 = tile * T, cnt = min(T, ns - s0);
        if (threadIdx.x == 0) mbar_expect_tx(bar + st, (uint32_t)(T * 64 + T * 32));
        __syncwarp();
        for (int g = threadIdx.x; g < T / 4; g += 32) {
            int r[4];
            for (int k = 0; k < 4; ++k) r[k] = (4 * g + k < cnt) ? __ldg(idx + s0 + 4 * g + k) : 0;
            tma_gather4(rows + ((size_t)st * T + 4 * g) * 8, &map, bar + st, r[0], r[1], r[2], r[3]);
        }
        if (threadIdx.x == 0) bulk_g2s(sr + (size_t)st * T * 4, srec + (size_t)s0 * 4, T * 32, bar + st);
    };
    int k = 0;
    double acc = 0.0;
    int tile = blockIdx.x;
    if (tile < ntile && threadIdx.x < 32) issue(tile, 0);
    for (; tile < ntile; tile += gridDim.x, ++k) {
        const int st = k & 1;
        const int nxt = tile + gridDim.x;
        if (nxt < ntile && threadIdx.x < 32) issue(nxt, st ^ 1);
        mbar_wait(bar + st, (k >> 1) & 1);
        for (int t = threadIdx.x; t < T; t += blockDim.x) {
            const double *a = rows + ((size_t)st * T + t) * 8;
            const double *c = sr + ((size_t)st * T + t) * 4;
            acc += a[0] * c[0] + a[1] * c[1] + a[2] * c[2] + a[3] * c[3] + a[4];
        }
        __syncthreads();   // stage st free before it is refilled (issue of tile k+2 at iteration k+1)
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}


// C: the sweep's structure: lanes per cell, (first slot, degree) -> index -> records, own record + write
template <int LPC>
__global__ void __launch_bounds__(128, 8) k_cell(int ncell, const int2 *__restrict__ sinfo, const int *__restrict__ idx,
                                                 const double *__restrict__ rec, const double *__restrict__ srec,
                                                 const double *__restrict__ xr, double *wout)
{
    const int nthr = gridDim.x * blockDim.x, gt = blockIdx.x * blockDim.x + threadIdx.x;
    const int rounds = (ncell * LPC + nthr - 1) / nthr;
    for (int r = 0; r < rounds; ++r) {
        const int g = gt + r * nthr, i = g / LPC, sub = g % LPC;
        double acc = 0.0;
        if (i < ncell) {
            const int2 sd = __ldg(sinfo + i);
            const int e1 = sd.x + sd.y;
            int e = sd.x + sub;
            int j = e < e1 ? __ldg(idx + e) : 0;
            for (; e < e1; e += LPC) {
                const int jn = e + LPC < e1 ? __ldg(idx + e + LPC) : 0;
                double a[4], b[4], c[4];
                ld4cs(srec + (size_t)e * 4, c);
                ld4nc(rec + (size_t)j * 8, a);
                ld4nc(rec + (size_t)j * 8 + 4, b);
                acc += a[0] * c[0] + a[1] * c[1] + a[2] * c[2] + a[3] * c[3] + b[0];
                j = jn;
            }
        }
        for (int o = LPC / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (i < ncell && sub == 0) {
            const double *x = xr + (size_t)i * 6;
            double v = acc + x[0] + x[5];
            double o4[4] = {v, v, v, v};
            asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(wout + (size_t)i * 8), "d"(o4[0]), "d"(o4[1]), "d"(o4[2]), "d"(o4[3]) : "memory");
            asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(wout + (size_t)i * 8 + 4), "d"(o4[0]), "d"(o4[1]), "d"(o4[2]), "d"(o4[3]) : "memory");
        }
    }
}

// D: thread per slot; warps own chunks of 32 slot positions holding whole cells (padded, idx -1);
// segmented warp reduction; the cell's head lane finishes it.  hd[s] = 1 at a cell's first slot.
__global__ void __launch_bounds__(128, 12) k_slot(int nchunk, const int *__restrict__ idx, const unsigned char *__restrict__ hd,
                                                  const int *__restrict__ cell0, const double *__restrict__ rec,
                                                  const double *__restrict__ srec, const double *__restrict__ xr, double *wout)
{
    const int lane = threadIdx.x & 31;
    const int nw = gridDim.x * (blockDim.x >> 5), w0 = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    for (int ch = w0; ch < nchunk; ch += nw) {
        const int e = ch * 32 + lane;
        const int j = __ldg(idx + e);
        const unsigned head = __ballot_sync(0xffffffffu, __ldg(hd + e) != 0);
        const int c0 = __ldg(cell0 + ch);
        // my cell: count of heads at or below my lane
        const int mycell = c0 + __popc(head & (0xffffffffu >> (31 - lane))) - 1;
        const bool ishead = (head >> lane) & 1u;
        double x0 = 0.0, x5 = 0.0;
        if (ishead) { x0 = __ldg(xr + (size_t)mycell * 6); x5 = __ldg(xr + (size_t)mycell * 6 + 5); }
        double acc = 0.0;
        if (j >= 0) {
            double a[4], b[4], c[4];
            ld4cs(srec + (size_t)e * 4, c);
            ld4nc(rec + (size_t)j * 8, a);
            ld4nc(rec + (size_t)j * 8 + 4, b);
            acc = a[0] * c[0] + a[1] * c[1] + a[2] * c[2] + a[3] * c[3] + b[0];
        }
        // segmented inclusive suffix sum (towards the head): add the value from lane+o if it is in my segment
        // segment end of lane l = next head above l (exclusive)
        const unsigned above = head & ~(0xffffffffu >> (31 - lane));   // heads strictly above me
        const int seg_end = above ? __ffs(above) - 1 : 32;              // first lane of the next cell
        for (int o = 1; o < 32; o <<= 1) {
            const double v = __shfl_down_sync(0xffffffffu, acc, o);
            if (lane + o < seg_end) acc += v;
        }
        if (ishead && j >= 0) {
            double v = acc + x0 + x5;
            asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(wout + (size_t)mycell * 8), "d"(v), "d"(v), "d"(v), "d"(v) : "memory");
            asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(wout + (size_t)mycell * 8 + 4), "d"(v), "d"(v), "d"(v), "d"(v) : "memory");
        }
    }
}

int main(int argc, char **argv)
{
    const int ncell = 306000, deg = 4;   // a big level-1 color phase: ~1.2-1.4 M slots
    const int nrec = 875000;
    const int ns = ncell * 9 / 2;
    std::vector<int> idx(ns);
    std::mt19937 rng(1);
    // neighbour j of cell i: near i * nrec / ncell (Morton-like locality), jitter +-256 records
    for (int s = 0; s < ns; ++s) {
        const int i = s * 2 / 9;
        long c = (long)i * nrec / ncell + (long)(rng() % 513) - 256;
        idx[s] = (int)std::min<long>(std::max<long>(c, 0), nrec - 1);
    }
    int *d_idx; double *d_rec, *d_sr, *d_out, *d_flush;
    CK(cudaMalloc(&d_idx, ns * 4));
    CK(cudaMalloc(&d_rec, (size_t)nrec * 64));
    CK(cudaMalloc(&d_sr, (size_t)ns * 32 + 4096));
    CK(cudaMalloc(&d_out, (size_t)ns * 8 + 4096));
    const size_t flush = 512u << 20;
    CK(cudaMalloc(&d_flush, flush));
    CK(cudaMemcpy(d_idx, idx.data(), ns * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(d_rec, 0, (size_t)nrec * 64));
    CK(cudaMemset(d_sr, 0, (size_t)ns * 32));
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q));
    CUtensorMap map;
    cuuint64_t dims[2] = {8, (cuuint64_t)nrec};
    cuuint64_t strides[1] = {64};
    cuuint32_t box[2] = {8, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d_rec, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    // cell structure: degrees 4 / 5 alternating (4.5 average), CSR
    std::vector<int2> sinfo(ncell);
    {
        int e = 0;
        for (int i = 0; i < ncell; ++i) { const int d = 4 + (i & 1); sinfo[i] = make_int2(e, std::min(d, ns - e)); e += d; }
    }
    // slot chunks of 32 with whole cells
    std::vector<int> cidx, cell0;
    std::vector<unsigned char> hd;
    {
        int i = 0;
        while (i < ncell) {
            cell0.push_back(i);
            int used = 0;
            while (i < ncell && used + sinfo[i].y <= 32) {
                for (int k = 0; k < sinfo[i].y; ++k) { cidx.push_back(idx[sinfo[i].x + k]); hd.push_back(k == 0); }
                used += sinfo[i].y; ++i;
            }
            for (; used < 32; ++used) { cidx.push_back(-1); hd.push_back(0); }
        }
    }
    const int nchunk = (int)cell0.size();
    int2 *d_sinfo; int *d_cidx, *d_cell0; unsigned char *d_hd; double *d_xr, *d_w, *d_sr2;
    CK(cudaMalloc(&d_sinfo, ncell * 8));
    CK(cudaMalloc(&d_cidx, cidx.size() * 4));
    CK(cudaMalloc(&d_cell0, cell0.size() * 4));
    CK(cudaMalloc(&d_hd, hd.size()));
    CK(cudaMalloc(&d_xr, (size_t)ncell * 48));
    CK(cudaMalloc(&d_w, (size_t)ncell * 64));
    CK(cudaMalloc(&d_sr2, cidx.size() * 32));
    CK(cudaMemcpy(d_sinfo, sinfo.data(), ncell * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_cidx, cidx.data(), cidx.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_cell0, cell0.data(), cell0.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_hd, hd.data(), hd.size(), cudaMemcpyHostToDevice));
    CK(cudaMemset(d_xr, 0, (size_t)ncell * 48));
    CK(cudaMemset(d_sr2, 0, cidx.size() * 32));
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double bytes = (double)ns * 96;
    auto run = [&](const char *name, auto fn) {
        float best = 1e9;
        for (int rep = 0; rep < 6; ++rep) {
            CK(cudaMemset(d_flush, rep, flush));
            cudaEventRecord(e0);
            fn();
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep) best = std::min(best, ms);
        }
        CK(cudaGetLastError());
        printf("%-28s %8.2f us  %7.0f GB/s\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9);
    };
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_ldg, 128, 0);
    run("ldg one wave", [&] { k_ldg<<<nsm * per, 128>>>(ns, d_idx, d_rec, d_sr, d_out); });
    run("ldg many waves", [&] { k_ldg<<<(ns + 127) / 128, 128>>>(ns, d_idx, d_rec, d_sr, d_out); });
    printf("(cell-structured: + own 48 B read + 64 B write per cell; %d chunks, %.1f%% padding)\n", nchunk,
           100.0 * (nchunk * 32.0 - ns) / (nchunk * 32.0));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_cell<2>, 128, 0);
    run("cell LPC2 one wave", [&] { k_cell<2><<<nsm * per, 128>>>(ncell, d_sinfo, d_idx, d_rec, d_sr, d_xr, d_w); });
    run("cell LPC2 many waves", [&] { k_cell<2><<<(ncell * 2 + 127) / 128, 128>>>(ncell, d_sinfo, d_idx, d_rec, d_sr, d_xr, d_w); });
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_cell<1>, 128, 0);
    run("cell LPC1 one wave", [&] { k_cell<1><<<nsm * per, 128>>>(ncell, d_sinfo, d_idx, d_rec, d_sr, d_xr, d_w); });
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_cell<4>, 128, 0);
    run("cell LPC4 one wave", [&] { k_cell<4><<<nsm * per, 128>>>(ncell, d_sinfo, d_idx, d_rec, d_sr, d_xr, d_w); });
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_slot, 128, 0);
    run("slot-parallel one wave", [&] { k_slot<<<nsm * per, 128>>>(nchunk, d_cidx, d_hd, d_cell0, d_rec, d_sr2, d_xr, d_w); });
    run("slot-parallel many waves", [&] { k_slot<<<(nchunk + 3) / 4, 128>>>(nchunk, d_cidx, d_hd, d_cell0, d_rec, d_sr2, d_xr, d_w); });
    {
        constexpr int T = 512;
        const size_t smem = 2 * T * 64 + 2 * T * 32 + 64;
        CK(cudaFuncSetAttribute(k_tma<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        run("tma gather4 T=512 1/SM", [&] { k_tma<T><<<nsm, 256, smem>>>(ns, d_idx, map, d_sr, d_out); });
        run("tma gather4 T=512 2/SM", [&] { k_tma<T><<<2 * nsm, 256, smem>>>(ns, d_idx, map, d_sr, d_out); });
    }
    {
        constexpr int T = 1024;
        const size_t smem = 2 * T * 64 + 2 * T * 32 + 64;
        CK(cudaFuncSetAttribute(k_tma<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        run("tma gather4 T=1024 1/SM", [&] { k_tma<T><<<nsm, 256, smem>>>(ns, d_idx, map, d_sr, d_out); });
    }
    {
        constexpr int T = 256;
        const size_t smem = 2 * T * 64 + 2 * T * 32 + 64;
        CK(cudaFuncSetAttribute(k_tma<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        run("tma gather4 T=256 2/SM", [&] { k_tma<T><<<2 * nsm, 256, smem>>>(ns, d_idx, map, d_sr, d_out); });
        run("tma gather4 T=256 4/SM", [&] { k_tma<T><<<4 * nsm, 256, smem>>>(ns, d_idx, map, d_sr, d_out); });
    }
    return 0;
}
