// setup_dev.cu -- device-side setup: Algorithm 1
// coloring and Algorithm 3 agglomeration on the GPU, producing EXACTLY the
// host results (setup.cpp color_level / agglomerate; oracle O2 / O3):
//
//  * Algorithm 1 (reading A24) is a FIFO breadth-first wave whose
//    cells take the least color no earlier-reached neighbour has.  The queue
//    order is reproduced level by level: a newly reached cell belongs to the
//    first frontier cell (queue order) that touches it, and each frontier cell
//    appends its cells in ascending id -- so positions follow from an atomicMin
//    claim, a per-frontier-cell count, an exclusive scan and an ordered write.
//    A cell's color depends only on neighbours with a smaller queue position;
//    inside a level those are resolved in rounds (a cell is colored once all
//    its earlier same-level neighbours are), which gives the sequential result.
//  * Algorithm 3 (readings A18-A22): "first face with a new hash
//    value" = the smallest eligible face id per hash value (atomicMin); the
//    skewness test of a candidate depends on geometry only; the sequential
//    merge loop is a greedy matching in candidate order, equal to the rounds
//    "a live candidate is taken iff it is the smallest live candidate at both
//    of its cells" (lexicographically-first maximal matching).  Coarse ids: an
//    ordered scan over the cells.
//
// Floating point in the skewness test uses explicit round-to-nearest
// intrinsics in the host's operation order (no FMA contraction), so the
// accept / reject decisions are bit-identical to setup.cpp and the oracle.
#include <algorithm>
#include <climits>
#include <memory>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include "gmg_internal.h"

namespace gmg {
namespace {

#define DCK(x)                                                                                 \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) throw std::runtime_error(std::string("device setup: ") + #x + ": " + \
                                                        cudaGetErrorString(e_));               \
    } while (0)

// stream-ordered allocations on the setup stream (pooled: no device-wide
// synchronisation per buffer as with cudaMalloc / cudaFree)
thread_local cudaStream_t t_stream = nullptr;

template <class T>
struct DBuf {
    T *p = nullptr;
    size_t n = 0;
    explicit DBuf(size_t count) : n(count)
    {
        if (count) DCK(cudaMallocAsync((void **)&p, count * sizeof(T), t_stream));
    }
    ~DBuf() { if (p) cudaFreeAsync(p, t_stream); }
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
};

inline int nb(int64_t n, int t = 256) { return (int)((n + t - 1) / t); }

// exclusive scan of n ints (in may equal out); returns the total
int64_t exclusive_scan(const int *in, int *out, int n, cudaStream_t s)
{
    if (n == 0) return 0;
    size_t tb = 0;
    DCK(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, s));
    DBuf<char> tmp(tb);
    int last_in = 0, last_out = 0;
    DCK(cudaMemcpyAsync(&last_in, in + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
    DCK(cudaStreamSynchronize(s));
    DCK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, n, s));
    DCK(cudaMemcpyAsync(&last_out, out + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
    DCK(cudaStreamSynchronize(s));
    return (int64_t)last_out + last_in;
}

// ---------------------------------------------------------------- adjacency
__global__ void k_deg(int nf, const int *__restrict__ fl, const int *__restrict__ fr, int *deg, bool faces)
{
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nf) return;
    const int r = fr[f];
    if (faces) {
        atomicAdd(deg + fl[f], 1);
        if (r >= 0) atomicAdd(deg + r, 1);
    } else if (r >= 0) {
        atomicAdd(deg + fl[f], 1);
        atomicAdd(deg + r, 1);
    }
}

// faces == false: neighbour cells; true: incident face ids
__global__ void k_fill_adj(int nf, const int *__restrict__ fl, const int *__restrict__ fr, int *cur, int *idx,
                           bool faces)
{
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nf) return;
    const int l = fl[f], r = fr[f];
    if (faces) {
        idx[atomicAdd(cur + l, 1)] = f;
        if (r >= 0) idx[atomicAdd(cur + r, 1)] = f;
    } else if (r >= 0) {
        idx[atomicAdd(cur + l, 1)] = r;
        idx[atomicAdd(cur + r, 1)] = l;
    }
}

// sort every (short) list ascending: insertion sort, one thread per cell
__global__ void k_sort_lists(int n, const int *__restrict__ off, int *idx)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int a0 = off[i], a1 = off[i + 1];
    for (int a = a0 + 1; a < a1; ++a) {
        const int v = idx[a];
        int b = a - 1;
        while (b >= a0 && idx[b] > v) { idx[b + 1] = idx[b]; --b; }
        idx[b + 1] = v;
    }
}

struct DevCsr {
    DBuf<int> off, idx;
    DevCsr(int n, int64_t m) : off(n + 1), idx(m > 0 ? m : 1) {}
};

DevCsr *build_adj(int n, int nf, const int *fl, const int *fr, bool faces, bool sorted, cudaStream_t s)
{
    DBuf<int> deg(n + 1);
    DCK(cudaMemsetAsync(deg.p, 0, sizeof(int) * (n + 1), s));
    if (nf) k_deg<<<nb(nf), 256, 0, s>>>(nf, fl, fr, deg.p, faces);
    DBuf<int> off(n + 1);
    const int64_t m = exclusive_scan(deg.p, off.p, n + 1, s);
    DevCsr *g = new DevCsr(n, m);
    DCK(cudaMemcpyAsync(g->off.p, off.p, sizeof(int) * (n + 1), cudaMemcpyDeviceToDevice, s));
    // cursors
    if (nf) k_fill_adj<<<nb(nf), 256, 0, s>>>(nf, fl, fr, off.p, g->idx.p, faces);
    if (sorted && n) k_sort_lists<<<nb(n), 256, 0, s>>>(n, g->off.p, g->idx.p);
    DCK(cudaGetLastError());
    return g;
}

// ---------------------------------------------------------------- Algorithm 1
__global__ void k_claim(int f0, int f1, const int *__restrict__ Q, const int *__restrict__ off,
                        const int *__restrict__ adj, const int *__restrict__ pos, int *ppos)
{
    const int t = f0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= f1) return;
    const int v = Q[t];
    for (int a = off[v]; a < off[v + 1]; ++a) {
        const int w = adj[a];
        if (pos[w] < 0) atomicMin(ppos + w, t);
    }
}

__global__ void k_count_wins(int f0, int f1, const int *__restrict__ Q, const int *__restrict__ off,
                             const int *__restrict__ adj, const int *__restrict__ ppos, int *wins)
{
    const int t = f0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= f1) return;
    const int v = Q[t];
    int c = 0, prev = -1;
    for (int a = off[v]; a < off[v + 1]; ++a) {
        const int w = adj[a];
        if (w != prev && ppos[w] == t) ++c;     // lists are sorted: skip repeated neighbours
        prev = w;
    }
    wins[t - f0] = c;
}

__global__ void k_place(int f0, int f1, const int *Q_in, const int *__restrict__ off,
                        const int *__restrict__ adj, const int *__restrict__ ppos, const int *__restrict__ woff,
                        int *Q, int *pos)
{
    const int t = f0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= f1) return;
    const int v = Q_in[t];
    int o = f1 + woff[t - f0], prev = -1;
    for (int a = off[v]; a < off[v + 1]; ++a) {
        const int w = adj[a];
        if (w != prev && ppos[w] == t) {   // ascending id = the order Algorithm 1 enqueues them
            Q[o] = w;
            pos[w] = o;
            ++o;
        }
        prev = w;
    }
}

// color cells of queue range [q0, q1) whose earlier neighbours are all colored
__global__ void k_color_round(int q0, int q1, const int *__restrict__ Q, const int *__restrict__ off,
                              const int *__restrict__ adj, const int *__restrict__ pos, int *color, int *pending)
{
    const int q = q0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= q1) return;
    const int w = Q[q];
    if (((volatile int *)color)[w] != 0) return;
    uint64_t used = 0;
    bool big = false;
    for (int a = off[w]; a < off[w + 1]; ++a) {
        const int u = adj[a];
        const int pu = pos[u];
        if (pu < 0 || pu >= q) continue;       // reached after w: not colored when w is reached
        const int c = ((volatile int *)color)[u];
        if (c == 0) { atomicAdd(pending, 1); return; }   // an earlier same-level neighbour is not done
        if (c < 64) used |= 1ull << c;
        else big = true;
    }
    int k = 1;
    while (k < 64 && (used >> k & 1ull)) ++k;
    if (k == 64 || big) {                       // more than 63 colors around: slow exact mex
        k = 1;
        for (;;) {
            bool taken = false;
            for (int a = off[w]; a < off[w + 1] && !taken; ++a) {
                const int u = adj[a];
                const int pu = pos[u];
                if (pu >= 0 && pu < q && ((volatile int *)color)[u] == k) taken = true;
            }
            if (!taken) break;
            ++k;
        }
    }
    ((volatile int *)color)[w] = k;
}

// one launch per level: a cell waits (spins) for its earlier same-level
// neighbours -- they have smaller queue positions, hence lower thread and
// block indices, which are dispatched first.  A bounded spin reports failure
// (*stuck) and the caller falls back to k_color_round.
__global__ void k_color_level(int q0, int q1, const int *__restrict__ Q, const int *__restrict__ off,
                              const int *__restrict__ adj, const int *__restrict__ pos, int *color, int *stuck)
{
    const int q = q0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= q1) return;
    const int w = Q[q];
    uint64_t used = 0;
    bool big = false;
    for (int a = off[w]; a < off[w + 1]; ++a) {
        const int u = adj[a];
        const int pu = pos[u];
        if (pu < 0 || pu >= q) continue;
        int c = ((volatile int *)color)[u];
        for (int spin = 0; c == 0; ++spin) {
            if (spin > (1 << 22) || *(volatile int *)stuck) { atomicExch(stuck, 1); return; }
            __nanosleep(32);
            c = ((volatile int *)color)[u];
        }
        if (c < 64) used |= 1ull << c;
        else big = true;
    }
    int k = 1;
    while (k < 64 && (used >> k & 1ull)) ++k;
    if (k == 64 || big) {
        k = 1;
        for (;;) {
            bool taken = false;
            for (int a = off[w]; a < off[w + 1] && !taken; ++a) {
                const int u = adj[a];
                const int pu = pos[u];
                if (pu >= 0 && pu < q && ((volatile int *)color)[u] == k) taken = true;
            }
            if (!taken) break;
            ++k;
        }
    }
    __threadfence();
    ((volatile int *)color)[w] = k;
}

__global__ void k_first_uncolored(int n, const int *__restrict__ color, int *first)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && color[i] == 0) atomicMin(first, i);
}

__global__ void k_seed(int v, int q, int *Q, int *pos, int *color)
{
    Q[q] = v;
    pos[v] = q;
    color[v] = 1;
}

// ---------------------------------------------------------------- Algorithm 3
__device__ __forceinline__ uint64_t face_hash(uint64_t l, uint64_t r, uint64_t m)
{
    return (23ull * (l + r) + l * r) % m;   // Eq.(hash value), uint64 (A19)
}

__global__ void k_hash_min(int nf, const int *__restrict__ fl, const int *__restrict__ fr,
                           const int *__restrict__ part, uint64_t n_int, int *win)
{
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nf) return;
    const int l = fl[f], r = fr[f];
    if (r < 0) return;                                  // boundary face
    if (part && part[l] != part[r]) return;             // parallel interface
    atomicMin(win + face_hash((uint64_t)l, (uint64_t)r, n_int), f);
}

__global__ void k_cand_flag(int nf, const int *__restrict__ fl, const int *__restrict__ fr,
                            const int *__restrict__ part, uint64_t n_int, const int *__restrict__ win, int *flag)
{
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nf) return;
    const int l = fl[f], r = fr[f];
    int ok = 0;
    if (r >= 0 && !(part && part[l] != part[r])) ok = win[face_hash((uint64_t)l, (uint64_t)r, n_int)] == f;
    flag[f] = ok;
}

__global__ void k_scatter_flagged(int n, const int *__restrict__ flag, const int *__restrict__ off, int *out)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && flag[i]) out[off[i]] = i;
}

// skewness test of candidate s (host agglomerate, same operation order)
__global__ void k_skew(int ncand, int dim, int n, int nf, const int *__restrict__ cand, const int *__restrict__ fl,
                       const int *__restrict__ fr, const double *__restrict__ vol, const double *__restrict__ ctr,
                       const double *__restrict__ avec, const double *__restrict__ fctr, const int *__restrict__ ioff,
                       const int *__restrict__ iidx, double theta, int *live)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= ncand) return;
    const int f = cand[s], l = fl[f], r = fr[f];
    const double Vl = vol[l], Vr = vol[r];
    double Cv[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < dim; ++k)
        Cv[k] = __ddiv_rn(__dadd_rn(__dmul_rn(Vl, ctr[(size_t)k * n + l]), __dmul_rn(Vr, ctr[(size_t)k * n + r])),
                          __dadd_rn(Vl, Vr));
    double smin = 2.0;
    for (int side = 0; side < 2; ++side) {
        const int c = side == 0 ? l : r;
        for (int a = ioff[c]; a < ioff[c + 1]; ++a) {
            const int g = iidx[a];
            const int gl = fl[g], gr = fr[g];
            if ((gl == l && gr == r) || (gl == r && gr == l)) continue;
            const double sg = (gl == c) ? 1.0 : -1.0;
            double A[3] = {0.0, 0.0, 0.0}, dv[3] = {0.0, 0.0, 0.0}, nv[3] = {0.0, 0.0, 0.0};
            for (int k = 0; k < dim; ++k) A[k] = avec[(size_t)k * nf + g];
            double S2 = __dmul_rn(A[0], A[0]);
            S2 = __dadd_rn(S2, __dmul_rn(A[1], A[1]));
            if (dim == 3) S2 = __dadd_rn(S2, __dmul_rn(A[2], A[2]));
            const double S = __dsqrt_rn(S2);
            for (int k = 0; k < dim; ++k) {
                nv[k] = __ddiv_rn(__dmul_rn(sg, A[k]), S);
                dv[k] = __dsub_rn(fctr[(size_t)k * nf + g], Cv[k]);
            }
            double dn = __dmul_rn(dv[0], nv[0]);
            dn = __dadd_rn(dn, __dmul_rn(dv[1], nv[1]));
            double dd = __dmul_rn(dv[0], dv[0]);
            dd = __dadd_rn(dd, __dmul_rn(dv[1], dv[1]));
            if (dim == 3) { dn = __dadd_rn(dn, __dmul_rn(dv[2], nv[2])); dd = __dadd_rn(dd, __dmul_rn(dv[2], dv[2])); }
            const double sk = (dd == 0.0) ? 1.0 : __ddiv_rn(dn, __dsqrt_rn(dd));
            if (sk < smin) smin = sk;
        }
    }
    live[s] = smin >= theta ? 1 : 0;
}

// greedy matching rounds over live candidates (index order = selection order)
__global__ void k_match_reset(int ncand, const int *__restrict__ cand, const int *__restrict__ fl,
                              const int *__restrict__ fr, const int *__restrict__ live, int *best)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= ncand || !live[s]) return;
    const int f = cand[s];
    best[fl[f]] = INT_MAX;
    best[fr[f]] = INT_MAX;
}

__global__ void k_match_min(int ncand, const int *__restrict__ cand, const int *__restrict__ fl,
                            const int *__restrict__ fr, const int *__restrict__ live, int *best)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= ncand || !live[s]) return;
    const int f = cand[s];
    atomicMin(best + fl[f], s);
    atomicMin(best + fr[f], s);
}

__global__ void k_match_take(int ncand, const int *__restrict__ cand, const int *__restrict__ fl,
                             const int *__restrict__ fr, const int *__restrict__ best, int *live, int *partner)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= ncand || !live[s]) return;
    const int f = cand[s], l = fl[f], r = fr[f];
    if (best[l] == s && best[r] == s) {
        partner[l] = r;
        partner[r] = l;
        live[s] = 2;                         // taken this round
    }
}

__global__ void k_match_kill(int ncand, const int *__restrict__ cand, const int *__restrict__ fl,
                             const int *__restrict__ fr, const int *__restrict__ partner, int *live, int *nlive)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= ncand || !live[s]) return;
    if (live[s] == 2) { live[s] = 0; return; }
    const int f = cand[s];
    if (partner[fl[f]] >= 0 || partner[fr[f]] >= 0) { live[s] = 0; return; }
    atomicAdd(nlive, 1);
}

__global__ void k_root_flag(int n, const int *__restrict__ partner, int *flag)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flag[i] = !(partner[i] >= 0 && partner[i] < i);
}

__global__ void k_parent(int n, const int *__restrict__ partner, const int *__restrict__ ids, int *parent)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int p = partner[i];
    parent[i] = (p >= 0 && p < i) ? ids[p] : ids[i];
}

struct Faces {
    DBuf<int> fl, fr;
    Faces(const HostLevel &L, cudaStream_t s) : fl(L.nf), fr(L.nf)
    {
        std::vector<int> l(L.nf), r(L.nf);
        for (int64_t f = 0; f < L.nf; ++f) {
            l[f] = (int)L.left[f];
            r[f] = L.right[f] >= 0 ? (int)L.right[f] : -1;
        }
        DCK(cudaMemcpyAsync(fl.p, l.data(), sizeof(int) * L.nf, cudaMemcpyHostToDevice, s));
        DCK(cudaMemcpyAsync(fr.p, r.data(), sizeof(int) * L.nf, cudaMemcpyHostToDevice, s));
        DCK(cudaStreamSynchronize(s));
    }
};

}  // namespace

// Algorithm 1 on the device; same colors as color_level(L)
int color_level_dev(HostLevel &L, cudaStream_t s, SetupStats *st)
{
    t_stream = s;
    const int n = (int)L.n, nf = (int)L.nf;
    Faces F(L, s);
    std::unique_ptr<DevCsr> g(build_adj(n, nf, F.fl.p, F.fr.p, false, true, s));
    DBuf<int> color(n), pos(n), ppos(n), Q(n), wins(n + 1), woff(n + 1), pend(1), first(1);
    DCK(cudaMemsetAsync(color.p, 0, sizeof(int) * n, s));
    DCK(cudaMemsetAsync(pos.p, 0xff, sizeof(int) * n, s));      // -1
    DCK(cudaMemsetAsync(ppos.p, 0x7f, sizeof(int) * n, s));     // large positive
    int qend = 0, seed = 0, levels = 0, rounds = 0;
    while (qend < n) {
        k_seed<<<1, 1, 0, s>>>(seed, qend, Q.p, pos.p, color.p);
        int f0 = qend, f1 = qend + 1;
        while (f1 > f0) {
            const int fn = f1 - f0;
            k_claim<<<nb(fn), 256, 0, s>>>(f0, f1, Q.p, g->off.p, g->idx.p, pos.p, ppos.p);
            k_count_wins<<<nb(fn), 256, 0, s>>>(f0, f1, Q.p, g->off.p, g->idx.p, ppos.p, wins.p);
            const int total = (int)exclusive_scan(wins.p, woff.p, fn, s);
            if (total) {
                k_place<<<nb(fn), 256, 0, s>>>(f0, f1, Q.p, g->off.p, g->idx.p, ppos.p, woff.p, Q.p, pos.p);
                int stuck = 0;
                DCK(cudaMemsetAsync(pend.p, 0, sizeof(int), s));
                k_color_level<<<nb(total), 256, 0, s>>>(f1, f1 + total, Q.p, g->off.p, g->idx.p, pos.p, color.p, pend.p);
                DCK(cudaMemcpyAsync(&stuck, pend.p, sizeof(int), cudaMemcpyDeviceToHost, s));
                DCK(cudaStreamSynchronize(s));
                ++rounds;
                while (stuck) {   // fallback: synchronous rounds (colors already set are final)
                    DCK(cudaMemsetAsync(pend.p, 0, sizeof(int), s));
                    k_color_round<<<nb(total), 256, 0, s>>>(f1, f1 + total, Q.p, g->off.p, g->idx.p, pos.p, color.p, pend.p);
                    DCK(cudaMemcpyAsync(&stuck, pend.p, sizeof(int), cudaMemcpyDeviceToHost, s));
                    DCK(cudaStreamSynchronize(s));
                    ++rounds;
                }
            }
            f0 = f1;
            f1 += total;
            ++levels;
        }
        qend = f1;
        if (qend >= n) break;
        // restart at the least uncolored id (disconnected mesh)
        const int big = INT_MAX;
        DCK(cudaMemcpyAsync(first.p, &big, sizeof(int), cudaMemcpyHostToDevice, s));
        k_first_uncolored<<<nb(n), 256, 0, s>>>(n, color.p, first.p);
        DCK(cudaMemcpyAsync(&seed, first.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        DCK(cudaStreamSynchronize(s));
        if (seed == INT_MAX) break;
    }
    std::vector<int> c(n);
    DCK(cudaMemcpyAsync(c.data(), color.p, sizeof(int) * n, cudaMemcpyDeviceToHost, s));
    DCK(cudaStreamSynchronize(s));
    L.color.assign(c.begin(), c.end());
    int nc = 0;
    for (int v : c) nc = std::max(nc, v);
    L.ncolor = nc;
    if (st) { st->color_levels += levels; st->color_rounds += rounds; }
    return nc;
}

// Algorithm 3 on the device; same parent map as agglomerate(L, theta, ...)
int64_t agglomerate_dev(const HostLevel &L, double theta, std::vector<int64_t> &parent, int64_t &nc, cudaStream_t s,
                        SetupStats *st)
{
    t_stream = s;
    const int n = (int)L.n, nf = (int)L.nf, d = L.dim;
    uint64_t n_int = 0;
    for (int64_t f = 0; f < L.nf; ++f) n_int += (L.right[f] >= 0);
    Faces F(L, s);
    DBuf<int> partner(n), part(L.part.empty() ? 0 : n);
    DCK(cudaMemsetAsync(partner.p, 0xff, sizeof(int) * n, s));
    if (!L.part.empty()) DCK(cudaMemcpyAsync(part.p, L.part.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
    int64_t merged = 0;
    int rounds = 0;
    if (n_int) {
        DBuf<int> win(n_int), flag(nf + 1), foff(nf + 1);
        DCK(cudaMemsetAsync(win.p, 0x7f, sizeof(int) * n_int, s));
        k_hash_min<<<nb(nf), 256, 0, s>>>(nf, F.fl.p, F.fr.p, part.p, n_int, win.p);
        k_cand_flag<<<nb(nf), 256, 0, s>>>(nf, F.fl.p, F.fr.p, part.p, n_int, win.p, flag.p);
        const int ncand = (int)exclusive_scan(flag.p, foff.p, nf, s);
        DBuf<int> cand(ncand > 0 ? ncand : 1), live(ncand > 0 ? ncand : 1), best(n), nlive(1);
        k_scatter_flagged<<<nb(nf), 256, 0, s>>>(nf, flag.p, foff.p, cand.p);
        // geometry
        DBuf<double> vol(n), ctr((size_t)d * n), avec((size_t)d * nf), fctr((size_t)d * nf);
        DCK(cudaMemcpyAsync(vol.p, L.vol.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
        DCK(cudaMemcpyAsync(ctr.p, L.ctr.data(), sizeof(double) * d * n, cudaMemcpyHostToDevice, s));
        DCK(cudaMemcpyAsync(avec.p, L.avec.data(), sizeof(double) * d * nf, cudaMemcpyHostToDevice, s));
        DCK(cudaMemcpyAsync(fctr.p, L.fctr.data(), sizeof(double) * d * nf, cudaMemcpyHostToDevice, s));
        std::unique_ptr<DevCsr> inc(build_adj(n, nf, F.fl.p, F.fr.p, true, false, s));
        if (ncand)
            k_skew<<<nb(ncand), 256, 0, s>>>(ncand, d, n, nf, cand.p, F.fl.p, F.fr.p, vol.p, ctr.p, avec.p, fctr.p,
                                             inc->off.p, inc->idx.p, theta, live.p);
        for (int nl = ncand; nl > 0;) {
            k_match_reset<<<nb(ncand), 256, 0, s>>>(ncand, cand.p, F.fl.p, F.fr.p, live.p, best.p);
            k_match_min<<<nb(ncand), 256, 0, s>>>(ncand, cand.p, F.fl.p, F.fr.p, live.p, best.p);
            k_match_take<<<nb(ncand), 256, 0, s>>>(ncand, cand.p, F.fl.p, F.fr.p, best.p, live.p, partner.p);
            DCK(cudaMemsetAsync(nlive.p, 0, sizeof(int), s));
            k_match_kill<<<nb(ncand), 256, 0, s>>>(ncand, cand.p, F.fl.p, F.fr.p, partner.p, live.p, nlive.p);
            DCK(cudaMemcpyAsync(&nl, nlive.p, sizeof(int), cudaMemcpyDeviceToHost, s));
            DCK(cudaStreamSynchronize(s));
            ++rounds;
        }
    }
    DBuf<int> rflag(n), ids(n), par(n);
    k_root_flag<<<nb(n), 256, 0, s>>>(n, partner.p, rflag.p);
    nc = exclusive_scan(rflag.p, ids.p, n, s);
    k_parent<<<nb(n), 256, 0, s>>>(n, partner.p, ids.p, par.p);
    std::vector<int> p(n), pa(n);
    DCK(cudaMemcpyAsync(p.data(), par.p, sizeof(int) * n, cudaMemcpyDeviceToHost, s));
    DCK(cudaMemcpyAsync(pa.data(), partner.p, sizeof(int) * n, cudaMemcpyDeviceToHost, s));
    DCK(cudaStreamSynchronize(s));
    parent.assign(p.begin(), p.end());
    for (int i = 0; i < n; ++i) merged += (pa[i] >= 0 && pa[i] > i);
    if (st) st->match_rounds += rounds;
    return merged;
}

}  // namespace gmg
