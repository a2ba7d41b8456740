// api.cu -- the C ABI of libgmg (include/gmg.h): context, workspace, data
// movement, kernel orchestration of residual / smoothing / V-cycle, halo
// exchange (NCCL between ranks, device copies between local domains) and the
// CUDA-graph capture of one V-cycle.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <stdexcept>

#include "gmg_internal.h"
#include "kernels.cuh"
#include "kernels_tried.cuh"

namespace gmg {
// ho.cu (NEXT-1): which = 0 k_ho_sr, 1 k_ho_recon, 2 k_ho_flux, 3 k_ho_gather(mode)
void ho_launch(int which, const DevLevel &L, const HoDev &H, const Phys &ph, const BCs &bc, const gmg_options &o,
               int mode, double *Rout, double *aout, cudaStream_t s);
}

using namespace gmg;

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            ctx->err = std::string(#x) + ": " + cudaGetErrorString(e_);               \
            return GMG_ECUDA;                                                         \
        }                                                                             \
    } while (0)

namespace {

inline int nblk(int64_t n, int b = 256) { return (int)std::max<int64_t>(1, (n + b - 1) / b); }

Phys phys(const gmg_ctx *ctx)
{
    Phys p;
    p.gamma = ctx->opt.gamma;
    p.gm1 = ctx->opt.gamma - 1.0;
    p.K = ctx->opt.dim == 3 ? (5.0 - 3.0 * p.gamma) / (p.gamma - 1.0) : (4.0 - 2.0 * p.gamma) / (p.gamma - 1.0);
    p.omega = ctx->opt.r_factor;
    return p;
}

BCs bcs(const gmg_ctx *ctx)
{
    BCs b;
    for (int q = 0; q < 5; ++q) b.winf[q] = ctx->winf[q];
    for (int k = 0; k < 16; ++k) b.kind[k] = k < (int)ctx->patch_kind.size() ? ctx->patch_kind[k] : 0;
    return b;
}

// ---------------------------------------------------------------------------
// NCCL, resolved at run time (the process normally already has torch's
// libnccl.so.2 loaded; no link-time dependency, single-GPU runs never load it)
// ---------------------------------------------------------------------------
struct Nccl {
    void *h = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char *(*ErrStr)(ncclResult_t) = nullptr;
    bool load(std::string &err)
    {
        if (h) return true;
        const char *cands[] = {std::getenv("GMG_NCCL_LIB"), "libnccl.so.2", "/usr/lib/x86_64-linux-gnu/libnccl.so.2"};
        for (const char *c : cands)
            if (c && (h = dlopen(c, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!h) { err = "libnccl.so.2 not found (set GMG_NCCL_LIB)"; return false; }
        CommInitRank = (decltype(CommInitRank))dlsym(h, "ncclCommInitRank");
        CommDestroy = (decltype(CommDestroy))dlsym(h, "ncclCommDestroy");
        Send = (decltype(Send))dlsym(h, "ncclSend");
        Recv = (decltype(Recv))dlsym(h, "ncclRecv");
        GroupStart = (decltype(GroupStart))dlsym(h, "ncclGroupStart");
        GroupEnd = (decltype(GroupEnd))dlsym(h, "ncclGroupEnd");
        AllReduce = (decltype(AllReduce))dlsym(h, "ncclAllReduce");
        ErrStr = (decltype(ErrStr))dlsym(h, "ncclGetErrorString");
        if (!CommInitRank || !Send || !Recv || !GroupStart || !GroupEnd || !AllReduce) {
            err = "libnccl.so.2 lacks required symbols";
            return false;
        }
        return true;
    }
};
Nccl &nccl()
{
    static Nccl n;
    return n;
}

// --------------------------------------------------------------------------
// launch bookkeeping: algorithmic bytes and optional per-launch CUDA events
// --------------------------------------------------------------------------
struct Launcher {
    gmg_ctx *ctx;
    cudaStream_t s;
    void pre(int)
    {
        if (ctx->prof.on) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            cudaEventRecord(e, s);
            ctx->prof.ev.push_back(e);
        }
    }
    void post(int cls, double bytes)
    {
        ctx->launches++;
        ctx->kbytes[cls] += bytes;
        if (ctx->prof.on) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            cudaEventRecord(e, s);
            ctx->prof.ev.push_back(e);
            ctx->prof.marks.push_back({cls, (int)ctx->prof.ev.size() - 2});
            ctx->prof.bytes.push_back(bytes);
        }
    }
};

// every V-cycle kernel goes through here: optional programmatic dependent
// launch (PDL) so a kernel's launch overlaps its predecessor's drain; the
// kernels call pdl_enter() (griddepcontrol.wait) before touching its outputs
template <typename... KP, typename... A>
void klaunch(gmg_ctx *ctx, void (*k)(KP...), dim3 g, dim3 b, cudaStream_t s, A... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = g;
    cfg.blockDim = b;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    if (ctx->pdl) {
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
    }
    cudaLaunchKernelEx(&cfg, k, args...);
}

constexpr int kRecStride = 12;   // Rec<2>::STRIDE == Rec<3>::STRIDE

// prep: the launch also writes the sweep slot records (A outward | S r) of
// both cells of every interior face (whole 32-byte records)
template <int D>
void enqueue_face(Launcher &Lc, Domain &dm, int l, const double *W, bool flux, bool from_rec, bool df = false,
                  bool prep = false)
{
    gmg_ctx *ctx = Lc.ctx;
    DevLevel &L = dm.dv[l];
    constexpr int RS = Rec<D>::STRIDE, NV = D + 2;
    Lc.pre(GMG_K_FACE);
    const dim3 g(nblk(L.nf)), b(256);
    const Phys ph = phys(ctx);
    const BCs bc = bcs(ctx);
    if (prep) {
        if (flux && df && !from_rec) klaunch(ctx, k_face<D, true, NV, true, true>, g, b, Lc.s, L, W, ph, bc);
        else if (flux && !df && from_rec) klaunch(ctx, k_face<D, true, RS, false, true>, g, b, Lc.s, L, W, ph, bc);
        else if (flux && !df && !from_rec) klaunch(ctx, k_face<D, true, NV, false, true>, g, b, Lc.s, L, W, ph, bc);
        else if (!flux && from_rec) klaunch(ctx, k_face<D, false, RS, false, true>, g, b, Lc.s, L, W, ph, bc);
        else if (!flux && !from_rec) klaunch(ctx, k_face<D, false, NV, false, true>, g, b, Lc.s, L, W, ph, bc);
        else { ctx->err = "enqueue_face: unsupported prep variant"; return; }
    } else if (flux && df) {
        if (from_rec) klaunch(ctx, k_face<D, true, RS, true, false>, g, b, Lc.s, L, W, ph, bc);
        else klaunch(ctx, k_face<D, true, NV, true, false>, g, b, Lc.s, L, W, ph, bc);
    } else if (flux) {
        if (from_rec) klaunch(ctx, k_face<D, true, RS, false, false>, g, b, Lc.s, L, W, ph, bc);
        else klaunch(ctx, k_face<D, true, NV, false, false>, g, b, Lc.s, L, W, ph, bc);
    } else {
        if (from_rec) klaunch(ctx, k_face<D, false, RS, false, false>, g, b, Lc.s, L, W, ph, bc);
        else klaunch(ctx, k_face<D, false, NV, false, false>, g, b, Lc.s, L, W, ph, bc);
    }
    Lc.post(GMG_K_FACE, (flux ? dm.lbytes[l].face_flux : dm.lbytes[l].face_prep) + (prep ? dm.lbytes[l].face_slots : 0.0));
}

// with G_NORM the domain's residual sums of squares land in d_sumsq[di]
template <int D>
void enqueue_gather(Launcher &Lc, Domain &dm, int di, int l, int flags, double *Wexp)
{
    gmg_ctx *ctx = Lc.ctx;
    DevLevel &L = dm.dv[l];
    if ((flags & G_PREPARE) && ctx->opt.df_mode == 3) flags |= G_BETA;   // fixed-beta relaxation
    GArgs a{flags, ctx->opt.cfl_imp, ctx->opt.cfl_exp, Wexp, L.partial, ctx->opt.beta};
    Lc.pre(GMG_K_GATHER);
    klaunch(Lc.ctx, k_gather<D>, dim3(nblk(L.n)), dim3(256), Lc.s, L, a);
    Lc.post(GMG_K_GATHER, dm.lbytes[l].gather);
    if (flags & G_NORM) {
        Lc.pre(GMG_K_NORM);
        klaunch(Lc.ctx, k_norm_sum, dim3(1), dim3(256), Lc.s, L.partial, nblk(L.n), L.nv, ctx->d_sumsq + (size_t)di * L.nv);
        Lc.post(GMG_K_NORM, (double)nblk(L.n) * L.nv * 8);
    }
}

// all-reduce the per-domain sums across ranks, then one history entry
void enqueue_norm_hist(Launcher &Lc)
{
    gmg_ctx *ctx = Lc.ctx;
    const int nv = ctx->opt.dim + 2;
    if (ctx->opt.nranks > 1)
        nccl().AllReduce(ctx->d_sumsq, ctx->d_sumsq, nv, ncclDouble, ncclSum, (ncclComm_t)ctx->nccl_comm, Lc.s);
    Lc.pre(GMG_K_NORM);
    klaunch(Lc.ctx, k_norm_hist, dim3(1), dim3(32), Lc.s, ctx->d_sumsq, (int)ctx->dom.size(), nv, ctx->d_hist, ctx->hist_cap, ctx->d_flag);
    Lc.post(GMG_K_NORM, 0.0);
}

// --------------------------------------------------------------------------
// halo exchange (a13).  kind: increments of one color, record W_lin (+ dW
// = 0) of all colors, or the state W of all colors.
// --------------------------------------------------------------------------
enum { EX_DW = 0, EX_WLIN = 1, EX_W = 2 };

template <int D>
void enqueue_exchange(Launcher &Lc, int l, int kind, int color)
{
    gmg_ctx *ctx = Lc.ctx;
    if (ctx->nparts <= 1) return;
    constexpr int NV = D + 2;
    using RC = Rec<D>;
    const int ncolor = ctx->lv[l].ncolor;
    int stride = RC::STRIDE, offset = RC::DW, zero_at = 0, nzero = 0;
    if (kind == EX_WLIN) { offset = RC::W; zero_at = RC::DW; nzero = NV; }
    if (kind == EX_W) { stride = NV; offset = 0; }
    auto src_of = [&](DevLevel &L) { return kind == EX_W ? L.W : L.rec; };
    auto grange = [&](const DomLevel &H, int &g0, int &g1) {
        const int np = (int)H.peers.size();
        g0 = color >= 0 ? color * np : 0;
        g1 = color >= 0 ? (color + 1) * np : ncolor * np;
    };
    // pack
    for (Domain &dm : ctx->dom) {
        const DomLevel &H = dm.lv[l];
        DevLevel &L = dm.dv[l];
        int g0, g1;
        grange(H, g0, g1);
        const int64_t s0 = H.send_off[g0], s1 = H.send_off[g1];
        if (s1 > s0) {
            Lc.pre(GMG_K_NORM);
            klaunch(Lc.ctx, k_pack, dim3(nblk(s1 - s0)), dim3(256), Lc.s, (int)(s1 - s0), L.send_idx + s0, src_of(L), stride, offset, NV,
                                                   L.sendbuf + s0 * NV);
            Lc.post(GMG_K_NORM, (double)(s1 - s0) * NV * 16);
        }
    }
    // transport
    if (ctx->opt.nranks > 1) {
        Domain &dm = ctx->dom[0];
        const DomLevel &H = dm.lv[l];
        DevLevel &L = dm.dv[l];
        const int np = (int)H.peers.size();
        int g0, g1;
        grange(H, g0, g1);
        nccl().GroupStart();
        for (int g = g0; g < g1; ++g) {
            const int peer = H.peers[g % np];
            const int64_t sc = H.send_off[g + 1] - H.send_off[g], rc = H.recv_off[g + 1] - H.recv_off[g];
            if (sc) nccl().Send(L.sendbuf + H.send_off[g] * NV, sc * NV, ncclDouble, peer, (ncclComm_t)ctx->nccl_comm, Lc.s);
            if (rc) nccl().Recv(L.recvbuf + H.recv_off[g] * NV, rc * NV, ncclDouble, peer, (ncclComm_t)ctx->nccl_comm, Lc.s);
        }
        nccl().GroupEnd();
    } else {
        for (Domain &dm : ctx->dom) {
            const DomLevel &H = dm.lv[l];
            const int np = (int)H.peers.size();
            int g0, g1;
            grange(H, g0, g1);
            for (int g = g0; g < g1; ++g) {
                const int64_t sc = H.send_off[g + 1] - H.send_off[g];
                if (!sc) continue;
                Domain &dp = ctx->dom[H.peers[g % np]];
                const DomLevel &Hp = dp.lv[l];
                const int npp = (int)Hp.peers.size();
                const int kk = (int)(std::lower_bound(Hp.peers.begin(), Hp.peers.end(), dm.rank) - Hp.peers.begin());
                const int gp = (g / np) * npp + kk;
                cudaMemcpyAsync(dp.dv[l].recvbuf + Hp.recv_off[gp] * NV, dm.dv[l].sendbuf + H.send_off[g] * NV,
                                sizeof(double) * sc * NV, cudaMemcpyDeviceToDevice, Lc.s);
            }
        }
    }
    // unpack
    for (Domain &dm : ctx->dom) {
        const DomLevel &H = dm.lv[l];
        DevLevel &L = dm.dv[l];
        int g0, g1;
        grange(H, g0, g1);
        const int64_t r0 = H.recv_off[g0], r1 = H.recv_off[g1];
        if (r1 > r0) {
            Lc.pre(GMG_K_NORM);
            klaunch(Lc.ctx, k_unpack, dim3(nblk(r1 - r0)), dim3(256), Lc.s, (int)(r1 - r0), L.recv_idx + r0, L.recvbuf + r0 * NV,
                                                     src_of(L), stride, offset, NV, zero_at, nzero);
            Lc.post(GMG_K_NORM, (double)(r1 - r0) * NV * 16);
        }
    }
    ctx->exchanges++;
}

template <int D>
void enqueue_ghost_wlin(Launcher &Lc, int l)
{
    for (Domain &dm : Lc.ctx->dom) {
        DevLevel &L = dm.dv[l];
        if (L.n_loc > L.n) {
            Lc.pre(GMG_K_NORM);
            klaunch(Lc.ctx, k_ghost_wlin<D>, dim3(nblk(L.n_loc - L.n)), dim3(256), Lc.s, L.n, L.n_loc, L.W, L.rec);
            Lc.post(GMG_K_NORM, 0.0);
        }
    }
}

template <int D>
void enqueue_ghost_w(Launcher &Lc, int l)
{
    for (Domain &dm : Lc.ctx->dom) {
        DevLevel &L = dm.dv[l];
        if (L.n_loc > L.n) {
            Lc.pre(GMG_K_NORM);
            klaunch(Lc.ctx, k_ghost_w<D>, dim3(nblk(L.n_loc - L.n)), dim3(256), Lc.s, L.n, L.n_loc, L.rec, L.W);
            Lc.post(GMG_K_NORM, 0.0);
        }
    }
}

// --------------------------------------------------------------------------
// sweeps
// --------------------------------------------------------------------------
// optional L2 access-policy window over the level's cell records (the
// gathered data), attached per launch so that graph capture keeps it
// sweep grid cap = resident waves x SMs x blocks/SM (set in gmg_set_workspace; 0 = one thread per cell)

template <class K>
void launch_with_window(K kernel, dim3 g, dim3 b, cudaStream_t s, const SweepArgs &a, const void *win, size_t win_bytes,
                        bool pdl, float hit = 1.0f)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = g;
    cfg.blockDim = b;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (win && win_bytes) {
        at[na].id = cudaLaunchAttributeAccessPolicyWindow;
        at[na].val.accessPolicyWindow.base_ptr = const_cast<void *>(win);
        at[na].val.accessPolicyWindow.num_bytes = win_bytes;
        at[na].val.accessPolicyWindow.hitRatio = hit;
        at[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        at[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        ++na;
    }
    if (pdl) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = na ? at : nullptr;
    cfg.numAttrs = na;
    cudaLaunchKernelEx(&cfg, kernel, a);
}

template <int D, int LPC>
void launch_sweep(const gmg_ctx *ctx, const SweepArgs &a, cudaStream_t s, const void *win, size_t win_bytes)
{
    const int minb = ctx->minb, sweep_var = ctx->sweep_var;
    const bool pdl = ctx->pdl != 0;
    // a window larger than the set-aside persists that fraction of its lines (GMG_L2FULL)
    const float hit = (ctx->l2_window && win_bytes > ctx->l2_window) ? (float)((double)ctx->l2_window / (double)win_bytes) : 1.0f;
    const int64_t nthreads = (int64_t)(a.cend - a.cbeg) * LPC;
    if (ctx->sweep_bs == 64 && sweep_var == 3 && minb == 4) {   // GMG_SWEEP_BS=64: 16 blocks of 64 per SM
        int nb = (int)((nthreads + 63) / 64);
        if (ctx->sweep_grid_cap > 0) nb = std::min(nb, 4 * ctx->sweep_grid_cap);
        launch_with_window(k_sweep64<D, LPC>, dim3(nb), dim3(64), s, a, win, win_bytes, pdl, hit);
        return;
    }
    if (ctx->sweep_bs == 128 && sweep_var == 3 && minb == 9) {   // GMG_MINB=9: 9 blocks of 128 per SM (56 registers)
        int nb = (int)((nthreads + 127) / 128);
        if (ctx->sweep_grid_cap > 0) nb = std::min(nb, (9 * ctx->sweep_grid_cap) / 4);
        launch_with_window(k_sweep128<D, LPC, 3 | 8, 9>, dim3(nb), dim3(128), s, a, win, win_bytes, pdl, hit);
        return;
    }
    if (ctx->sweep_bs == 128 && (sweep_var == 3 || sweep_var == 19 || sweep_var == 35) && minb == 4) {   // default; the variants run at 256
        int nb = (int)((nthreads + 127) / 128);
        if (ctx->sweep_grid_cap > 0) nb = std::min(nb, 2 * ctx->sweep_grid_cap);
        if (sweep_var == 19) launch_with_window(k_sweep128<D, LPC, 3 | 8 | 16>, dim3(nb), dim3(128), s, a, win, win_bytes, pdl, hit);
        else if (sweep_var == 35) launch_with_window(k_sweep128<D, LPC, 3 | 8 | 32>, dim3(nb), dim3(128), s, a, win, win_bytes, pdl, hit);
        else launch_with_window(k_sweep128<D, LPC>, dim3(nb), dim3(128), s, a, win, win_bytes, pdl, hit);
        return;
    }
    int nb = nblk(nthreads);
    if (ctx->sweep_grid_cap > 0) nb = std::min(nb, ctx->sweep_grid_cap);
    const dim3 g(nb), b(256);
    // variants kept for the record; 3 is the default
    if (sweep_var == 0) { launch_with_window(k_sweep<D, LPC, 4, 0>, g, b, s, a, win, win_bytes, pdl); return; }
    if (sweep_var == 1) { launch_with_window(k_sweep<D, LPC, 4, 1>, g, b, s, a, win, win_bytes, pdl); return; }
    if (sweep_var == 2) { launch_with_window(k_sweep<D, LPC, 4, 2>, g, b, s, a, win, win_bytes, pdl); return; }
    if (sweep_var == 7) { launch_with_window(k_sweep<D, LPC, 4, 7>, g, b, s, a, win, win_bytes, pdl); return; }
    switch (minb) {
        case 6: launch_with_window(k_sweep<D, LPC, 6>, g, b, s, a, win, win_bytes, pdl); break;
        case 8: launch_with_window(k_sweep<D, LPC, 8>, g, b, s, a, win, win_bytes, pdl); break;
        default: launch_with_window(k_sweep<D, LPC, 4>, g, b, s, a, win, win_bytes, pdl); break;
    }
}

// one color block of one domain (Eq.(gpu-forward-relaxation) / (gpu-backward-relaxation))
// part: 0 = whole block, 1 = its boundary cells (ghost neighbours), 2 = its interior cells
// first_fwd: a phase of the first forward half-sweep of a smoothing step --
// owned neighbours of later colors still hold dW = +0 (zeroed before the
// step), so their terms are exactly +0 and the kernel skips them
template <int D>
void enqueue_sweep_color(Launcher &Lc, Domain &dm, int l, int c, const double *rhs, double *Wout, int part = 0,
                         bool first_fwd = false)
{
    gmg_ctx *ctx = Lc.ctx;
    DevLevel &L = dm.dv[l];
    const DomLevel &H = dm.lv[l];
    int b0 = (int)H.blk[c], b1 = (int)H.blk[c + 1];
    const int zlo = (first_fwd && ctx->skip_zero) ? (int)H.blk[c + 1] : 0;
    const int zhi = (first_fwd && ctx->skip_zero) ? (int)H.n_own : 0;
    if (part) {
        const int mid = b0 + (int)H.nbnd[c];
        const double frac = b1 > b0 ? (double)(part == 1 ? mid - b0 : b1 - mid) / (b1 - b0) : 0.0;
        if (part == 1) b1 = mid;
        else b0 = mid;
        SweepArgs a{b0, b1, ctx->opt.gamma - 1.0, L.rec, L.ecell, L.deg_int, L.sinfo, L.sJe, L.sRe, rhs, Wout, zlo, zhi};
        if (b1 <= b0) return;
        Lc.pre(GMG_K_SWEEP);
        switch (ctx->lpc) {
            case 1: launch_sweep<D, 1>(ctx, a, Lc.s, nullptr, 0); break;
            case 4: launch_sweep<D, 4>(ctx, a, Lc.s, nullptr, 0); break;
            default: launch_sweep<D, 2>(ctx, a, Lc.s, nullptr, 0); break;
        }
        Lc.post(GMG_K_SWEEP, frac * (dm.lbytes[l].sweep[c] + (Wout ? dm.lbytes[l].sweep_out[c] : 0.0)));
        return;
    }
    SweepArgs a{b0, b1, ctx->opt.gamma - 1.0, L.rec, L.ecell, L.deg_int, L.sinfo, L.sJe, L.sRe, rhs, Wout, zlo, zhi};
    if (a.cend <= a.cbeg) return;
    Lc.pre(GMG_K_SWEEP);
    if (ctx->pipe) {
        PipeLayout pl{dm.lbytes[l].max_pipe};
        const size_t smem = (size_t)kPW * pl.warp() * sizeof(double);
        const int nb = (a.cend - a.cbeg + kPB - 1) / kPB;
        int per_sm = 0, nsm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sweep_pipe<D>, kPW * 32, smem);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->opt.device);
        const int grid = std::max(1, std::min((nb + kPW - 1) / kPW, nsm * std::max(per_sm, 1)));
        k_sweep_pipe<D><<<grid, kPW * 32, smem, Lc.s>>>(a, pl);
        Lc.post(GMG_K_SWEEP, dm.lbytes[l].sweep[c] + (Wout ? dm.lbytes[l].sweep_out[c] : 0.0));
        return;
    }
    if (ctx->spsweep) {
        const int64_t g0 = H.sp_off[c], ng = H.sp_off[c + 1] - g0 - 1;
        klaunch(ctx, k_sweep_sp<D>, dim3((unsigned)ng), dim3(kSpT), Lc.s, a, L.spcell + g0);
        Lc.post(GMG_K_SWEEP, dm.lbytes[l].sweep[c] + (Wout ? dm.lbytes[l].sweep_out[c] : 0.0));
        return;
    }
    if (ctx->wsweep) {
        const int W = ctx->wsweep, ms = dm.lbytes[l].max_ws;
        const size_t smem = (size_t)W * ms * (kRecS + kSlotRec) * sizeof(double);
        const int groups = (a.cend - a.cbeg + 31) / 32;
        const dim3 g((groups + W - 1) / W), b(W * 32);
        if (W == 1) k_sweep_ws<D, 1><<<g, b, smem, Lc.s>>>(a, ms);
        else if (W == 4) k_sweep_ws<D, 4><<<g, b, smem, Lc.s>>>(a, ms);
        else k_sweep_ws<D, 2><<<g, b, smem, Lc.s>>>(a, ms);
        Lc.post(GMG_K_SWEEP, dm.lbytes[l].sweep[c] + (Wout ? dm.lbytes[l].sweep_out[c] : 0.0));
        return;
    }
    const void *win = ctx->l2_window ? (const void *)L.rec : nullptr;
    const size_t rec_bytes = (size_t)L.n_loc * kRecStride * sizeof(double);
    const size_t wb = ctx->l2_window ? std::min<size_t>(ctx->l2_full ? ctx->l2_maxw : ctx->l2_window, rec_bytes) : 0;
    // small color blocks are latency bound (one partial wave, each lane walks
    // its slots one dependent gather after the other): spread the slots over
    // more lanes while the whole block still fits in one resident wave
    int lpc = (l < 8 && ctx->lpc_level[l] > 0) ? ctx->lpc_level[l] : ctx->lpc;
    if (ctx->adapt_lpc && ctx->sweep_grid_cap > 0) {
        const int64_t wave = (int64_t)ctx->sweep_grid_cap * 256, cells = a.cend - a.cbeg;
        while (lpc < 16 && cells * lpc * 2 <= wave) lpc *= 2;
    }
    switch (lpc) {
        case 1: launch_sweep<D, 1>(ctx, a, Lc.s, win, wb); break;
        case 4: launch_sweep<D, 4>(ctx, a, Lc.s, win, wb); break;
        case 8: launch_sweep<D, 8>(ctx, a, Lc.s, win, wb); break;
        case 16: launch_sweep<D, 16>(ctx, a, Lc.s, win, wb); break;
        default: launch_sweep<D, 2>(ctx, a, Lc.s, win, wb); break;
    }
    Lc.post(GMG_K_SWEEP, dm.lbytes[l].sweep[c] + (Wout ? dm.lbytes[l].sweep_out[c] : 0.0));
}

// one color phase with the fused P2P halo on every domain (an empty phase,
// c < 0, is a pure synchronisation point that advances the phase count)
template <int D>
void enqueue_p2p_phase(Launcher &Lc, int l, int c, bool last, bool ff, std::function<const double *(DevLevel &)> rhs,
                       std::function<double *(DevLevel &)> wout)
{
    gmg_ctx *ctx = Lc.ctx;
    for (Domain &dm : ctx->dom) {
        DevLevel &L = dm.dv[l];
        const DomLevel &H = dm.lv[l];
        const int b0 = c < 0 ? 0 : (int)H.blk[c], b1 = c < 0 ? 0 : (int)H.blk[c + 1];
        const bool z = c >= 0 && ff && ctx->skip_zero;
        SweepArgs a{b0, b1, ctx->opt.gamma - 1.0, L.rec, L.ecell, L.deg_int, L.sinfo, L.sJe, L.sRe, rhs(L),
                    last ? wout(L) : nullptr, z ? (int)H.blk[c + 1] : 0, z ? (int)H.n_own : 0};
        P2PArgs p{L.p2p_off, L.p2p_k, L.p2p_g, L.peer_rec, L.npeer, L.p2p_wait, L.p2p_sig, L.p2p_flags, L.p2p_ctl};
        int lpc = ctx->lpc;
        const int64_t cells = b1 - b0;
        if (ctx->adapt_lpc && ctx->sweep_grid_cap > 0)
            while (lpc < 16 && cells * lpc * 2 <= (int64_t)ctx->sweep_grid_cap * 256) lpc *= 2;
        int nb = nblk(cells * lpc);
        if (ctx->sweep_grid_cap > 0) nb = std::min(nb, ctx->sweep_grid_cap);
        const dim3 g(std::max(nb, 1)), b(256);
        Lc.pre(GMG_K_SWEEP);
        switch (lpc) {
            case 1: k_sweep_p2p<D, 1><<<g, b, 0, Lc.s>>>(a, p); break;
            case 4: k_sweep_p2p<D, 4><<<g, b, 0, Lc.s>>>(a, p); break;
            case 8: k_sweep_p2p<D, 8><<<g, b, 0, Lc.s>>>(a, p); break;
            case 16: k_sweep_p2p<D, 16><<<g, b, 0, Lc.s>>>(a, p); break;
            default: k_sweep_p2p<D, 2><<<g, b, 0, Lc.s>>>(a, p); break;
        }
        Lc.post(GMG_K_SWEEP, c < 0 ? 0.0 : dm.lbytes[l].sweep[c] + (last ? dm.lbytes[l].sweep_out[c] : 0.0));
    }
}

// n_sweeps x (forward colors 1..Nc, backward Nc..1), Algorithm 2;
// after every color its increments go to the ranks/domains that ghost them.
// The record's W_lin is the linearisation state; the last backward pass also
// writes W = W_lin + dW (rhs/Wout select the domain's arrays).
template <int D>
void enqueue_sweeps(Launcher &Lc, int l, int n_sweeps, std::function<const double *(DevLevel &)> rhs,
                    std::function<double *(DevLevel &)> wout)
{
    gmg_ctx *ctx = Lc.ctx;
    const int nc = ctx->lv[l].ncolor;
    struct Ph { int c; bool last; bool ff; };
    std::vector<Ph> seq;
    // Algorithm 2's phase list.  A color phase that directly follows a phase
    // of the SAME color (the turn of every forward -> backward and backward ->
    // forward pass: c_N then c_N, c_1 then c_1) is idempotent: a cell's update
    // reads only other-colored neighbours, none of which changed in between,
    // and never its own dW -- so it recomputes bit-identical values and is
    // dropped (its W = W_lin + dW write, if any, moves to the kept phase).
    // Exact, not an approximation: the oracle runs every phase.
    for (int s = 0; s < n_sweeps; ++s)
        for (int half = 0; half < 2; ++half)
            for (int cc = 0; cc < nc; ++cc) {
                const Ph ph{half == 0 ? cc : nc - 1 - cc, (s == n_sweeps - 1) && half == 1, s == 0 && half == 0};
                if (ctx->skip_repeat && !seq.empty() && seq.back().c == ph.c) seq.back().last |= ph.last;
                else seq.push_back(ph);
            }
    // fused P2P halo: increments go to the ghosts from the sweep epilogue; a
    // synchronisation phase before (the ghosts' local zeroing is done) and
    // after (the peers' last increments have landed) the step
    if (ctx->p2p && ctx->p2p_ready && ctx->nparts > 1) {
        enqueue_p2p_phase<D>(Lc, l, -1, false, false, rhs, wout);
        for (const Ph &ph : seq) enqueue_p2p_phase<D>(Lc, l, ph.c, ph.last, ph.ff, rhs, wout);
        enqueue_p2p_phase<D>(Lc, l, -1, false, false, rhs, wout);
        return;
    }
    // dependency-driven persistent sweep: one launch for the whole smoothing step
    if (ctx->flow && ctx->flow_grid > 0 && ctx->nparts == 1 && ctx->dom.size() == 1 && ctx->dom[0].dv[l].nchunk > 0 &&
        (int)seq.size() <= kFlowMaxPh && !ctx->pipe && !ctx->spsweep && !ctx->wsweep) {
        Domain &dm = ctx->dom[0];
        DevLevel &L = dm.dv[l];
        FlowArgs f{};
        f.nph = (int)seq.size();
        f.K = L.nchunk;
        f.n_own = L.n;
        f.seg = L.seg;
        f.cnoff = L.cnoff;
        f.cnidx = L.cnidx;
        f.prog = L.prog;
        f.err = ctx->d_flag + 2;
        double bytes = 0;
        for (size_t k = 0; k < seq.size(); ++k) {
            f.ph[k] = (unsigned short)(seq[k].c | (seq[k].last ? 1 << 8 : 0) | (seq[k].ff && ctx->skip_zero ? 1 << 9 : 0));
            bytes += dm.lbytes[l].sweep[seq[k].c] + (seq[k].last ? dm.lbytes[l].sweep_out[seq[k].c] : 0.0);
        }
        SweepArgs a{0, 0, ctx->opt.gamma - 1.0, L.rec, L.ecell, L.deg_int, L.sinfo, L.sJe, L.sRe, rhs(L), wout(L), 0, 0};
        cudaMemsetAsync(L.prog, 0, sizeof(int) * L.nchunk, Lc.s);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(std::min(ctx->flow_grid, L.nchunk));
        cfg.blockDim = dim3(256);
        cfg.stream = Lc.s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (ctx->flow == 2) cfg.gridDim = dim3(std::min(ctx->flow_grid, (L.nchunk + 7) / 8));
        Lc.pre(GMG_K_SWEEP);
        if (ctx->flow == 2) cudaLaunchKernelEx(&cfg, k_sweep_flow_w<D>, a, f);
        else cudaLaunchKernelEx(&cfg, k_sweep_flow<D>, a, f);
        Lc.post(GMG_K_SWEEP, bytes);
        return;
    }
    const bool fuse = ctx->tail_cells > 0 && ctx->nparts == 1 && ctx->dom.size() == 1;
    const bool tailc = ctx->tailc && !fuse && ctx->tailc_grid > 0 && ctx->nparts == 1 && ctx->dom.size() == 1 &&
                       ctx->sweep_grid_cap > 0 && !ctx->pipe && !ctx->spsweep && !ctx->wsweep;
    const bool overlap = (ctx->overlap < 0 ? ctx->opt.nranks > 1 : ctx->overlap != 0) && ctx->nparts > 1 && ctx->side && !ctx->pipe && !ctx->spsweep && !ctx->wsweep;
    for (size_t k = 0; k < seq.size();) {
        if (fuse) {
            // a run of >= 2 consecutive tiny color phases -> one single-CTA launch
            Domain &dm = ctx->dom[0];
            const DomLevel &H = dm.lv[l];
            auto tiny = [&](size_t t) {
                return t < seq.size() && H.blk[seq[t].c + 1] - H.blk[seq[t].c] <= ctx->tail_cells;
            };
            size_t r = k;
            while (tiny(r) && r - k < (size_t)kTailMaxPh) ++r;
            if (r - k >= 2) {
                DevLevel &L = dm.dv[l];
                TailArgs t{};
                t.nph = (int)(r - k);
                for (size_t p = k; p < r; ++p) {
                    t.cbeg[p - k] = (int)H.blk[seq[p].c];
                    t.cend[p - k] = (int)H.blk[seq[p].c + 1];
                    t.wout[p - k] = seq[p].last ? 1 : 0;
                }
                t.a = SweepArgs{0, 0, ctx->opt.gamma - 1.0, L.rec, L.ecell, L.deg_int, L.sinfo, L.sJe, L.sRe, rhs(L), wout(L)};
                double bytes = 0;
                for (size_t p = k; p < r; ++p)
                    bytes += dm.lbytes[l].sweep[seq[p].c] + (seq[p].last ? dm.lbytes[l].sweep_out[seq[p].c] : 0.0);
                Lc.pre(GMG_K_SWEEP);
                klaunch(ctx, k_sweep_tail<D>, dim3(1), dim3(kTailT), Lc.s, t);
                Lc.post(GMG_K_SWEEP, bytes);
                k = r;
                continue;
            }
        }
        if (tailc) {
            // a run of >= 2 consecutive small phases (each fits one resident wave at 2 lanes per
            // cell) -> one cooperative launch, grid barriers between the phases
            Domain &dm = ctx->dom[0];
            const DomLevel &H = dm.lv[l];
            const int64_t small = ctx->tailc_cells > 0 ? ctx->tailc_cells : (int64_t)ctx->sweep_grid_cap * 256 / 2;
            auto is_small = [&](size_t t) { return t < seq.size() && H.blk[seq[t].c + 1] - H.blk[seq[t].c] <= small; };
            size_t r = k;
            int64_t mx = 0;
            while (is_small(r) && r - k < (size_t)kTailMaxPh) { mx = std::max<int64_t>(mx, H.blk[seq[r].c + 1] - H.blk[seq[r].c]); ++r; }
            if (r - k >= 2) {
                DevLevel &L = dm.dv[l];
                TailArgs t{};
                t.nph = (int)(r - k);
                double bytes = 0;
                for (size_t p = k; p < r; ++p) {
                    t.cbeg[p - k] = (int)H.blk[seq[p].c];
                    t.cend[p - k] = (int)H.blk[seq[p].c + 1];
                    t.wout[p - k] = seq[p].last ? 1 : 0;
                    bytes += dm.lbytes[l].sweep[seq[p].c] + (seq[p].last ? dm.lbytes[l].sweep_out[seq[p].c] : 0.0);
                }
                t.a = SweepArgs{0, 0, ctx->opt.gamma - 1.0, L.rec, L.ecell, L.deg_int, L.sinfo, L.sJe, L.sRe, rhs(L), wout(L)};
                const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ctx->tailc_grid, (mx * 16 + 255) / 256));
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(grid);
                cfg.blockDim = dim3(256);
                cfg.stream = Lc.s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeCooperative;
                at[0].val.cooperative = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                int *bar = ctx->d_bar;
                Lc.pre(GMG_K_SWEEP);
                cudaLaunchKernelEx(&cfg, k_sweep_tailc<D>, t, bar);
                Lc.post(GMG_K_SWEEP, bytes);
                k = r;
                continue;
            }
        }
        const int c = seq[k].c;
        if (overlap) {
            // boundary cells of color c first; their increments travel on the
            // side stream while the interior cells of c (no ghost neighbours)
            // are swept; the next color waits for the ghosts (fork / join)
            for (Domain &dm : ctx->dom)
                enqueue_sweep_color<D>(Lc, dm, l, c, rhs(dm.dv[l]), seq[k].last ? wout(dm.dv[l]) : nullptr, 1, seq[k].ff);
            cudaEventRecord(ctx->ev_fork, Lc.s);
            cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0);
            Launcher Ls{ctx, ctx->side};
            enqueue_exchange<D>(Ls, l, EX_DW, c);
            cudaEventRecord(ctx->ev_join, ctx->side);
            for (Domain &dm : ctx->dom)
                enqueue_sweep_color<D>(Lc, dm, l, c, rhs(dm.dv[l]), seq[k].last ? wout(dm.dv[l]) : nullptr, 2, seq[k].ff);
            cudaStreamWaitEvent(Lc.s, ctx->ev_join, 0);
        } else {
            for (Domain &dm : ctx->dom)
                enqueue_sweep_color<D>(Lc, dm, l, c, rhs(dm.dv[l]), seq[k].last ? wout(dm.dv[l]) : nullptr, 0, seq[k].ff);
            enqueue_exchange<D>(Lc, l, EX_DW, c);
        }
        ++k;
    }
}

template <int D>
void enqueue_restrict(Launcher &Lc, Domain &dm, int l)
{
    DevLevel &C = dm.dv[l];
    DevLevel &Fn = dm.dv[l - 1];
    Lc.pre(GMG_K_RESTRICT);
    klaunch(Lc.ctx, k_restrict<D>, dim3(nblk(C.n)), dim3(256), Lc.s, C, Fn, Fn.W, Fn.Rt);
    Lc.post(GMG_K_RESTRICT, dm.lbytes[l].restrict_);
}

// NEXT-1 halo (partitioned runs): owned -> ghost copies of a level-0 per-cell
// array of ncomp doubles (slopes, polynomials, Dt), all colors at once
void enqueue_exchange_ho(Launcher &Lc, double *HoDev::*arr, int ncomp)
{
    gmg_ctx *ctx = Lc.ctx;
    if (ctx->nparts <= 1) return;
    for (Domain &dm : ctx->dom) {
        const DomLevel &H = dm.lv[0];
        DevLevel &L = dm.dv[0];
        const int64_t s1 = H.send_off.back();
        if (s1 > 0) {
            Lc.pre(GMG_K_NORM);
            klaunch(ctx, k_pack, dim3(nblk(s1)), dim3(256), Lc.s, (int)s1, L.send_idx, (const double *)(L.ho.*arr), ncomp, 0,
                    ncomp, dm.ho.sendbuf);
            Lc.post(GMG_K_NORM, (double)s1 * ncomp * 16);
        }
    }
    if (ctx->opt.nranks > 1) {
        Domain &dm = ctx->dom[0];
        const DomLevel &H = dm.lv[0];
        const int np = (int)H.peers.size(), ng = (int)H.send_off.size() - 1;
        nccl().GroupStart();
        for (int g = 0; g < ng; ++g) {
            const int peer = H.peers[g % np];
            const int64_t sc = H.send_off[g + 1] - H.send_off[g], rc = H.recv_off[g + 1] - H.recv_off[g];
            if (sc) nccl().Send(dm.ho.sendbuf + H.send_off[g] * ncomp, sc * ncomp, ncclDouble, peer, (ncclComm_t)ctx->nccl_comm, Lc.s);
            if (rc) nccl().Recv(dm.ho.recvbuf + H.recv_off[g] * ncomp, rc * ncomp, ncclDouble, peer, (ncclComm_t)ctx->nccl_comm, Lc.s);
        }
        nccl().GroupEnd();
    } else {
        for (Domain &dm : ctx->dom) {
            const DomLevel &H = dm.lv[0];
            const int np = (int)H.peers.size(), ng = (int)H.send_off.size() - 1;
            for (int g = 0; g < ng; ++g) {
                const int64_t sc = H.send_off[g + 1] - H.send_off[g];
                if (!sc) continue;
                Domain &dp = ctx->dom[H.peers[g % np]];
                const DomLevel &Hp = dp.lv[0];
                const int npp = (int)Hp.peers.size();
                const int kk = (int)(std::lower_bound(Hp.peers.begin(), Hp.peers.end(), dm.rank) - Hp.peers.begin());
                const int gp = (g / np) * npp + kk;
                cudaMemcpyAsync(dp.ho.recvbuf + Hp.recv_off[gp] * ncomp, dm.ho.sendbuf + H.send_off[g] * ncomp,
                                sizeof(double) * sc * ncomp, cudaMemcpyDeviceToDevice, Lc.s);
            }
        }
    }
    for (Domain &dm : ctx->dom) {
        const DomLevel &H = dm.lv[0];
        DevLevel &L = dm.dv[0];
        const int64_t r1 = H.recv_off.back();
        if (r1 > 0) {
            Lc.pre(GMG_K_NORM);
            klaunch(ctx, k_unpack, dim3(nblk(r1)), dim3(256), Lc.s, (int)r1, L.recv_idx, (const double *)dm.ho.recvbuf,
                    L.ho.*arr, ncomp, 0, ncomp, 0, 0);
            Lc.post(GMG_K_NORM, (double)r1 * ncomp * 16);
        }
    }
    ctx->exchanges++;
}

// NEXT-1: one evaluation of the third-order CGKS operator on the fine level
// (ho.cu): S r, reconstruction, Gauss-point BGK fluxes, gather(mode).  Every
// domain; on partitioned runs the ghosts' W, slopes, then polynomials and Dt
// come by halo exchange.  Rout / aout: per-domain outputs (ABI), or null.
template <int D>
void enqueue_ho_eval(Launcher &Lc, int mode, double *DevLevel::*Rout = nullptr, double *DevLevel::*aout = nullptr,
                     bool recon_only = false)
{
    gmg_ctx *ctx = Lc.ctx;
    const Phys ph = phys(ctx);
    const BCs bc = bcs(ctx);
    constexpr int NV = D + 2, NC = 1 + D + D * (D + 1) / 2;
    enqueue_exchange<D>(Lc, 0, EX_W, -1);
    enqueue_exchange_ho(Lc, &HoDev::G_, NV * D);
    for (Domain &dm : ctx->dom) {
        DevLevel &L = dm.dv[0];
        Lc.pre(GMG_K_HO_RECON);
        ho_launch(0, L, L.ho, ph, bc, ctx->opt, 0, nullptr, nullptr, Lc.s);
        Lc.post(GMG_K_HO_RECON, dm.ho.bytes_sr);
        Lc.pre(GMG_K_HO_RECON);
        ho_launch(1, L, L.ho, ph, bc, ctx->opt, 0, nullptr, nullptr, Lc.s);
        Lc.post(GMG_K_HO_RECON, dm.ho.bytes_recon);
    }
    if (recon_only) return;
    enqueue_exchange_ho(Lc, &HoDev::poly, NV * NC);
    enqueue_exchange_ho(Lc, &HoDev::dt, 1);
    for (size_t di = 0; di < ctx->dom.size(); ++di) {
        Domain &dm = ctx->dom[di];
        DevLevel &L = dm.dv[0];
        Lc.pre(GMG_K_HO_FLUX);
        ho_launch(2, L, L.ho, ph, bc, ctx->opt, 0, nullptr, nullptr, Lc.s);
        Lc.post(GMG_K_HO_FLUX, dm.ho.bytes_flux);
        Lc.pre(GMG_K_GATHER);
        ho_launch(3, L, L.ho, ph, bc, ctx->opt, mode, Rout ? L.*Rout : nullptr, aout ? L.*aout : nullptr, Lc.s);
        Lc.post(GMG_K_GATHER, dm.ho.bytes_gather);
        if (mode & HO_NORM) {
            Lc.pre(GMG_K_NORM);
            klaunch(Lc.ctx, k_norm_sum, dim3(1), dim3(256), Lc.s, L.partial, nblk(L.n), L.nv, ctx->d_sumsq + di * L.nv);
            Lc.post(GMG_K_NORM, (double)nblk(L.n) * L.nv * 8);
        }
    }
}

// O8 -- one V-cycle, all on the device
template <int D>
void enqueue_vcycle(Launcher &Lc)
{
    gmg_ctx *ctx = Lc.ctx;
    const int nl = (int)ctx->lv.size();
    const bool df0 = ctx->opt.df_mode == 0 || ctx->opt.df_mode == 3;   // DF helper alpha (prolongation)
    auto &doms = ctx->dom;
    if (ctx->opt.fine_operator == 1) {
        // NEXT-1, reading C14: CGKS3 evaluation at (W, G, alpha) -> history, Eq.(smo), slopes, DF;
        // a second evaluation at the updated state -> restricted residual and DF
        enqueue_ho_eval<D>(Lc, HO_NORM | HO_UPDATE);
        enqueue_norm_hist(Lc);
        if (nl == 1) return;
        enqueue_ho_eval<D>(Lc, HO_RT);
    } else {
    // 1-2. fine residual at the cycle start (history entry) + fine pre-smoothing
    enqueue_exchange<D>(Lc, 0, EX_W, -1);
    for (Domain &dm : doms)
        enqueue_face<D>(Lc, dm, 0, dm.dv[0].W, true, false, ctx->opt.fine_smoother == 1 && df0, ctx->opt.fine_smoother == 1);
    if (ctx->opt.fine_smoother == 0) {
        for (size_t d = 0; d < doms.size(); ++d)
            enqueue_gather<D>(Lc, doms[d], (int)d, 0, G_FLUX | G_NORM | G_EXPLICIT, doms[d].dv[0].W);   // Eq.(smo), A9
        enqueue_norm_hist(Lc);
        enqueue_exchange<D>(Lc, 0, EX_W, -1);
    } else {
        for (size_t d = 0; d < doms.size(); ++d)
            enqueue_gather<D>(Lc, doms[d], (int)d, 0,
                              G_FLUX | G_NORM | G_WRITE_RT | G_PREPARE | G_ZERO_DW | G_COPY_W | (df0 ? G_ALPHA : 0),
                              nullptr);
        enqueue_norm_hist(Lc);
        enqueue_ghost_wlin<D>(Lc, 0);
        enqueue_sweeps<D>(Lc, 0, ctx->opt.n_sweeps, [](DevLevel &L) { return (const double *)L.Rt; },
                          [](DevLevel &L) { return L.W; });
        enqueue_ghost_w<D>(Lc, 0);
    }
    if (nl == 1) return;
    // 3. residual at the smoothed state (A10) -> restricted
    for (size_t d = 0; d < doms.size(); ++d) {
        enqueue_face<D>(Lc, doms[d], 0, doms[d].dv[0].W, true, false, df0);
        enqueue_gather<D>(Lc, doms[d], (int)d, 0, G_FLUX | G_WRITE_RT | (df0 ? G_ALPHA : 0), nullptr);
    }
    }
    // 4. coarse levels
    for (int l = 1; l < nl; ++l) {
        const bool last = (l == nl - 1);
        for (Domain &dm : doms) enqueue_restrict<D>(Lc, dm, l);                // W0, Res*, alpha, dW = 0
        enqueue_exchange<D>(Lc, l, EX_WLIN, -1);                                // ghosts' W0, dW = 0
        for (size_t d = 0; d < doms.size(); ++d) {
            enqueue_face<D>(Lc, doms[d], l, doms[d].dv[l].rec, !last, true, false, true);   // R(W0) only if F is needed later
            enqueue_gather<D>(Lc, doms[d], (int)d, l, (last ? 0 : (G_FLUX | G_SET_F)) | G_PREPARE, nullptr);
        }
        enqueue_sweeps<D>(Lc, l, ctx->opt.n_sweeps, [](DevLevel &L) { return (const double *)L.Rs; },
                          [](DevLevel &L) { return L.W; });                      // RHS = Res* (A8)
        if (!last) {
            enqueue_ghost_w<D>(Lc, l);
            for (size_t d = 0; d < doms.size(); ++d) {
                enqueue_face<D>(Lc, doms[d], l, doms[d].dv[l].W, true, false);
                enqueue_gather<D>(Lc, doms[d], (int)d, l, G_FLUX | G_WRITE_RT | G_ADD_F, nullptr);   // Rt = R(W) + F (A11)
            }
        }
    }
    // 5. DF-limited prolongation 2 -> 1 -> 0 (fused; rank-local)
    for (Domain &dm : doms) {
        Lc.pre(GMG_K_PROLONG);
        klaunch(Lc.ctx, k_prolong<D>, dim3(nblk(dm.dv[0].n)), dim3(256), Lc.s, dm.dv[0], dm.dv[1], nl >= 3 ? dm.dv[2] : dm.dv[1], nl);
        Lc.post(GMG_K_PROLONG, dm.lbytes[0].prolong);
    }
}

// final history entry: residual at the end state
template <int D>
void enqueue_final_norm(Launcher &Lc)
{
    gmg_ctx *ctx = Lc.ctx;
    if (ctx->opt.fine_operator == 1) {
        enqueue_ho_eval<D>(Lc, HO_NORM);
        enqueue_norm_hist(Lc);
        return;
    }
    enqueue_exchange<D>(Lc, 0, EX_W, -1);
    for (size_t d = 0; d < ctx->dom.size(); ++d) {
        enqueue_face<D>(Lc, ctx->dom[d], 0, ctx->dom[d].dv[0].W, true, false);
        enqueue_gather<D>(Lc, ctx->dom[d], (int)d, 0, G_FLUX | G_NORM, nullptr);
    }
    enqueue_norm_hist(Lc);
}

gmg_status check_ready(gmg_ctx *ctx, bool need_state = true)
{
    if (!ctx->built) { ctx->err = "hierarchy not built"; return GMG_ESTATE; }
    if (!ctx->ws_ready) { ctx->err = "workspace not set"; return GMG_ESTATE; }
    if (need_state && !ctx->state_set) { ctx->err = "state not set"; return GMG_ESTATE; }
    return GMG_OK;
}

// natural SoA [ncomp][N] (host or device) -> every domain's local cells
// (owned + ghosts), AoS (stride, offset)
gmg_status put_natural(gmg_ctx *ctx, int l, const double *src, int ncomp, std::function<double *(DevLevel &)> dst,
                       bool with_ghosts, int stride = -1, int offset = 0)
{
    const int64_t N = ctx->lv[l].n;
    if (stride < 0) stride = ncomp;
    CK(cudaMemcpyAsync(ctx->d_stage, src, sizeof(double) * ncomp * N, cudaMemcpyDefault, ctx->stream));
    for (Domain &dm : ctx->dom) {
        DevLevel &L = dm.dv[l];
        const int cnt = with_ghosts ? L.n_loc : L.n;
        k_to_internal<<<nblk(cnt), 256, 0, ctx->stream>>>(cnt, (int)N, ncomp, L.perm, ctx->d_stage, dst(L), stride, offset);
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));   // caller's host buffer may be released on return
    return GMG_OK;
}

// every domain's owned cells -> natural SoA; with nranks > 1 only this rank's
// owned entries of dst are written
gmg_status get_natural(gmg_ctx *ctx, int l, std::function<const double *(DevLevel &)> src, int ncomp, double *dst,
                       int stride = -1, int offset = 0)
{
    const int64_t N = ctx->lv[l].n;
    if (stride < 0) stride = ncomp;
    if (ctx->opt.nranks > 1)
        CK(cudaMemcpyAsync(ctx->d_stage, dst, sizeof(double) * ncomp * N, cudaMemcpyDefault, ctx->stream));
    for (Domain &dm : ctx->dom) {
        DevLevel &L = dm.dv[l];
        k_to_natural<<<nblk(L.n), 256, 0, ctx->stream>>>(L.n, (int)N, ncomp, L.perm, src(L), ctx->d_stage, stride, offset);
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(dst, ctx->d_stage, sizeof(double) * ncomp * N, cudaMemcpyDefault, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return GMG_OK;
}

// ----------------------------------------------------------------- workspace
struct Bump {
    char *base;
    size_t off = 0;
    template <class T>
    T *take(size_t count)
    {
        off = (off + 255) & ~(size_t)255;
        T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
        off += count * sizeof(T) + 16;
        return p;
    }
};

void carve(gmg_ctx *ctx, Bump &b)
{
    const int d = ctx->opt.dim, nv = d + 2;
    const int nl = (int)ctx->lv.size();
    int64_t nmax = 0;
    for (const HostLevel &G : ctx->lv) nmax = std::max(nmax, G.n);
    for (Domain &dm : ctx->dom) {
        dm.dv.assign(nl, DevLevel{});
        int *flags = b.take<int>(std::max(ctx->nparts, 1));   // P2P phase counts published by the peers
        int *ctl = b.take<int>(4);
        for (int l = 0; l < nl; ++l) {
            const HostLevel &G = ctx->lv[l];
            const DomLevel &H = dm.lv[l];
            DevLevel &L = dm.dv[l];
            const int64_t n = H.n_own, nloc = H.n_loc, nf = H.nf;
            L.dim = d; L.nv = nv; L.ncolor = G.ncolor;
            L.p2p_flags = flags;
            L.p2p_ctl = ctl;
            L.n = (int)n; L.n_loc = (int)nloc; L.nf = (int)nf;
            L.fl = b.take<int>(nf); L.fr = b.take<int>(nf);
            L.fA = b.take<double>((size_t)d * nf); L.fM = b.take<int8_t>(nf);
            L.Frec = b.take<double>((size_t)kFaceRec * nf);
            L.vol = b.take<double>(n);
            L.W = b.take<double>((size_t)nv * nloc); L.Rt = b.take<double>((size_t)nv * n);
            L.rec = b.take<double>((size_t)kRecStride * nloc);
            L.tmp = b.take<double>(n);
            L.Rs = b.take<double>((size_t)nv * n); L.F = b.take<double>((size_t)nv * n);
            L.alpha = b.take<double>(n); L.sigma = b.take<double>(n);
            L.deg_int = b.take<uint8_t>(n); L.deg_all = b.take<uint8_t>(n);
            L.gbase = b.take<int>(n);
            L.gface = b.take<int>(H.ng_entries);
            L.ecell = b.take<int>(n); L.estride = b.take<int>(n);
            L.spcell = b.take<int>(H.sp_cell.size());
            L.sinfo = b.take<int2>(n);
            L.fslot = b.take<int2>(nf);
            L.npeer = (int)H.peers.size();
            L.p2p_off = b.take<int>(H.p2p_off.size());
            L.p2p_k = b.take<int>(H.p2p_k.size());
            L.p2p_g = b.take<int>(H.p2p_g.size());
            L.peer_rec = b.take<double *>(H.peers.size());
            L.p2p_sig = b.take<int *>(H.peers.size());
            L.p2p_wait = b.take<int>(H.peers.size());
            L.nchunk = H.nchunk;
            L.seg = b.take<int>(H.seg.size());
            L.cnoff = b.take<int>(H.cnoff.size());
            L.cnidx = b.take<int>(H.cnidx.size());
            L.prog = b.take<int>(H.nchunk);
            L.ginfo = b.take<int4>(n);
            L.sJe = b.take<int>(H.sJe.size());
            L.sRe = b.take<double>(H.sRe.size());
            L.perm = b.take<int>(nloc);
            L.child = l > 0 ? b.take<int>(2 * n) : nullptr;
            L.parent = l + 1 < nl ? b.take<int>(n) : nullptr;
            L.partial = b.take<double>((size_t)nblk(n) * nv);
            L.n_send = (int)H.send_idx.size();
            L.n_recv = (int)H.recv_idx.size();
            L.send_idx = b.take<int>(L.n_send);
            L.recv_idx = b.take<int>(L.n_recv);
            L.sendbuf = b.take<double>((size_t)L.n_send * nv);
            L.recvbuf = b.take<double>((size_t)L.n_recv * nv);
        }
    }
    // natural-order staging: nv components; with the NEXT-1 geometry also the slopes (nv d) and the
    // polynomials (nv (1 + d + d(d+1)/2)) of gmg_set/get_ho_state, gmg_ho_residual, gmg_ho_recon
    const int stage_comp = ctx->ho ? nv * (1 + d + d * (d + 1) / 2) : nv;
    ctx->d_stage = b.take<double>((size_t)stage_comp * nmax);
    for (int k = 0; k < 2; ++k) {               // pipelined host I/O staging (fine level, natural order)
        ctx->stage_in[k] = b.take<double>((size_t)nv * ctx->lv[0].n);
        ctx->stage_out[k] = b.take<double>((size_t)nv * ctx->lv[0].n);
    }
    ctx->hist_cap = 4096;
    ctx->d_hist = b.take<double>((size_t)ctx->hist_cap * nv);
    ctx->d_flag = b.take<int>(4);
    ctx->d_bar = b.take<int>(2);
    ctx->d_emu = b.take<char>(sizeof(EmuDom) * kEmuMaxDom);
    ctx->d_emu_bar = b.take<int>(2 * kEmuMaxDom);
    ctx->d_sumsq = b.take<double>((size_t)std::max<size_t>(1, ctx->dom.size()) * nv);
    if (ctx->ho && ctx->ho->prepared) {                       // NEXT-1 (fine level)
        const HoHost &HH = *ctx->ho;
        for (Domain &dm : ctx->dom) {
            const HoLocal &H = dm.ho;
            HoDev &V = dm.dv[0].ho;
            const DomLevel &D0 = dm.lv[0];
            const int64_t n = D0.n_own, nl = D0.n_loc, nf = D0.nf;
            V.G = HH.G;
            V.nq = d * (d + 1) / 2;
            V.nk = d + V.nq;
            V.nc = 1 + V.nk;
            V.ctr = b.take<double>((size_t)nl * d);
            V.m2 = b.take<double>((size_t)nl * V.nq);
            V.gp = b.take<double>((size_t)nf * HH.G * d);
            V.gw = b.take<double>((size_t)nf * HH.G);
            V.hfoff = b.take<int>(n + 1);
            V.hface = b.take<int>(H.hface.size());
            V.hrec = b.take<double>(H.hrec.size());
            V.poff = b.take<int>(n + 1);
            V.P = b.take<double>(H.P.size());
            V.G_ = b.take<double>((size_t)nl * nv * d);
            V.alpha = b.take<double>(n);
            V.poly = b.take<double>((size_t)nl * nv * V.nc);
            V.flags = b.take<int>(n);
            V.sr = b.take<double>(nf);
            V.dt = b.take<double>(nl);
            V.frec = b.take<double>((size_t)nf * 12);
            V.Gout = b.take<double>((size_t)n * nv * d);
            dm.ho.sendbuf = b.take<double>(D0.send_idx.size() * (size_t)nv * V.nc);
            dm.ho.recvbuf = b.take<double>(D0.recv_idx.size() * (size_t)nv * V.nc);
        }
    }
}

void compute_bytes(gmg_ctx *ctx)
{
    const int d = ctx->opt.dim, nv = d + 2;
    const int nl = (int)ctx->lv.size();
    for (Domain &dm : ctx->dom) {
        dm.lbytes.assign(nl, LevelBytes{});
        for (int l = 0; l < nl; ++l) {
            const DomLevel &H = dm.lv[l];
            const int ncolor = ctx->lv[l].ncolor;
            LevelBytes &B = dm.lbytes[l];
            int64_t nint = 0;
            for (int64_t f = 0; f < H.nf; ++f) nint += H.fr[f] >= 0;
            const double nb = (double)(H.nf - nint);
            // face: cells' W (interior 2, boundary 1), A, l/r, M; writes S F, S r, alpha^M
            const double face_in = (double)nint * 2 * nv * 8 + nb * nv * 8 + (double)H.nf * (d * 8 + 8 + 1);
            B.face_flux = face_in + (double)H.nf * (nv * 8 + 16);
            B.face_prep = face_in + (double)H.nf * 8;
            // prep launches: fslot read + the (A outward | S r) slot record of each side that has one
            double nslot = 0;
            for (int32_t e : H.fslot) nslot += e >= 0;
            B.face_slots = (double)H.nf * 8 + nslot * kSlotRec * 8;
            // gather: per slot the face id + S F + S r + alpha^M; per cell bases/degrees + outputs
            double slots = 0;
            for (int64_t i = 0; i < H.n_own; ++i) slots += H.deg_all[i];
            B.gather = slots * (4 + nv * 8 + 16) + (double)H.n_own * (10 + 2 * nv * 8);
            // sweep (compulsory): own Rt, 1/D, alpha/2, dW write; neighbour-unique W, dW;
            // face data (A, S r) once per face + 4 B per slot
            B.sweep.assign(ncolor, 0.0);
            B.sweep_out.assign(ncolor, 0.0);
            for (int c = 0; c < ncolor; ++c) {
                double s = 0;
                for (int64_t i = H.blk[c]; i < H.blk[c + 1]; ++i)
                    s += (2 * nv * 8 + 16) + 2 * nv * 8 + H.deg_int[i] * ((d + 1) * 8 / 2.0 + 4);
                B.sweep[c] = s;
                B.sweep_out[c] = (double)(H.blk[c + 1] - H.blk[c]) * 2 * nv * 8;
            }
            B.restrict_ = l > 0 ? (double)dm.lv[l - 1].n_own * (2 * nv * 8 + 16) + (double)H.n_own * (3 * nv * 8 + 16) : 0;
            B.prolong = (double)H.n_own * (2 * nv * 8 + 8 + 4) + (nl > 1 ? (double)dm.lv[1].n_own * (nv * 8 + 12) : 0) +
                        (nl > 2 ? (double)dm.lv[2].n_own * nv * 8 : 0);
            B.update = (double)H.n_own * 3 * nv * 8;
            int mws = 1;
            for (int c = 0; c < ncolor; ++c)
                for (int64_t i0 = H.blk[c]; i0 < H.blk[c + 1]; i0 += kChunk) {
                    const int64_t i1 = std::min<int64_t>(i0 + kChunk, H.blk[c + 1]);
                    int s = 0;
                    for (int64_t i = i0; i < i1; ++i) s += H.deg_int[i];
                    mws = std::max(mws, s);
                }
            B.max_ws = mws;
            int mp = 1;
            for (int c = 0; c < ncolor; ++c)
                for (int64_t i0 = H.blk[c]; i0 < H.blk[c + 1]; i0 += kPB) {
                    const int64_t i1 = std::min<int64_t>(i0 + kPB, H.blk[c + 1]);
                    int s = 0;
                    for (int64_t i = i0; i < i1; ++i) s += H.deg_int[i];
                    mp = std::max(mp, s);
                }
            B.max_pipe = std::min(mp, 128);   // batch slots live in 4 registers per lane
        }
    }
}

template <int D>
void vcycle_dispatch(Launcher &Lc) { enqueue_vcycle<D>(Lc); }

}  // namespace

// =============================================================================
// ABI
// =============================================================================
extern "C" {

void gmg_default_options(gmg_options *o)
{
    std::memset(o, 0, sizeof(*o));
    o->dim = 3;
    o->gamma = 1.4;
    o->cfl_imp = 10.0;
    o->cfl_exp = 0.5;
    o->n_sweeps = 6;
    o->n_levels = 3;
    o->pre_smooth = 1;
    o->post_smooth = 0;
    o->skew_limit = 0.5;
    o->r_factor = 1.0;
    o->fine_smoother = 0;
    o->df_mode = 0;
    o->rank = 0;
    o->nranks = 1;
    o->nccl_id = nullptr;
    o->device = 0;
    o->stream = nullptr;
    o->local_domains = 1;
    o->setup_device = 0;
    o->beta = 0.5;
    o->fine_operator = 0;
    o->ho_c1 = 0.05;
    o->ho_c2 = 1.0;
    o->ho_gam0 = 0.95;
    o->ho_eps = 1e-14;
}

gmg_status gmg_create(const gmg_options *opt, gmg_ctx **out)
{
    if (!opt || !out) return GMG_EINVAL;
    *out = nullptr;
    if ((opt->dim != 2 && opt->dim != 3) || !(opt->gamma > 1.0) || !(opt->cfl_imp > 0) || !(opt->cfl_exp > 0) ||
        opt->n_sweeps < 1 || opt->n_levels < 1 || opt->n_levels > 3 || opt->pre_smooth != 1 || opt->post_smooth != 0 ||
        !(opt->r_factor >= 1.0) || opt->fine_smoother < 0 || opt->fine_smoother > 1 || opt->df_mode < 0 ||
        opt->fine_operator < 0 || opt->fine_operator > 1 ||
        (opt->fine_operator == 1 && (opt->fine_smoother != 0 || opt->df_mode != 0 || !(opt->ho_c1 > 0.0) ||
                                     !(opt->ho_c2 >= 0.0) || !(opt->ho_gam0 > 0.0 && opt->ho_gam0 <= 1.0) ||
                                     !(opt->ho_eps > 0.0))) ||
        opt->df_mode > 3 || (opt->df_mode == 3 && !(opt->beta >= 0.0 && opt->beta <= 1.0)) || opt->nranks < 1 ||
        opt->rank < 0 || opt->rank >= opt->nranks || opt->local_domains < 1 ||
        opt->local_domains > 64 || (opt->nranks > 1 && (opt->local_domains != 1 || !opt->nccl_id)) ||
        opt->setup_device < 0 || opt->setup_device > 1)
        return GMG_EINVAL;
    gmg_ctx *ctx = new (std::nothrow) gmg_ctx();
    if (!ctx) return GMG_ENOMEM;
    ctx->opt = *opt;
    ctx->stream = (cudaStream_t)opt->stream;
    ctx->nparts = std::max(opt->nranks, opt->local_domains);
    if (const char *e = std::getenv("GMG_LPC")) ctx->lpc = std::atoi(e);   // lanes per cell in the sweep
    if (const char *e = std::getenv("GMG_LPC_LEVELS")) {                     // per level: "2,2,4"
        int k = 0;
        for (const char *p = e; *p && k < 8; ++k) {
            ctx->lpc_level[k] = std::atoi(p);
            while (*p && *p != ',') ++p;
            if (*p == ',') ++p;
        }
    }
    if (const char *e = std::getenv("GMG_MINB")) ctx->minb = std::atoi(e); // min resident blocks (occupancy)
    // programmatic dependent launch between the V-cycle kernels: every kernel launched with the attribute
    // waits (griddepcontrol.wait) before touching its predecessor's outputs; the sweep phases load their
    // static slot indices before that wait, overlapping the previous phase's tail (v16: -3.5 % per
    // V-cycle).  GMG_PDL=0 disables
    ctx->pdl = 1;
    if (const char *e = std::getenv("GMG_PDL")) ctx->pdl = std::atoi(e);
    if (const char *e = std::getenv("GMG_WSWEEP")) ctx->wsweep = std::atoi(e);   // warp-staged sweep
    if (const char *e = std::getenv("GMG_SPSWEEP")) ctx->spsweep = std::atoi(e); // slot-parallel sweep
    if (const char *e = std::getenv("GMG_TAIL")) ctx->tail_cells = std::atoi(e);  // tiny-color fusion threshold
    if (const char *e = std::getenv("GMG_PIPE")) ctx->pipe = std::atoi(e);        // pipelined warp sweep
    if (const char *e = std::getenv("GMG_OVERLAP")) ctx->overlap = std::atoi(e);  // boundary-first exchange overlap
    if (const char *e = std::getenv("GMG_ALPC")) ctx->adapt_lpc = std::atoi(e);   // wider lanes for small colors
    if (const char *e = std::getenv("GMG_SKIP_REPEAT")) ctx->skip_repeat = std::atoi(e);   // drop idempotent phases
    if (const char *e = std::getenv("GMG_SKIP_ZERO")) ctx->skip_zero = std::atoi(e);       // skip +0 neighbour terms
    if (const char *e = std::getenv("GMG_FLOW")) ctx->flow = std::atoi(e);                 // dependency-driven sweep
    if (const char *e = std::getenv("GMG_P2P")) ctx->p2p = std::atoi(e);                   // fused P2P halo
    if (const char *e = std::getenv("GMG_TAILC")) ctx->tailc = std::atoi(e);               // cooperative small-phase runs
    if (const char *e = std::getenv("GMG_TAILC_CELLS")) ctx->tailc_cells = std::atoi(e);
    if (const char *e = std::getenv("GMG_CHUNK_ORDER")) ctx->chunk_order = std::atoi(e);   // (color, chunk, id) order
    if (const char *e = std::getenv("GMG_ORDER_CHUNK")) ctx->order_chunk = std::max(8, std::atoi(e));
    if (const char *e = std::getenv("GMG_FLOW_CHUNK")) ctx->flow_chunk = std::max(32, std::atoi(e));
    *out = ctx;
    return GMG_OK;
}

gmg_status gmg_load_mesh(gmg_ctx *ctx, int64_t n_cells, const double *vol, const double *centroid, int64_t n_faces,
                         const int64_t *left, const int64_t *right, const double *area_vec, const double *face_ctr,
                         const int8_t *n_gauss, int n_patches, const int32_t *patch_kind, const int32_t *part)
{
    if (!ctx) return GMG_EINVAL;
    if (n_cells < 1 || n_faces < 1 || !vol || !centroid || !left || !right || !area_vec || !face_ctr || !n_gauss ||
        n_patches < 0 || n_patches > 16 || (n_patches > 0 && !patch_kind) || n_cells >= INT32_MAX / 8 ||
        n_faces >= INT32_MAX / 8) {
        ctx->err = "gmg_load_mesh: bad arguments";
        return GMG_EINVAL;
    }
    if (ctx->nparts > 1) {
        if (!part) { ctx->err = "partitioned run needs part[]"; return GMG_EINVAL; }
        for (int64_t i = 0; i < n_cells; ++i)
            if (part[i] < 0 || part[i] >= ctx->nparts) { ctx->err = "part[] out of range"; return GMG_EINVAL; }
    }
    ctx->n_patches = n_patches;
    ctx->patch_kind.assign(patch_kind, patch_kind + n_patches);
    for (int k = 0; k < n_patches; ++k)
        if (patch_kind[k] < 0 || patch_kind[k] > 3) { ctx->err = "bad patch kind"; return GMG_EINVAL; }
    gmg_status st = load_mesh(ctx, n_cells, vol, centroid, n_faces, left, right, area_vec, face_ctr, n_gauss,
                              ctx->nparts > 1 ? part : nullptr);
    if (st != GMG_OK) return st;
    ctx->mesh_loaded = true;
    ctx->built = ctx->ws_ready = ctx->state_set = false;
    return GMG_OK;
}

gmg_status gmg_set_coloring(gmg_ctx *ctx, int level, const int32_t *color)
{
    if (!ctx) return GMG_EINVAL;
    if (!ctx->mesh_loaded || ctx->built) { ctx->err = "set_coloring must follow load_mesh and precede build"; return GMG_ESTATE; }
    if (level != 0) { ctx->err = "only the fine level accepts a user coloring"; return GMG_EINVAL; }
    if (!color) { ctx->user_color0.clear(); return GMG_OK; }
    std::vector<int32_t> c(color, color + ctx->lv[0].n);
    if (!validate_coloring(ctx->lv[0], c)) { ctx->err = "invalid coloring: face neighbours share a color or color < 1"; return GMG_ECOLOR; }
    ctx->user_color0 = std::move(c);
    return GMG_OK;
}

gmg_status gmg_build_hierarchy(gmg_ctx *ctx, int n_levels, int *n_levels_built)
{
    if (!ctx) return GMG_EINVAL;
    if (!ctx->mesh_loaded) { ctx->err = "mesh not loaded"; return GMG_ESTATE; }
    if (n_levels < 1 || n_levels > 3) { ctx->err = "n_levels must be 1..3"; return GMG_EINVAL; }
    gmg_status ret = GMG_OK;
    // GMG_SETUP_TIMES=1: per-phase host setup times on stderr (dev aid)
    const bool tm = std::getenv("GMG_SETUP_TIMES") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto lap = [&](const char *what, int l) {
        if (!tm) return;
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[setup] L%d %-14s %8.3f s\n", l, what, std::chrono::duration<double>(t - t_last).count());
        t_last = t;
    };
    const bool dev = ctx->opt.setup_device == 1;
    cudaStream_t ss = nullptr;
    SetupStats sst;
    if (dev) {
        CK(cudaSetDevice(ctx->opt.device));
        CK(cudaStreamCreateWithFlags(&ss, cudaStreamNonBlocking));
    }
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { if (s) cudaStreamDestroy(s); }
    } sguard{ss};
    try {
        ctx->lv.resize(1);
        for (int l = 0;; ++l) {
            HostLevel &H = ctx->lv[l];
            if (l == 0 && !ctx->user_color0.empty()) {
                H.color = ctx->user_color0;
                H.ncolor = *std::max_element(H.color.begin(), H.color.end());
            } else if (dev) {
                color_level_dev(H, ss, &sst);
            } else {
                color_level(H);
            }
            lap("color", l);
            renumber(H);
            lap("renumber", l);
            H.parent.clear();
            if (l + 1 >= n_levels) break;
            std::vector<int64_t> parent;
            int64_t nc = 0;
            const int64_t merged = dev ? agglomerate_dev(H, ctx->opt.skew_limit, parent, nc, ss, &sst)
                                       : agglomerate(H, ctx->opt.skew_limit, parent, nc);
            lap("agglomerate", l);
            if (merged == 0) {
                ret = GMG_ESTALL;
                ctx->err = "level " + std::to_string(l) + " merged nothing; hierarchy truncated";
                break;
            }
            H.parent = std::move(parent);
            H.n_coarse = nc;
            HostLevel C;
            build_coarse(ctx->lv[l], C);
            lap("build_coarse", l);
            ctx->lv.push_back(std::move(C));
        }
        // domains driven by this process
        ctx->dom.clear();
        const int nd = ctx->opt.nranks > 1 ? 1 : ctx->opt.local_domains;
        for (int k = 0; k < nd; ++k) {
            Domain dm;
            dm.rank = ctx->opt.nranks > 1 ? ctx->opt.rank : k;
            dm.lv.resize(ctx->lv.size());
            for (size_t l = 0; l < ctx->lv.size(); ++l) {
                build_domain_level(ctx->lv[l], dm.rank, dm.lv[l],
                                   ctx->nparts != 1 ? 0 : ctx->flow ? ctx->flow_chunk : ctx->chunk_order ? ctx->order_chunk : 0,
                                   ctx->flow != 0);
                lap("domain_level", (int)l);
            }
            for (size_t l = 0; l + 1 < ctx->lv.size(); ++l)
                link_domain_levels(ctx->lv[l], ctx->lv[l + 1], dm.lv[l], dm.lv[l + 1]);
            lap("link", 0);
            if (tm && dev)
                std::fprintf(stderr, "[setup] device: %lld BFS levels, %lld color rounds, %lld matching rounds\n",
                             (long long)sst.color_levels, (long long)sst.color_rounds, (long long)sst.match_rounds);
            ctx->dom.push_back(std::move(dm));
        }
        if (ctx->p2p && ctx->nparts > 1) {   // fused P2P halo targets
            for (Domain &dm : ctx->dom)
                for (size_t l = 0; l < ctx->lv.size(); ++l) {
                    DomLevel &D = dm.lv[l];
                    std::vector<DomLevel> tmp(D.peers.size());
                    std::vector<const DomLevel *> pd(D.peers.size());
                    for (size_t k = 0; k < D.peers.size(); ++k) {
                        const int q = D.peers[k];
                        if (ctx->opt.nranks > 1) {
                            build_domain_level(ctx->lv[l], q, tmp[k]);
                            pd[k] = &tmp[k];
                        } else {
                            pd[k] = &ctx->dom[q].lv[l];
                        }
                    }
                    build_p2p_targets(D, dm.rank, ctx->lv[l].ncolor, pd);
                }
            lap("p2p_targets", 0);
        }
    } catch (const std::exception &e) {
        ctx->err = e.what();
        return GMG_ETOPO;
    }
    ctx->built = true;
    ctx->ws_ready = ctx->state_set = false;
    if (ctx->graph) { cudaGraphExecDestroy(ctx->graph); ctx->graph = nullptr; }
    if (n_levels_built) *n_levels_built = (int)ctx->lv.size();
    compute_bytes(ctx);
    return ret;
}

gmg_status gmg_get_level_info(gmg_ctx *ctx, int level, int64_t *n_cells, int *n_colors, int64_t *n_faces)
{
    if (!ctx) return GMG_EINVAL;
    if (!ctx->built) { ctx->err = "hierarchy not built"; return GMG_ESTATE; }
    if (level < 0 || level >= (int)ctx->lv.size()) { ctx->err = "bad level"; return GMG_EINVAL; }
    const HostLevel &H = ctx->lv[level];
    if (n_cells) *n_cells = H.n;
    if (n_colors) *n_colors = H.ncolor;
    if (n_faces) *n_faces = H.nf;
    return GMG_OK;
}

gmg_status gmg_get_maps(gmg_ctx *ctx, int level, int32_t *color, int64_t *perm, int64_t *parent)
{
    if (!ctx) return GMG_EINVAL;
    if (!ctx->built) { ctx->err = "hierarchy not built"; return GMG_ESTATE; }
    if (level < 0 || level >= (int)ctx->lv.size()) { ctx->err = "bad level"; return GMG_EINVAL; }
    const HostLevel &H = ctx->lv[level];
    if (color) std::copy(H.color.begin(), H.color.end(), color);
    if (perm) std::copy(H.perm.begin(), H.perm.end(), perm);
    if (parent) {
        if (H.parent.empty()) std::fill(parent, parent + H.n, (int64_t)-1);
        else std::copy(H.parent.begin(), H.parent.end(), parent);
    }
    return GMG_OK;
}

gmg_status gmg_get_level_geometry(gmg_ctx *ctx, int level, double *vol, double *centroid, int64_t *left,
                                  int64_t *right, double *area_vec, double *face_ctr, int8_t *n_gauss)
{
    if (!ctx) return GMG_EINVAL;
    if (!ctx->built) { ctx->err = "hierarchy not built"; return GMG_ESTATE; }
    if (level < 0 || level >= (int)ctx->lv.size()) { ctx->err = "bad level"; return GMG_EINVAL; }
    const HostLevel &H = ctx->lv[level];
    if (vol) std::copy(H.vol.begin(), H.vol.end(), vol);
    if (centroid) std::copy(H.ctr.begin(), H.ctr.end(), centroid);
    if (left) std::copy(H.left.begin(), H.left.end(), left);
    if (right) std::copy(H.right.begin(), H.right.end(), right);
    if (area_vec) std::copy(H.avec.begin(), H.avec.end(), area_vec);
    if (face_ctr) std::copy(H.fctr.begin(), H.fctr.end(), face_ctr);
    if (n_gauss) std::copy(H.ngauss.begin(), H.ngauss.end(), n_gauss);
    return GMG_OK;
}

size_t gmg_workspace_bytes(gmg_ctx *ctx)
{
    if (!ctx || !ctx->built) return 0;
    if (ctx->ho && ho_prepare(ctx) != GMG_OK) return 0;
    Bump b{nullptr};
    carve(ctx, b);
    return b.off + 256;
}

gmg_status gmg_set_workspace(gmg_ctx *ctx, void *dptr, size_t bytes)
{
    if (!ctx) return GMG_EINVAL;
    if (!ctx->built) { ctx->err = "hierarchy not built"; return GMG_ESTATE; }
    if (!dptr || ((uintptr_t)dptr & 15)) { ctx->err = "workspace must be a 16-byte aligned device pointer"; return GMG_EINVAL; }
    if (ctx->ho) {
        const gmg_status hs = ho_prepare(ctx);
        if (hs) return hs;
    }
    if (ctx->opt.fine_operator == 1 && !ctx->ho) { ctx->err = "fine_operator 1 needs gmg_load_ho_geometry"; return GMG_ESTATE; }
    const size_t need = gmg_workspace_bytes(ctx);
    if (bytes < need) { ctx->err = "workspace too small: need " + std::to_string(need); return GMG_ENOMEM; }
    CK(cudaSetDevice(ctx->opt.device));
    Bump b{(char *)dptr};
    carve(ctx, b);
    ctx->ws = dptr;
    ctx->ws_bytes = bytes;
    const int nl = (int)ctx->lv.size();
    std::vector<std::vector<int>> ki;          // host staging kept alive until the sync
    std::vector<std::vector<double>> kd;
    auto up_i = [&](const int *dst, std::vector<int> v) -> cudaError_t {
        ki.push_back(std::move(v));
        return cudaMemcpyAsync((void *)dst, ki.back().data(), ki.back().size() * sizeof(int), cudaMemcpyHostToDevice, ctx->stream);
    };
    auto up_raw = [&](const void *dst, const void *src, size_t bytes_) -> cudaError_t {
        if (!bytes_) return cudaSuccess;
        return cudaMemcpyAsync((void *)dst, src, bytes_, cudaMemcpyHostToDevice, ctx->stream);
    };
    for (Domain &dm : ctx->dom) {
        for (int l = 0; l < nl; ++l) {
            const HostLevel &G = ctx->lv[l];
            const DomLevel &H = dm.lv[l];
            DevLevel &L = dm.dv[l];
            CK(up_raw(L.fl, H.fl.data(), H.fl.size() * sizeof(int)));
            CK(up_raw(L.fr, H.fr.data(), H.fr.size() * sizeof(int)));
            std::vector<double> fA((size_t)G.dim * H.nf);
            std::vector<int> fM8((H.nf + 3) / 4 + 1, 0);
            std::vector<int8_t> fM(H.nf);
            for (int64_t k = 0; k < H.nf; ++k) {
                for (int q = 0; q < G.dim; ++q) fA[(size_t)q * H.nf + k] = G.avec[(size_t)q * G.nf + H.fnat[k]];
                fM[k] = G.ngauss[H.fnat[k]];
            }
            std::memcpy(fM8.data(), fM.data(), fM.size());
            kd.push_back(std::move(fA));
            CK(up_raw(L.fA, kd.back().data(), kd.back().size() * sizeof(double)));
            ki.push_back(std::move(fM8));
            CK(up_raw(L.fM, ki.back().data(), (size_t)H.nf));
            CK(up_raw(L.vol, H.vol.data(), H.vol.size() * sizeof(double)));
            CK(up_raw(L.deg_int, H.deg_int.data(), H.deg_int.size()));
            CK(up_raw(L.deg_all, H.deg_all.data(), H.deg_all.size()));
            CK(up_raw(L.gbase, H.gbase.data(), H.gbase.size() * sizeof(int)));
            CK(up_raw(L.gface, H.gface.data(), H.gface.size() * sizeof(int)));
            CK(up_raw(L.ecell, H.ell_cell.data(), H.ell_cell.size() * sizeof(int)));
            CK(up_raw(L.spcell, H.sp_cell.data(), H.sp_cell.size() * sizeof(int)));
            CK(up_raw(L.fslot, H.fslot.data(), H.fslot.size() * sizeof(int)));
            CK(up_raw(L.p2p_off, H.p2p_off.data(), H.p2p_off.size() * sizeof(int)));
            CK(up_raw(L.p2p_k, H.p2p_k.data(), H.p2p_k.size() * sizeof(int)));
            CK(up_raw(L.p2p_g, H.p2p_g.data(), H.p2p_g.size() * sizeof(int)));
            CK(up_raw(L.p2p_wait, H.peers.data(), H.peers.size() * sizeof(int)));
            if (H.nchunk) {
                std::vector<int> sg(H.seg.begin(), H.seg.end());
                CK(up_i(L.seg, std::move(sg)));
                CK(up_raw(L.cnoff, H.cnoff.data(), H.cnoff.size() * sizeof(int)));
                CK(up_raw(L.cnidx, H.cnidx.data(), H.cnidx.size() * sizeof(int)));
            }
            {
                std::vector<int> si(2 * H.n_own);
                for (int64_t i = 0; i < H.n_own; ++i) { si[2 * i] = H.ell_cell[i]; si[2 * i + 1] = H.deg_int[i]; }
                CK(up_i((const int *)L.sinfo, std::move(si)));
                std::vector<int> gi(4 * H.n_own);
                for (int64_t i = 0; i < H.n_own; ++i) {
                    gi[4 * i] = H.gbase[i];
                    gi[4 * i + 1] = (int)H.deg_all[i] | ((int)H.deg_int[i] << 16);
                    gi[4 * i + 2] = H.ell_cell[i];
                    gi[4 * i + 3] = H.ell_stride[i];
                }
                CK(up_i((const int *)L.ginfo, std::move(gi)));
            }
            CK(up_raw(L.estride, H.ell_stride.data(), H.ell_stride.size() * sizeof(int)));
            CK(up_raw(L.sJe, H.sJe.data(), H.sJe.size() * sizeof(int)));
            CK(up_raw(L.sRe, H.sRe.data(), H.sRe.size() * sizeof(double)));
            std::vector<int> perm(H.n_loc);
            for (int64_t i = 0; i < H.n_loc; ++i) perm[i] = (int)H.l2n[i];
            CK(up_i(L.perm, std::move(perm)));
            if (l > 0) CK(up_raw(L.child, H.child.data(), H.child.size() * sizeof(int)));
            if (l + 1 < nl) CK(up_raw(L.parent, H.parent.data(), H.parent.size() * sizeof(int)));
            CK(up_raw(L.send_idx, H.send_idx.data(), H.send_idx.size() * sizeof(int)));
            CK(up_raw(L.recv_idx, H.recv_idx.data(), H.recv_idx.size() * sizeof(int)));
            // alpha = 1 until set (df_mode 2 keeps it)
            k_fill<<<nblk(H.n_own), 256, 0, ctx->stream>>>((int)H.n_own, L.alpha, 1.0);
            CK(cudaMemsetAsync(L.rec, 0, sizeof(double) * kRecStride * H.n_loc, ctx->stream));
        }
    }
    CK(cudaMemsetAsync(ctx->d_flag, 0, 4 * sizeof(int), ctx->stream));
    CK(cudaMemsetAsync(ctx->d_bar, 0, 2 * sizeof(int), ctx->stream));
    for (Domain &dm : ctx->dom) {   // P2P phase counts / control
        CK(cudaMemsetAsync(dm.dv[0].p2p_flags, 0, sizeof(int) * std::max(ctx->nparts, 1), ctx->stream));
        CK(cudaMemsetAsync(dm.dv[0].p2p_ctl, 0, sizeof(int) * 4, ctx->stream));
    }
    ctx->p2p_ready = false;
    if (ctx->p2p && ctx->nparts > 1 && ctx->opt.nranks == 1) {   // local domains: peers are in this process
        CK(cudaStreamSynchronize(ctx->stream));
        for (Domain &dm : ctx->dom)
            for (int l = 0; l < nl; ++l) {
                const DomLevel &H = dm.lv[l];
                std::vector<double *> pr(H.peers.size());
                std::vector<int *> sg(H.peers.size());
                for (size_t k = 0; k < H.peers.size(); ++k) {
                    DevLevel &Q = ctx->dom[H.peers[k]].dv[l];
                    pr[k] = Q.rec;
                    sg[k] = Q.p2p_flags + dm.rank;
                }
                if (!pr.empty()) {
                    CK(cudaMemcpy(dm.dv[l].peer_rec, pr.data(), pr.size() * sizeof(double *), cudaMemcpyHostToDevice));
                    CK(cudaMemcpy(dm.dv[l].p2p_sig, sg.data(), sg.size() * sizeof(int *), cudaMemcpyHostToDevice));
                }
            }
        ctx->p2p_ready = true;
    }
    if (!ctx->copy) {                      // copy stream + events of the pipelined host I/O
        CK(cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&ctx->copy_out, cudaStreamNonBlocking));
        for (int k = 0; k < 2; ++k) {
            CK(cudaEventCreateWithFlags(&ctx->ev_in_ready[k], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ctx->ev_in_free[k], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ctx->ev_out_ready[k], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ctx->ev_out_free[k], cudaEventDisableTiming));
            CK(cudaEventRecord(ctx->ev_in_free[k], ctx->stream));
            CK(cudaEventRecord(ctx->ev_out_free[k], ctx->copy_out));
        }
    }
    if (ctx->nparts > 1 && !ctx->side) {   // side stream + events of the exchange overlap
        CK(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    {   // persisting-L2 window over the gathered cell records, attached to the sweep launches only, with a
        // 40 MB set-aside (GMG_L2PERSIST: 0 = off, 1 = the largest set-aside, > 1 = that many MB).  Measured
        // (DESIGN §6): 40 MB -3 % per V-cycle; the largest set-aside speeds the sweeps but starves the rest
        const char *e = std::getenv("GMG_L2PERSIST");
        if (!e) e = "40";
        if (std::atoi(e) > 0) {
            int maxp = 0, maxw = 0;
            cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, ctx->opt.device);
            cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, ctx->opt.device);
            // GMG_L2PERSIST=1: the largest set-aside; > 1: that many MB
            const size_t want = std::atoi(e) > 1 ? (size_t)std::atoi(e) << 20 : (size_t)maxp;
            const size_t setaside = std::min<size_t>((size_t)maxp, want);
            CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, setaside));
            ctx->l2_window = std::min<size_t>((size_t)maxw, setaside);
            ctx->l2_maxw = (size_t)maxw;
            if (const char *f = std::getenv("GMG_L2FULL")) ctx->l2_full = std::atoi(f);
        }
    }
    {   // sweep grid: whole resident waves only (grid-stride kernel), GMG_SWEEP_WAVES (0 = uncapped)
        int waves = 1, nsm = 0, per_sm = 0;
        if (const char *e = std::getenv("GMG_SWEEP_WAVES")) waves = std::atoi(e);
        if (const char *e = std::getenv("GMG_SWEEPV")) ctx->sweep_var = std::atoi(e);
        if (const char *e = std::getenv("GMG_SWEEP_BS")) ctx->sweep_bs = std::atoi(e);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->opt.device);
        if (ctx->opt.dim == 3)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sweep<3, 2, 4, 3>, 256, 0);
        else
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sweep<2, 2, 4, 3>, 256, 0);
        ctx->sweep_grid_cap = waves > 0 ? waves * nsm * std::max(per_sm, 1) : 0;
        int per_flow = 0;
        if (ctx->opt.dim == 3) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_flow, k_sweep_flow<3>, 256, 0);
        else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_flow, k_sweep_flow<2>, 256, 0);
        ctx->flow_grid = per_flow * nsm;
        int per_tail = 0;
        if (ctx->opt.dim == 3) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_tail, k_sweep_tailc<3>, 256, 0);
        else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_tail, k_sweep_tailc<2>, 256, 0);
        ctx->tailc_grid = per_tail * nsm;
    }
    {   // dynamic shared memory of the warp-staged sweep (may exceed the 48 KB default)
        int mx = 1;
        for (Domain &dm : ctx->dom)
            for (auto &B : dm.lbytes) mx = std::max(mx, B.max_ws);
        const int per_warp = mx * (kRecS + kSlotRec) * (int)sizeof(double);
        CK(cudaFuncSetAttribute(k_sweep_ws<3, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, std::min(per_warp, 227 * 1024)));
        CK(cudaFuncSetAttribute(k_sweep_ws<3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, std::min(2 * per_warp, 227 * 1024)));
        CK(cudaFuncSetAttribute(k_sweep_ws<3, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, std::min(4 * per_warp, 227 * 1024)));
        CK(cudaFuncSetAttribute(k_sweep_ws<2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, std::min(per_warp, 227 * 1024)));
        CK(cudaFuncSetAttribute(k_sweep_ws<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, std::min(2 * per_warp, 227 * 1024)));
        CK(cudaFuncSetAttribute(k_sweep_ws<2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, std::min(4 * per_warp, 227 * 1024)));
        if (ctx->wsweep && ctx->wsweep * per_warp > 227 * 1024) ctx->wsweep = 1;
        int mp = 1;
        for (Domain &dm : ctx->dom)
            for (auto &B : dm.lbytes) mp = std::max(mp, B.max_pipe);
        const int pipe_bytes = std::min(kPW * PipeLayout{mp}.warp() * (int)sizeof(double), 227 * 1024);
        CK(cudaFuncSetAttribute(k_sweep_pipe<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, pipe_bytes));
        CK(cudaFuncSetAttribute(k_sweep_pipe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, pipe_bytes));
    }
    if (ctx->opt.nranks > 1 && !ctx->nccl_comm) {
        if (!nccl().load(ctx->err)) return GMG_ENCCL;
        ncclUniqueId id;
        std::memcpy(&id, ctx->opt.nccl_id, sizeof(id));
        ncclComm_t comm;
        const ncclResult_t r = nccl().CommInitRank(&comm, ctx->opt.nranks, id, ctx->opt.rank);
        if (r != ncclSuccess) {
            ctx->err = std::string("ncclCommInitRank: ") + (nccl().ErrStr ? nccl().ErrStr(r) : "error");
            return GMG_ENCCL;
        }
        ctx->nccl_comm = comm;
    }
    if (ctx->ho) {
        const int nvd = (ctx->opt.dim + 2) * ctx->opt.dim;
        for (Domain &dm : ctx->dom) {
            const HoLocal &H = dm.ho;
            HoDev &V = dm.dv[0].ho;
            const int64_t nl = dm.lv[0].n_loc, n = dm.lv[0].n_own;
            CK(cudaMemcpyAsync((void *)V.ctr, H.ctr.data(), H.ctr.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
            CK(cudaMemcpyAsync((void *)V.m2, H.m2l.data(), H.m2l.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
            CK(cudaMemcpyAsync((void *)V.gp, H.gpl.data(), H.gpl.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
            CK(cudaMemcpyAsync((void *)V.gw, H.gwl.data(), H.gwl.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
            CK(cudaMemcpyAsync((void *)V.hfoff, H.hfoff.data(), H.hfoff.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
            CK(cudaMemcpyAsync((void *)V.hface, H.hface.data(), H.hface.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
            CK(cudaMemcpyAsync((void *)V.hrec, H.hrec.data(), H.hrec.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
            CK(cudaMemcpyAsync((void *)V.poff, H.poff.data(), H.poff.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
            if (!H.P.empty())
                CK(cudaMemcpyAsync((void *)V.P, H.P.data(), H.P.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
            k_fill<<<nblk(nl * nvd), 256, 0, ctx->stream>>>((int)(nl * nvd), V.G_, 0.0);   // reading C1
            k_fill<<<nblk(n), 256, 0, ctx->stream>>>((int)n, V.alpha, 1.0);
        }
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(ctx->stream));
    }
    if (ctx->graph) { cudaGraphExecDestroy(ctx->graph); ctx->graph = nullptr; }
    ctx->ws_ready = true;
    ctx->state_set = false;
    return GMG_OK;
}

gmg_status gmg_set_state(gmg_ctx *ctx, const double *W, const double *W_inf)
{
    if (!ctx) return GMG_EINVAL;
    gmg_status st = check_ready(ctx, false);
    if (st) return st;
    if (!W || !W_inf) { ctx->err = "null state"; return GMG_EINVAL; }
    const int nv = ctx->opt.dim + 2;
    bool same = true;
    for (int q = 0; q < nv; ++q) {
        same = same && std::memcmp(&ctx->winf[q], &W_inf[q], sizeof(double)) == 0;
        ctx->winf[q] = W_inf[q];
    }
    // the far-field state is a kernel parameter of the captured V-cycle: re-capture only if it changed
    if (ctx->graph && !same) { cudaGraphExecDestroy(ctx->graph); ctx->graph = nullptr; }
    st = put_natural(ctx, 0, W, nv, [](DevLevel &L) { return L.W; }, true);
    if (st) return st;
    ctx->state_set = true;
    return GMG_OK;
}

gmg_status gmg_set_level_state(gmg_ctx *ctx, int level, const double *W)
{
    if (!ctx) return GMG_EINVAL;
    gmg_status st = check_ready(ctx, false);
    if (st) return st;
    if (level < 0 || level >= (int)ctx->lv.size() || !W) { ctx->err = "bad level / null"; return GMG_EINVAL; }
    st = put_natural(ctx, level, W, ctx->opt.dim + 2, [](DevLevel &L) { return L.W; }, true);
    if (st) return st;
    if (level == 0) ctx->state_set = true;
    return GMG_OK;
}

gmg_status gmg_get_state(gmg_ctx *ctx, int level, double *W_out)
{
    if (!ctx) return GMG_EINVAL;
    gmg_status st = check_ready(ctx, false);
    if (st) return st;
    if (level < 0 || level >= (int)ctx->lv.size() || !W_out) { ctx->err = "bad level / null"; return GMG_EINVAL; }
    return get_natural(ctx, level, [](DevLevel &L) { return (const double *)L.W; }, ctx->opt.dim + 2, W_out);
}

gmg_status gmg_set_alpha(gmg_ctx *ctx, const double *alpha)
{
    if (!ctx) return GMG_EINVAL;
    gmg_status st = check_ready(ctx, false);
    if (st) return st;
    if (!alpha) { ctx->err = "null alpha"; return GMG_EINVAL; }
    return put_natural(ctx, 0, alpha, 1, [](DevLevel &L) { return L.alpha; }, false);
}

gmg_status gmg_residual(gmg_ctx *ctx, int level, double *R_out, double *alpha_out, double *sigma_out)
{
    if (!ctx) return GMG_EINVAL;
    gmg_status st = check_ready(ctx, level == 0);
    if (st) return st;
    if (level < 0 || level >= (int)ctx->lv.size()) { ctx->err = "bad level"; return GMG_EINVAL; }
    Launcher Lc{ctx, ctx->stream};
    for (size_t d = 0; d < ctx->dom.size(); ++d) {
        Domain &dm = ctx->dom[d];
        DevLevel &L = dm.dv[level];
        double *save_alpha = L.alpha;
        L.alpha = L.tmp;    // scratch: the level's own alpha stays intact
        if (ctx->opt.dim == 2) {
            enqueue_face<2>(Lc, dm, level, L.W, true, false, true);
            enqueue_gather<2>(Lc, dm, (int)d, level, G_FLUX | G_WRITE_RT | G_ALPHA | G_SIGMA, nullptr);
        } else {
            enqueue_face<3>(Lc, dm, level, L.W, true, false, true);
            enqueue_gather<3>(Lc, dm, (int)d, level, G_FLUX | G_WRITE_RT | G_ALPHA | G_SIGMA, nullptr);
        }
        L.alpha = save_alpha;
    }
    CK(cudaGetLastError());
    const int nv = ctx->opt.dim + 2;
    if (R_out) { st = get_natural(ctx, level, [](DevLevel &L) { return (const double *)L.Rt; }, nv, R_out); if (st) return st; }
    if (alpha_out) { st = get_natural(ctx, level, [](DevLevel &L) { return (const double *)L.tmp; }, 1, alpha_out); if (st) return st; }
    if (sigma_out) { st = get_natural(ctx, level, [](DevLevel &L) { return (const double *)L.sigma; }, 1, sigma_out); if (st) return st; }
    CK(cudaStreamSynchronize(ctx->stream));
    return GMG_OK;
}

gmg_status gmg_set_level_inputs(gmg_ctx *ctx, int level, const double *Rt, const double *alpha)
{
    if (!ctx) return GMG_EINVAL;
    gmg_status st = check_ready(ctx, false);
    if (st) return st;
    if (level < 0 || level >= (int)ctx->lv.size()) { ctx->err = "bad level"; return GMG_EINVAL; }
    // owned cells only (Rt and alpha have no ghost entries)
    if (Rt) {
        st = put_natural(ctx, level, Rt, ctx->opt.dim + 2, [](DevLevel &L) { return L.Rt; }, false);
        if (st) return st;
    }
    if (alpha) { st = put_natural(ctx, level, alpha, 1, [](DevLevel &L) { return L.alpha; }, false); if (st) return st; }
    CK(cudaStreamSynchronize(ctx->stream));
    return GMG_OK;
}

// test only: one smoothing step of every local domain in ONE cooperative
// launch, one block group per domain, running the fused-P2P-halo protocol
// concurrently (kernels.cuh k_p2p_emulate)
gmg_status gmg_p2p_emulate_smooth(gmg_ctx *ctx, int level, int n_sweeps, double *dW_out)
{
    if (!ctx) return GMG_EINVAL;
    gmg_status st = check_ready(ctx, false);
    if (st) return st;
    if (level < 0 || level >= (int)ctx->lv.size() || n_sweeps < 1) { ctx->err = "bad level / n_sweeps"; return GMG_EINVAL; }
    const int P = (int)ctx->dom.size();
    if (!ctx->p2p || !ctx->p2p_ready || ctx->opt.nranks != 1 || P < 2 || P > kEmuMaxDom ||
        ctx->lv[level].ncolor > kEmuMaxCol) {
        ctx->err = "P2P emulation needs GMG_P2P=1, 2..16 local domains, <= 24 colors";
        return GMG_ESTATE;
    }
    Launcher Lc{ctx, ctx->stream};
    const int gf = G_PREPARE | G_SIGMA | G_COPY_W | G_ZERO_DW;
    for (size_t d = 0; d < ctx->dom.size(); ++d) {
        if (ctx->opt.dim == 2) {
            enqueue_face<2>(Lc, ctx->dom[d], level, ctx->dom[d].dv[level].W, false, false, false, true);
            enqueue_gather<2>(Lc, ctx->dom[d], (int)d, level, gf, nullptr);
        } else {
            enqueue_face<3>(Lc, ctx->dom[d], level, ctx->dom[d].dv[level].W, false, false, false, true);
            enqueue_gather<3>(Lc, ctx->dom[d], (int)d, level, gf, nullptr);
        }
    }
    if (ctx->opt.dim == 2) enqueue_ghost_wlin<2>(Lc, level);
    else enqueue_ghost_wlin<3>(Lc, level);
    // phases: a synchronisation phase, Algorithm 2 (repeated phases dropped), a synchronisation phase
    const int nc = ctx->lv[level].ncolor;
    EmuArgs e{};
    std::vector<int> seq{255};
    for (int sw = 0; sw < n_sweeps; ++sw)
        for (int half = 0; half < 2; ++half)
            for (int cc = 0; cc < nc; ++cc) {
                const int c = half == 0 ? cc : nc - 1 - cc;
                if (!(ctx->skip_repeat && seq.size() > 1 && seq.back() == c)) seq.push_back(c);
            }
    seq.push_back(255);
    if ((int)seq.size() > kFlowMaxPh) { ctx->err = "too many phases"; return GMG_EINVAL; }
    e.ndom = P;
    e.nph = (int)seq.size();
    for (size_t k = 0; k < seq.size(); ++k) e.ph[k] = (unsigned short)seq[k];
    std::vector<EmuDom> ed(P);
    for (int d = 0; d < P; ++d) {
        DevLevel &L = ctx->dom[d].dv[level];
        const DomLevel &H = ctx->dom[d].lv[level];
        ed[d].a = SweepArgs{0, 0, ctx->opt.gamma - 1.0, L.rec, L.ecell, L.deg_int, L.sinfo, L.sJe, L.sRe, L.Rt, nullptr, 0, 0};
        ed[d].p = P2PArgs{L.p2p_off, L.p2p_k, L.p2p_g, L.peer_rec, L.npeer, L.p2p_wait, L.p2p_sig, L.p2p_flags, L.p2p_ctl};
        for (int c = 0; c <= nc; ++c) ed[d].blk[c] = (int)H.blk[c];
        ed[d].n_own = (int)H.n_own;
        ed[d].rank = ctx->dom[d].rank;
        ed[d].bar = ctx->d_emu_bar + 2 * d;
    }
    CK(cudaMemsetAsync(ctx->d_emu_bar, 0, sizeof(int) * 2 * kEmuMaxDom, ctx->stream));
    CK(cudaMemcpyAsync(ctx->d_emu, ed.data(), sizeof(EmuDom) * P, cudaMemcpyHostToDevice, ctx->stream));
    e.dom = (const EmuDom *)ctx->d_emu;
    int per_sm = 0, nsm = 0;
    if (ctx->opt.dim == 2) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_p2p_emulate<2>, 256, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_p2p_emulate<3>, 256, 0);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->opt.device);
    e.per_group = std::max(1, per_sm * nsm / P);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(e.per_group * P);
    cfg.blockDim = dim3(256);
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (ctx->opt.dim == 2) CK(cudaLaunchKernelEx(&cfg, k_p2p_emulate<2>, e));
    else CK(cudaLaunchKernelEx(&cfg, k_p2p_emulate<3>, e));
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    for (Domain &dm : ctx->dom) {
        int c2 = 0;
        CK(cudaMemcpy(&c2, dm.dv[0].p2p_ctl + 2, sizeof(int), cudaMemcpyDeviceToHost));
        if (c2) { ctx->err = "P2P emulation: peer phase wait timed out"; return GMG_ECUDA; }
    }
    const int nv = ctx->opt.dim + 2;
    const int RD = ctx->opt.dim == 3 ? Rec<3>::DW : Rec<2>::DW;
    if (dW_out) return get_natural(ctx, level, [](DevLevel &L) { return (const double *)L.rec; }, nv, dW_out, kRecStride, RD);
    return GMG_OK;
}

gmg_status gmg_smooth(gmg_ctx *ctx, int level, int n_sweeps, double *dW_out)
{
    if (!ctx) return GMG_EINVAL;
    gmg_status st = check_ready(ctx, false);
    if (st) return st;
    if (level < 0 || level >= (int)ctx->lv.size() || n_sweeps < 1) { ctx->err = "bad level / n_sweeps"; return GMG_EINVAL; }
    Launcher Lc{ctx, ctx->stream};
    const int gf = G_PREPARE | G_SIGMA | G_COPY_W | G_ZERO_DW;
    auto rhs = [](DevLevel &L) { return (const double *)L.Rt; };
    auto nowout = [](DevLevel &) { return (double *)nullptr; };
    if (ctx->opt.dim == 2) {
        for (size_t d = 0; d < ctx->dom.size(); ++d) {
            enqueue_face<2>(Lc, ctx->dom[d], level, ctx->dom[d].dv[level].W, false, false, false, true);
            enqueue_gather<2>(Lc, ctx->dom[d], (int)d, level, gf, nullptr);
        }
        enqueue_ghost_wlin<2>(Lc, level);
        enqueue_sweeps<2>(Lc, level, n_sweeps, rhs, nowout);
    } else {
        for (size_t d = 0; d < ctx->dom.size(); ++d) {
            enqueue_face<3>(Lc, ctx->dom[d], level, ctx->dom[d].dv[level].W, false, false, false, true);
            enqueue_gather<3>(Lc, ctx->dom[d], (int)d, level, gf, nullptr);
        }
        enqueue_ghost_wlin<3>(Lc, level);
        enqueue_sweeps<3>(Lc, level, n_sweeps, rhs, nowout);
    }
    CK(cudaGetLastError());
    {
        int fe = 0;
        CK(cudaMemcpyAsync(&fe, ctx->d_flag + 2, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        if (fe) { ctx->err = "dependency-driven sweep: progress wait timed out"; return GMG_ECUDA; }
    }
    const int nv = ctx->opt.dim + 2;
    const int RD = ctx->opt.dim == 3 ? Rec<3>::DW : Rec<2>::DW;
    if (dW_out) {
        st = get_natural(ctx, level, [](DevLevel &L) { return (const double *)L.rec; }, nv, dW_out, kRecStride, RD);
        if (st) return st;
    }
    return GMG_OK;
}

static gmg_status build_graph(gmg_ctx *ctx)
{
    cudaStream_t cs;
    CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t g;
    Launcher Lc{ctx, cs};
    ctx->launches = 0;
    ctx->exchanges = 0;
    for (double &b : ctx->kbytes) b = 0;
    cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
        if (ctx->opt.dim == 2) vcycle_dispatch<2>(Lc);
        else vcycle_dispatch<3>(Lc);
        e = cudaStreamEndCapture(cs, &g);
    }
    cudaStreamDestroy(cs);
    if (e != cudaSuccess) { ctx->err = std::string("graph capture: ") + cudaGetErrorString(e); return GMG_ECUDA; }
    e = cudaGraphInstantiate(&ctx->graph, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) { ctx->err = std::string("graph instantiate: ") + cudaGetErrorString(e); return GMG_ECUDA; }
    ctx->graph_launches = ctx->launches;
    return GMG_OK;
}

static gmg_status finish_history(gmg_ctx *ctx, int n_cycles, double *res_hist)
{
    const int nv = ctx->opt.dim + 2;
    int flags[3] = {0, 0, 0};
    CK(cudaMemcpyAsync(flags, ctx->d_flag, 3 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    if (res_hist)
        CK(cudaMemcpyAsync(res_hist, ctx->d_hist, sizeof(double) * nv * std::min(n_cycles + 1, ctx->hist_cap),
                           cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (flags[2]) { ctx->err = "dependency-driven sweep: progress wait timed out"; return GMG_ECUDA; }
    if (ctx->p2p) {
        for (Domain &dm : ctx->dom) {
            int c2 = 0;
            CK(cudaMemcpy(&c2, dm.dv[0].p2p_ctl + 2, sizeof(int), cudaMemcpyDeviceToHost));
            if (c2) { ctx->err = "P2P halo: peer phase wait timed out"; return GMG_ECUDA; }
        }
    }
    if (flags[1]) { ctx->err = "non-finite residual (level 0)"; return GMG_ENONFINITE; }
    return GMG_OK;
}

gmg_status gmg_vcycle(gmg_ctx *ctx, int n_cycles, double *res_hist)
{
    if (!ctx) return GMG_EINVAL;
    gmg_status st = check_ready(ctx);
    if (st) return st;
    if (n_cycles < 0 || n_cycles + 1 > ctx->hist_cap) { ctx->err = "n_cycles out of range"; return GMG_EINVAL; }
    if (!ctx->graph) { st = build_graph(ctx); if (st) return st; }
    CK(cudaMemsetAsync(ctx->d_flag, 0, 3 * sizeof(int), ctx->stream));
    for (int k = 0; k < n_cycles; ++k) CK(cudaGraphLaunch(ctx->graph, ctx->stream));
    Launcher Lc{ctx, ctx->stream};
    if (ctx->opt.dim == 2) enqueue_final_norm<2>(Lc);
    else enqueue_final_norm<3>(Lc);
    CK(cudaGetLastError());
    return finish_history(ctx, n_cycles, res_hist);
}

// ---------------------------------------------------------------- pipelined host I/O
static gmg_status async_ready(gmg_ctx *ctx, bool need_state, bool natural = true)
{
    gmg_status st = check_ready(ctx, need_state);
    if (st) return st;
    if (natural && ctx->opt.nranks > 1) { ctx->err = "natural-order pipelined host I/O is single-rank (use *_owned_async)"; return GMG_EINVAL; }
    if (!natural && ctx->dom.size() != 1) { ctx->err = "owned-layout host I/O needs one domain per process"; return GMG_EINVAL; }
    if (!ctx->async_flag_reset) {
        CK(cudaMemsetAsync(ctx->d_flag, 0, 3 * sizeof(int), ctx->stream));
        ctx->async_flag_reset = true;
    }
    return GMG_OK;
}

gmg_status gmg_set_state_async(gmg_ctx *ctx, const double *W, const double *W_inf)
{
    if (!ctx) return GMG_EINVAL;
    gmg_status st = async_ready(ctx, false);
    if (st) return st;
    if (!W || !W_inf) { ctx->err = "null state"; return GMG_EINVAL; }
    const int nv = ctx->opt.dim + 2;
    bool same = true;
    for (int q = 0; q < nv; ++q) {
        same = same && std::memcmp(&ctx->winf[q], &W_inf[q], sizeof(double)) == 0;
        ctx->winf[q] = W_inf[q];
    }
    if (ctx->graph && !same) { cudaGraphExecDestroy(ctx->graph); ctx->graph = nullptr; }
    const int k = ctx->in_slot;
    const int64_t N = ctx->lv[0].n;
    // copy stream: wait until the compute stream has consumed this slot, then H2D
    CK(cudaStreamWaitEvent(ctx->copy, ctx->ev_in_free[k], 0));
    CK(cudaMemcpyAsync(ctx->stage_in[k], W, sizeof(double) * nv * N, cudaMemcpyDefault, ctx->copy));
    CK(cudaEventRecord(ctx->ev_in_ready[k], ctx->copy));
    // compute stream: scatter into every domain's local state (owned + ghosts)
    CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_in_ready[k], 0));
    for (Domain &dm : ctx->dom) {
        DevLevel &L = dm.dv[0];
        k_to_internal<<<nblk(L.n_loc), 256, 0, ctx->stream>>>(L.n_loc, (int)N, nv, L.perm, ctx->stage_in[k], L.W, nv, 0);
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(ctx->ev_in_free[k], ctx->stream));
    ctx->in_slot ^= 1;
    ctx->state_set = true;
    return GMG_OK;
}

gmg_status gmg_vcycle_async(gmg_ctx *ctx, int n_cycles)
{
    if (!ctx) return GMG_EINVAL;
    gmg_status st = async_ready(ctx, true, ctx->opt.nranks == 1);
    if (st) return st;
    if (n_cycles < 0) { ctx->err = "n_cycles out of range"; return GMG_EINVAL; }
    if (!ctx->graph) { st = build_graph(ctx); if (st) return st; }
    for (int k = 0; k < n_cycles; ++k) CK(cudaGraphLaunch(ctx->graph, ctx->stream));
    Launcher Lc{ctx, ctx->stream};
    if (ctx->opt.dim == 2) enqueue_final_norm<2>(Lc);
    else enqueue_final_norm<3>(Lc);
    CK(cudaGetLastError());
    return GMG_OK;
}

gmg_status gmg_get_state_async(gmg_ctx *ctx, double *W_out)
{
    if (!ctx) return GMG_EINVAL;
    gmg_status st = async_ready(ctx, false);
    if (st) return st;
    if (!W_out) { ctx->err = "null output"; return GMG_EINVAL; }
    const int nv = ctx->opt.dim + 2;
    const int k = ctx->out_slot;
    const int64_t N = ctx->lv[0].n;
    // compute stream: wait until the previous D2H of this slot has drained, gather to natural order
    CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_out_free[k], 0));
    for (Domain &dm : ctx->dom) {
        DevLevel &L = dm.dv[0];
        k_to_natural<<<nblk(L.n), 256, 0, ctx->stream>>>(L.n, (int)N, nv, L.perm, L.W, ctx->stage_out[k], nv, 0);
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(ctx->ev_out_ready[k], ctx->stream));
    // result copy stream (its own FIFO, so the next input copy never queues behind it): D2H once gathered
    CK(cudaStreamWaitEvent(ctx->copy_out, ctx->ev_out_ready[k], 0));
    CK(cudaMemcpyAsync(W_out, ctx->stage_out[k], sizeof(double) * nv * N, cudaMemcpyDefault, ctx->copy_out));
    CK(cudaEventRecord(ctx->ev_out_free[k], ctx->copy_out));
    ctx->out_slot ^= 1;
    return GMG_OK;
}

static bool winf_update(gmg_ctx *ctx, const double *W_inf)
{
    const int nv = ctx->opt.dim + 2;
    bool same = true;
    for (int q = 0; q < nv; ++q) {
        same = same && std::memcmp(&ctx->winf[q], &W_inf[q], sizeof(double)) == 0;
        ctx->winf[q] = W_inf[q];
    }
    if (ctx->graph && !same) { cudaGraphExecDestroy(ctx->graph); ctx->graph = nullptr; }
    return same;
}

gmg_status gmg_set_state_owned_async(gmg_ctx *ctx, const double *W_owned, const double *W_inf)
{
    if (!ctx) return GMG_EINVAL;
    gmg_status st = async_ready(ctx, false, false);
    if (st) return st;
    if (!W_owned || !W_inf) { ctx->err = "null state"; return GMG_EINVAL; }
    winf_update(ctx, W_inf);
    const int nv = ctx->opt.dim + 2, k = ctx->in_slot;
    DevLevel &L = ctx->dom[0].dv[0];
    CK(cudaStreamWaitEvent(ctx->copy, ctx->ev_in_free[k], 0));
    CK(cudaMemcpyAsync(ctx->stage_in[k], W_owned, sizeof(double) * nv * L.n, cudaMemcpyDefault, ctx->copy));
    CK(cudaEventRecord(ctx->ev_in_ready[k], ctx->copy));
    CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_in_ready[k], 0));
    k_soa_to_aos<<<nblk(L.n), 256, 0, ctx->stream>>>(L.n, nv, ctx->stage_in[k], L.W);   // ghosts: V-cycle halo
    CK(cudaGetLastError());
    CK(cudaEventRecord(ctx->ev_in_free[k], ctx->stream));
    ctx->in_slot ^= 1;
    ctx->state_set = true;
    return GMG_OK;
}

gmg_status gmg_get_state_owned_async(gmg_ctx *ctx, double *W_owned_out)
{
    if (!ctx) return GMG_EINVAL;
    gmg_status st = async_ready(ctx, false, false);
    if (st) return st;
    if (!W_owned_out) { ctx->err = "null output"; return GMG_EINVAL; }
    const int nv = ctx->opt.dim + 2, k = ctx->out_slot;
    DevLevel &L = ctx->dom[0].dv[0];
    CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_out_free[k], 0));
    k_aos_to_soa<<<nblk(L.n), 256, 0, ctx->stream>>>(L.n, nv, L.W, ctx->stage_out[k]);
    CK(cudaGetLastError());
    CK(cudaEventRecord(ctx->ev_out_ready[k], ctx->stream));
    CK(cudaStreamWaitEvent(ctx->copy_out, ctx->ev_out_ready[k], 0));
    CK(cudaMemcpyAsync(W_owned_out, ctx->stage_out[k], sizeof(double) * nv * L.n, cudaMemcpyDefault, ctx->copy_out));
    CK(cudaEventRecord(ctx->ev_out_free[k], ctx->copy_out));
    ctx->out_slot ^= 1;
    return GMG_OK;
}

gmg_status gmg_sync(gmg_ctx *ctx)
{
    if (!ctx) return GMG_EINVAL;
    if (!ctx->ws_ready) { ctx->err = "workspace not set"; return GMG_ESTATE; }
    int flags[3] = {0, 0, 0};
    CK(cudaMemcpyAsync(flags, ctx->d_flag, 3 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaStreamSynchronize(ctx->copy));
    CK(cudaStreamSynchronize(ctx->copy_out));
    ctx->async_flag_reset = false;
    if (flags[1]) { ctx->err = "non-finite residual (level 0)"; return GMG_ENONFINITE; }
    return GMG_OK;
}

gmg_status gmg_profile_vcycle(gmg_ctx *ctx, int n_cycles, double *ms_out, int64_t *count_out, double *bytes_out)
{
    if (!ctx) return GMG_EINVAL;
    gmg_status st = check_ready(ctx);
    if (st) return st;
    if (n_cycles < 1 || n_cycles + 1 > ctx->hist_cap) { ctx->err = "n_cycles out of range"; return GMG_EINVAL; }
    ctx->prof.on = true;
    ctx->prof.ev.clear();
    ctx->prof.marks.clear();
    ctx->prof.bytes.clear();
    for (double &b : ctx->kbytes) b = 0;
    ctx->launches = 0;
    CK(cudaMemsetAsync(ctx->d_flag, 0, 3 * sizeof(int), ctx->stream));
    Launcher Lc{ctx, ctx->stream};
    for (int k = 0; k < n_cycles; ++k) {
        if (ctx->opt.dim == 2) vcycle_dispatch<2>(Lc);
        else vcycle_dispatch<3>(Lc);
    }
    ctx->prof.on = false;
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    double ms[GMG_K_COUNT] = {0};
    int64_t cnt[GMG_K_COUNT] = {0};
    FILE *dump = nullptr;   // dev aid: per-launch (class, ms, algorithmic bytes)
    if (const char *e = std::getenv("GMG_PROF_DUMP")) dump = std::fopen(e, "w");
    for (size_t q = 0; q < ctx->prof.marks.size(); ++q) {
        const auto &m = ctx->prof.marks[q];
        float t = 0.f;
        cudaEventElapsedTime(&t, ctx->prof.ev[m.second], ctx->prof.ev[m.second + 1]);
        ms[m.first] += t;
        cnt[m.first] += 1;
        if (dump) std::fprintf(dump, "%d %.6f %.0f\n", m.first, t, ctx->prof.bytes[q]);
    }
    if (dump) std::fclose(dump);
    ctx->prof.bytes.clear();
    for (auto e : ctx->prof.ev) cudaEventDestroy(e);
    ctx->prof.ev.clear();
    ctx->prof.marks.clear();
    for (int k = 0; k < GMG_K_COUNT; ++k) {
        if (ms_out) ms_out[k] = ms[k];
        if (count_out) count_out[k] = cnt[k];
        if (bytes_out) bytes_out[k] = ctx->kbytes[k];
    }
    return GMG_OK;
}

gmg_status gmg_time_smooth(gmg_ctx *ctx, int level, int n_sweeps, int reps, double *ms, double *cell_updates,
                           double *bytes)
{
    if (!ctx) return GMG_EINVAL;
    gmg_status st = check_ready(ctx, false);
    if (st) return st;
    if (level < 0 || level >= (int)ctx->lv.size() || n_sweeps < 1 || reps < 1) { ctx->err = "bad args"; return GMG_EINVAL; }
    cudaStream_t cs;
    CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    Launcher Lc{ctx, cs};
    for (double &b : ctx->kbytes) b = 0;
    cudaGraph_t g;
    cudaGraphExec_t ge;
    // the launches of the V-cycle's smoothing step on this level, unchanged: the last backward half-sweep
    // also writes W = W_lin + dW (the level's W is an output of the step, rewritten by every V-cycle)
    auto rhs = [](DevLevel &L) { return (const double *)L.Rt; };
    auto wout = [](DevLevel &L) { return L.W; };
    CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    if (ctx->opt.dim == 2) enqueue_sweeps<2>(Lc, level, n_sweeps, rhs, wout);
    else enqueue_sweeps<3>(Lc, level, n_sweeps, rhs, wout);
    CK(cudaStreamEndCapture(cs, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    cudaGraphDestroy(g);
    const double b1 = ctx->kbytes[GMG_K_SWEEP];
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    CK(cudaGraphLaunch(ge, ctx->stream));   // warm-up
    CK(cudaEventRecord(e0, ctx->stream));
    for (int r = 0; r < reps; ++r) CK(cudaGraphLaunch(ge, ctx->stream));
    CK(cudaEventRecord(e1, ctx->stream));
    CK(cudaEventSynchronize(e1));
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaGraphExecDestroy(ge);
    cudaStreamDestroy(cs);
    int64_t nown = 0;
    for (Domain &dm : ctx->dom) nown += dm.lv[level].n_own;
    if (ms) *ms = t;
    if (cell_updates) *cell_updates = (double)nown * 2.0 * n_sweeps * reps;
    if (bytes) *bytes = b1 * reps;
    return GMG_OK;
}

int64_t gmg_vcycle_launches(gmg_ctx *ctx)
{
    if (!ctx) return -1;
    if (!ctx->graph && check_ready(ctx) == GMG_OK) build_graph(ctx);
    return ctx->graph_launches;
}

gmg_status gmg_partition_rcb(int64_t n_cells, int dim, const double *centroid, int nparts, int32_t *part_out)
{
    if (n_cells < 1 || (dim != 2 && dim != 3) || !centroid || nparts < 1 || !part_out) return GMG_EINVAL;
    partition_rcb(n_cells, dim, centroid, nparts, part_out);
    return GMG_OK;
}

gmg_status gmg_p2p_layout(gmg_ctx *ctx, int64_t *out)
{
    if (!ctx || !out) return GMG_EINVAL;
    if (!ctx->ws_ready && !ctx->ws) { ctx->err = "workspace not set"; return GMG_ESTATE; }
    const int nl = (int)ctx->lv.size();
    const Domain &dm = ctx->dom[0];
    for (int l = 0; l < nl; ++l) out[l] = (int64_t)((const char *)dm.dv[l].rec - (const char *)ctx->ws);
    out[nl] = (int64_t)((const char *)dm.dv[0].p2p_flags - (const char *)ctx->ws);
    return GMG_OK;
}

gmg_status gmg_get_p2p_targets(gmg_ctx *ctx, int level, int dom, int64_t *n_targets, int32_t *off,
                               int32_t *peer_slot, int32_t *ghost_local)
{
    if (!ctx) return GMG_EINVAL;
    if (!ctx->built) { ctx->err = "hierarchy not built"; return GMG_ESTATE; }
    if (level < 0 || level >= (int)ctx->lv.size() || dom < 0 || dom >= (int)ctx->dom.size()) {
        ctx->err = "bad level / domain";
        return GMG_EINVAL;
    }
    const DomLevel &H = ctx->dom[dom].lv[level];
    if (!ctx->p2p || ctx->nparts < 2 || H.p2p_off.empty()) { ctx->err = "no P2P targets (GMG_P2P=1, > 1 partition)"; return GMG_ESTATE; }
    if (n_targets) *n_targets = (int64_t)H.p2p_k.size();
    if (off && peer_slot && ghost_local) {
        std::copy(H.p2p_off.begin(), H.p2p_off.end(), off);
        std::copy(H.p2p_k.begin(), H.p2p_k.end(), peer_slot);
        std::copy(H.p2p_g.begin(), H.p2p_g.end(), ghost_local);
    }
    return GMG_OK;
}

gmg_status gmg_p2p_import(gmg_ctx *ctx, const void *handles, const int64_t *base_off, const int64_t *layouts)
{
    if (!ctx || !handles || !base_off || !layouts) return GMG_EINVAL;
    if (!ctx->ws) { ctx->err = "workspace not set"; return GMG_ESTATE; }
    if (ctx->opt.nranks < 2 || !ctx->p2p) { ctx->err = "P2P import needs nranks > 1 and GMG_P2P=1"; return GMG_ESTATE; }
    CK(cudaSetDevice(ctx->opt.device));
    const int nl = (int)ctx->lv.size(), me = ctx->opt.rank;
    Domain &dm = ctx->dom[0];
    std::vector<char *> base(ctx->opt.nranks, nullptr);
    for (int l = 0; l < nl; ++l)
        for (int q : dm.lv[l].peers) {
            if (base[q]) continue;
            cudaIpcMemHandle_t h;
            std::memcpy(&h, (const char *)handles + 64 * (size_t)q, sizeof(h));
            void *p = nullptr;
            const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) {
                ctx->err = std::string("cudaIpcOpenMemHandle (rank ") + std::to_string(q) + "): " + cudaGetErrorString(e);
                return GMG_ECUDA;
            }
            ctx->p2p_opened.push_back(p);
            base[q] = (char *)p + base_off[q];
        }
    for (int l = 0; l < nl; ++l) {
        const DomLevel &H = dm.lv[l];
        std::vector<double *> pr(H.peers.size());
        std::vector<int *> sg(H.peers.size());
        for (size_t k = 0; k < H.peers.size(); ++k) {
            const int q = H.peers[k];
            const int64_t *lay = layouts + (size_t)q * (nl + 1);
            pr[k] = (double *)(base[q] + lay[l]);
            sg[k] = (int *)(base[q] + lay[nl]) + me;
        }
        if (!pr.empty()) {
            CK(cudaMemcpy(dm.dv[l].peer_rec, pr.data(), pr.size() * sizeof(double *), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dm.dv[l].p2p_sig, sg.data(), sg.size() * sizeof(int *), cudaMemcpyHostToDevice));
        }
    }
    ctx->p2p_ready = true;
    if (ctx->graph) { cudaGraphExecDestroy(ctx->graph); ctx->graph = nullptr; }
    return GMG_OK;
}

gmg_status gmg_get_halo(gmg_ctx *ctx, int level, int dom, int64_t *n_owned, int64_t *n_ghost, int *n_peers,
                        int64_t *n_send, int64_t *n_recv, int64_t *owned, int64_t *ghost, int32_t *peers,
                        int64_t *send_nat, int64_t *send_off, int64_t *recv_nat, int64_t *recv_off)
{
    if (!ctx) return GMG_EINVAL;
    if (!ctx->built) { ctx->err = "hierarchy not built"; return GMG_ESTATE; }
    if (level < 0 || level >= (int)ctx->lv.size() || dom < 0 || dom >= (int)ctx->dom.size()) {
        ctx->err = "bad level / domain";
        return GMG_EINVAL;
    }
    const DomLevel &H = ctx->dom[dom].lv[level];
    if (n_owned) *n_owned = H.n_own;
    if (n_ghost) *n_ghost = H.n_loc - H.n_own;
    if (n_peers) *n_peers = (int)H.peers.size();
    if (n_send) *n_send = (int64_t)H.send_idx.size();
    if (n_recv) *n_recv = (int64_t)H.recv_idx.size();
    if (owned && ghost && peers && send_nat && send_off && recv_nat && recv_off) {
        std::copy(H.l2n.begin(), H.l2n.begin() + H.n_own, owned);
        std::copy(H.l2n.begin() + H.n_own, H.l2n.end(), ghost);
        std::copy(H.peers.begin(), H.peers.end(), peers);
        for (size_t k = 0; k < H.send_idx.size(); ++k) send_nat[k] = H.l2n[H.send_idx[k]];
        for (size_t k = 0; k < H.recv_idx.size(); ++k) recv_nat[k] = H.l2n[H.recv_idx[k]];
        std::copy(H.send_off.begin(), H.send_off.end(), send_off);
        std::copy(H.recv_off.begin(), H.recv_off.end(), recv_off);
    }
    return GMG_OK;
}

const char *gmg_last_error(gmg_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

// ---------------------------------------------------------------- NEXT-1
gmg_status gmg_load_ho_geometry(gmg_ctx *ctx, const double *m2, int G, const double *gp, const double *gw)
{
    if (!ctx) return GMG_EINVAL;
    if (!ctx->mesh_loaded) { ctx->err = "gmg_load_ho_geometry before gmg_load_mesh"; return GMG_ESTATE; }
    if (ctx->ws_ready) { ctx->err = "gmg_load_ho_geometry after gmg_set_workspace"; return GMG_ESTATE; }
    const int d = ctx->opt.dim;
    if (!m2 || !gp || !gw || G != (d == 3 ? 4 : 2)) { ctx->err = "ho geometry: null pointer or G != 4 (3D) / 2 (2D)"; return GMG_EINVAL; }
    const HostLevel &L0 = ctx->lv[0];
    const int64_t n = L0.n, nf = L0.nf;
    const int nq = d * (d + 1) / 2;
    delete ctx->ho;
    ctx->ho = new HoHost;
    ctx->ho->G = G;
    ctx->ho->m2.assign(m2, m2 + (size_t)nq * n);
    ctx->ho->gp.assign(gp, gp + (size_t)d * G * nf);
    ctx->ho->gw.assign(gw, gw + (size_t)G * nf);
    return GMG_OK;
}

static gmg_status ho_ready(gmg_ctx *ctx, bool need_state)
{
    gmg_status st = check_ready(ctx, need_state);
    if (st) return st;
    if (!ctx->ho || !ctx->ho->prepared) { ctx->err = "no high-order geometry (gmg_load_ho_geometry)"; return GMG_ESTATE; }
    return GMG_OK;
}

gmg_status gmg_set_ho_state(gmg_ctx *ctx, const double *G, const double *alpha)
{
    if (!ctx) return GMG_EINVAL;
    gmg_status st = ho_ready(ctx, false);
    if (st) return st;
    const int d = ctx->opt.dim, nvd = (d + 2) * d;
    if (G) { st = put_natural(ctx, 0, G, nvd, [](DevLevel &L) { return L.ho.G_; }, true); if (st) return st; }
    else
        for (Domain &dm : ctx->dom)
            k_fill<<<nblk((int64_t)dm.dv[0].n_loc * nvd), 256, 0, ctx->stream>>>(dm.dv[0].n_loc * nvd, dm.dv[0].ho.G_, 0.0);
    if (alpha) { st = put_natural(ctx, 0, alpha, 1, [](DevLevel &L) { return L.ho.alpha; }, false); if (st) return st; }
    else
        for (Domain &dm : ctx->dom) k_fill<<<nblk(dm.dv[0].n), 256, 0, ctx->stream>>>(dm.dv[0].n, dm.dv[0].ho.alpha, 1.0);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    return GMG_OK;
}

gmg_status gmg_get_ho_state(gmg_ctx *ctx, double *G_out, double *alpha_out)
{
    if (!ctx) return GMG_EINVAL;
    gmg_status st = ho_ready(ctx, false);
    if (st) return st;
    const int d = ctx->opt.dim;
    if (G_out) { st = get_natural(ctx, 0, [](DevLevel &L) { return (const double *)L.ho.G_; }, (d + 2) * d, G_out); if (st) return st; }
    if (alpha_out) { st = get_natural(ctx, 0, [](DevLevel &L) { return (const double *)L.ho.alpha; }, 1, alpha_out); if (st) return st; }
    return GMG_OK;
}

gmg_status gmg_ho_residual(gmg_ctx *ctx, double *R_out, double *G_out, double *alpha_out, double *sigma_out)
{
    if (!ctx) return GMG_EINVAL;
    gmg_status st = ho_ready(ctx, true);
    if (st) return st;
    Launcher Lc{ctx, ctx->stream};
    if (ctx->opt.dim == 2) enqueue_ho_eval<2>(Lc, HO_OUT, &DevLevel::Rt, &DevLevel::tmp);
    else enqueue_ho_eval<3>(Lc, HO_OUT, &DevLevel::Rt, &DevLevel::tmp);
    CK(cudaGetLastError());
    const int d = ctx->opt.dim, nv = d + 2;
    if (R_out) { st = get_natural(ctx, 0, [](DevLevel &L_) { return (const double *)L_.Rt; }, nv, R_out); if (st) return st; }
    if (G_out) { st = get_natural(ctx, 0, [](DevLevel &L_) { return (const double *)L_.ho.Gout; }, nv * d, G_out); if (st) return st; }
    if (alpha_out) { st = get_natural(ctx, 0, [](DevLevel &L_) { return (const double *)L_.tmp; }, 1, alpha_out); if (st) return st; }
    if (sigma_out) { st = get_natural(ctx, 0, [](DevLevel &L_) { return (const double *)L_.sigma; }, 1, sigma_out); if (st) return st; }
    CK(cudaStreamSynchronize(ctx->stream));
    return GMG_OK;
}

gmg_status gmg_ho_recon(gmg_ctx *ctx, double *poly_out, int32_t *flags_out)
{
    if (!ctx) return GMG_EINVAL;
    gmg_status st = ho_ready(ctx, true);
    if (st) return st;
    Launcher Lc{ctx, ctx->stream};
    if (ctx->opt.dim == 2) enqueue_ho_eval<2>(Lc, 0, nullptr, nullptr, true);
    else enqueue_ho_eval<3>(Lc, 0, nullptr, nullptr, true);
    CK(cudaGetLastError());
    const int d = ctx->opt.dim, nv = d + 2, nc = 1 + d + d * (d + 1) / 2;
    if (poly_out) { st = get_natural(ctx, 0, [](DevLevel &L) { return (const double *)L.ho.poly; }, nv * nc, poly_out); if (st) return st; }
    if (flags_out) {
        for (Domain &dm : ctx->dom) {
            const DomLevel &D0 = dm.lv[0];
            std::vector<int> fl(D0.n_own);
            CK(cudaMemcpyAsync(fl.data(), dm.dv[0].ho.flags, fl.size() * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
            for (int64_t i = 0; i < D0.n_own; ++i) flags_out[D0.l2n[i]] = fl[i];
        }
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return GMG_OK;
}

void gmg_destroy(gmg_ctx *ctx)
{
    if (!ctx) return;
    if (ctx->graph) cudaGraphExecDestroy(ctx->graph);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    if (ctx->copy) {
        cudaStreamSynchronize(ctx->copy);
        cudaStreamSynchronize(ctx->copy_out);
        cudaStreamDestroy(ctx->copy);
        cudaStreamDestroy(ctx->copy_out);
        for (int k = 0; k < 2; ++k) {
            cudaEventDestroy(ctx->ev_in_ready[k]);
            cudaEventDestroy(ctx->ev_in_free[k]);
            cudaEventDestroy(ctx->ev_out_ready[k]);
            cudaEventDestroy(ctx->ev_out_free[k]);
        }
    }
    if (ctx->nccl_comm && nccl().CommDestroy) nccl().CommDestroy((ncclComm_t)ctx->nccl_comm);
    for (void *p : ctx->p2p_opened) cudaIpcCloseMemHandle(p);
    delete ctx->ho;
    delete ctx;
}

}  // extern "C"
