// launch.cuh -- internal to api.cu (included once, inside its anonymous
// namespace): run-time NCCL, launch bookkeeping, and the kernel orchestration
// of the residual, smoothing, halo exchange and V-cycle (enqueued on a stream
// or captured into the V-cycle CUDA graph).
#pragma once

inline int nblk(int64_t n, int b = 256) { return (int)std::max<int64_t>(1, (n + b - 1) / b); }

// one domain on one rank: the residual-norm sums need no combination, so the
// reduction kernel writes the history entry itself (one launch less)
inline bool norm_fused(const gmg_ctx *ctx) { return ctx->dom.size() == 1 && ctx->opt.nranks == 1; }

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
    if (ctx->opt.pdl) {
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
    }
    cudaLaunchKernelEx(&cfg, k, args...);
}

// prep: the launch also writes the sweep slot records (A outward | S r) of
// both cells of every interior face (whole 32-byte records).  from_rec: W is
// a W_lin state array (Wp<D> layout), else a W array (stride nv)
template <int D>
void enqueue_face(Launcher &Lc, Domain &dm, int l, const double *W, bool flux, bool from_rec, bool df = false,
                  bool prep = false, bool sr = true)
{
    gmg_ctx *ctx = Lc.ctx;
    DevLevel &L = dm.dv[l];
    constexpr int RS = 0, NV = D + 2;   // RS: the state-array layout (k_face STRIDE 0)
    Lc.pre(GMG_K_FACE);
    const dim3 g(nblk(L.nf)), b(256);
    const Phys ph = phys(ctx);
    const BCs bc = bcs(ctx);
    if (prep) {
        if (flux && df && !from_rec) klaunch(ctx, k_face<D, true, NV, true, true>, g, b, Lc.s, L, W, ph, bc, (int)sr);
        else if (flux && !df && from_rec) klaunch(ctx, k_face<D, true, RS, false, true>, g, b, Lc.s, L, W, ph, bc, (int)sr);
        else if (flux && !df && !from_rec) klaunch(ctx, k_face<D, true, NV, false, true>, g, b, Lc.s, L, W, ph, bc, (int)sr);
        else if (!flux && from_rec) klaunch(ctx, k_face<D, false, RS, false, true>, g, b, Lc.s, L, W, ph, bc, (int)sr);
        else if (!flux && !from_rec) klaunch(ctx, k_face<D, false, NV, false, true>, g, b, Lc.s, L, W, ph, bc, (int)sr);
        else { ctx->err = "enqueue_face: unsupported prep variant"; return; }
    } else if (flux && df) {
        if (from_rec) klaunch(ctx, k_face<D, true, RS, true, false>, g, b, Lc.s, L, W, ph, bc, (int)sr);
        else klaunch(ctx, k_face<D, true, NV, true, false>, g, b, Lc.s, L, W, ph, bc, (int)sr);
    } else if (flux) {
        if (from_rec) klaunch(ctx, k_face<D, true, RS, false, false>, g, b, Lc.s, L, W, ph, bc, (int)sr);
        else klaunch(ctx, k_face<D, true, NV, false, false>, g, b, Lc.s, L, W, ph, bc, (int)sr);
    } else {
        if (from_rec) klaunch(ctx, k_face<D, false, RS, false, false>, g, b, Lc.s, L, W, ph, bc, (int)sr);
        else klaunch(ctx, k_face<D, false, NV, false, false>, g, b, Lc.s, L, W, ph, bc, (int)sr);
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
    const dim3 g(nblk(L.n)), b(256);
    switch (flags) {   // the V-cycle's combinations as compile-time flag sets
        case G_FLUX | G_NORM | G_EXPLICIT: klaunch(Lc.ctx, k_gather<D, G_FLUX | G_NORM | G_EXPLICIT>, g, b, Lc.s, L, a); break;
        case G_FLUX | G_WRITE_RT | G_ALPHA: klaunch(Lc.ctx, k_gather<D, G_FLUX | G_WRITE_RT | G_ALPHA>, g, b, Lc.s, L, a); break;
        case G_FLUX | G_SET_F | G_PREPARE: klaunch(Lc.ctx, k_gather<D, G_FLUX | G_SET_F | G_PREPARE>, g, b, Lc.s, L, a); break;
        case G_FLUX | G_WRITE_RT | G_ADD_F: klaunch(Lc.ctx, k_gather<D, G_FLUX | G_WRITE_RT | G_ADD_F>, g, b, Lc.s, L, a); break;
        case G_PREPARE: klaunch(Lc.ctx, k_gather<D, G_PREPARE>, g, b, Lc.s, L, a); break;
        default: klaunch(Lc.ctx, k_gather<D, -1>, g, b, Lc.s, L, a); break;
    }
    Lc.post(GMG_K_GATHER, dm.lbytes[l].gather);
    if (flags & G_NORM) {
        Lc.pre(GMG_K_NORM);
        klaunch(Lc.ctx, k_norm_sum, dim3(1), dim3(1024), Lc.s, L.partial, nblk(L.n), L.nv, ctx->d_sumsq + (size_t)di * L.nv,
                ctx->d_hist, ctx->hist_cap, ctx->d_flag, (int)norm_fused(ctx));
        Lc.post(GMG_K_NORM, (double)nblk(L.n) * L.nv * 8);
    }
}

// all-reduce the per-domain sums across ranks, then one history entry
void enqueue_norm_hist(Launcher &Lc)
{
    gmg_ctx *ctx = Lc.ctx;
    if (norm_fused(ctx)) return;   // k_norm_sum already wrote the history entry
    const int nv = ctx->opt.dim + 2;
    if (ctx->opt.nranks > 1)
        nccl().AllReduce(ctx->d_sumsq, ctx->d_sumsq, nv, ncclDouble, ncclSum, (ncclComm_t)ctx->nccl_comm, Lc.s);
    Lc.pre(GMG_K_NORM);
    klaunch(Lc.ctx, k_norm_hist, dim3(1), dim3(32), Lc.s, ctx->d_sumsq, (int)ctx->dom.size(), nv, ctx->d_hist, ctx->hist_cap, ctx->d_flag);
    Lc.post(GMG_K_NORM, 0.0);
}

// --------------------------------------------------------------------------
// halo exchange (a13).  kind: the W' of one color (after its sweep phase),
// W_lin of all colors (the ghosts' W' set to it), or the state W of all colors.
// --------------------------------------------------------------------------
enum { EX_WP = 0, EX_WLIN = 1, EX_W = 2 };

template <int D>
void enqueue_exchange(Launcher &Lc, int l, int kind, int color)
{
    gmg_ctx *ctx = Lc.ctx;
    if (ctx->nparts <= 1) return;
    constexpr int NV = D + 2;
    const int ncolor = ctx->lv[l].ncolor;
    const int stride = kind == EX_W ? NV : 4, offset = 0;
    auto split_of = [&](DevLevel &L) { return (kind != EX_W && D == 3) ? L.n_loc : 0; };
    auto src_of = [&](DevLevel &L) { return kind == EX_W ? L.W : kind == EX_WLIN ? L.wlin : L.wp; };
    auto dst2_of = [&](DevLevel &L) { return kind == EX_WLIN ? L.wp : (double *)nullptr; };
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
            Lc.pre(GMG_K_HALO);
            klaunch(Lc.ctx, k_pack, dim3(nblk(s1 - s0)), dim3(256), Lc.s, (int)(s1 - s0), L.send_idx + s0, src_of(L), stride, offset, NV,
                                                   L.sendbuf + s0 * NV, split_of(L));
            Lc.post(GMG_K_HALO, (double)(s1 - s0) * NV * 16);
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
            Lc.pre(GMG_K_HALO);
            klaunch(Lc.ctx, k_unpack, dim3(nblk(r1 - r0)), dim3(256), Lc.s, (int)(r1 - r0), L.recv_idx + r0, L.recvbuf + r0 * NV,
                                                     src_of(L), stride, offset, NV, dst2_of(L), split_of(L));
            Lc.post(GMG_K_HALO, (double)(r1 - r0) * NV * (kind == EX_WLIN ? 24 : 16));
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
            Lc.pre(GMG_K_HALO);
            klaunch(Lc.ctx, k_ghost_wlin<D>, dim3(nblk(L.n_loc - L.n)), dim3(256), Lc.s, L.n, L.n_loc, L.W, L.wlin, L.wp);
            Lc.post(GMG_K_HALO, (double)(L.n_loc - L.n) * (D + 2) * 24);
        }
    }
}

template <int D>
void enqueue_ghost_w(Launcher &Lc, int l)
{
    for (Domain &dm : Lc.ctx->dom) {
        DevLevel &L = dm.dv[l];
        if (L.n_loc > L.n) {
            Lc.pre(GMG_K_HALO);
            klaunch(Lc.ctx, k_ghost_w<D>, dim3(nblk(L.n_loc - L.n)), dim3(256), Lc.s, L.n, L.n_loc, L.wp, L.W);
            Lc.post(GMG_K_HALO, (double)(L.n_loc - L.n) * (D + 2) * 16);
        }
    }
}

// --------------------------------------------------------------------------
// sweeps
// --------------------------------------------------------------------------
// optional persisting-L2 access-policy window over the level's W' records
// (the gathered data), attached per launch so that graph capture keeps it
template <class K>
void launch_with_window(K kernel, dim3 g, dim3 b, cudaStream_t s, const SweepArgs &a, const void *win, size_t win_bytes,
                        bool pdl)
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
        at[na].val.accessPolicyWindow.hitRatio = 1.0f;
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

// lanes per cell of a color block: the configured lanes for large blocks; a
// block that still fits one resident wave at twice the lanes gets them (up to
// 16) -- small trailing colors are latency chains of ceil(deg/LPC) gathers
#ifndef GMG_MAX_LPC
#define GMG_MAX_LPC 16
#endif
constexpr int kMaxLpc = GMG_MAX_LPC;
int sweep_lpc(const gmg_ctx *ctx, int64_t cells)
{
    int lpc = ctx->lpc;
    if (ctx->adapt_lpc && ctx->sweep_grid_cap > 0) {
        const int64_t wave = (int64_t)ctx->sweep_grid_cap * 128;
        while (lpc < kMaxLpc && cells * lpc * 2 <= wave) lpc *= 2;
    }
    return lpc;
}

template <int D, int LPC, bool FF>
void launch_sweep_lpc(const gmg_ctx *ctx, const SweepArgs &a, cudaStream_t s, const void *win, size_t win_bytes)
{
    const int64_t nthreads = (int64_t)(a.cend - a.cbeg) * LPC;
    int nb = (int)((nthreads + 127) / 128);
    if (FF && a.lo == 0 && a.n_own == a.n_loc) {   // first color, no ghosts: no W' gathers
        const int cap = ctx->sweep_grid_cap_ff1;
        if (cap > 0) nb = std::min(nb, cap);
        if (a.Wout)
            launch_with_window(k_sweep<D, LPC, 2, 1>, dim3(std::max(nb, 1)), dim3(128), s, a, win, win_bytes,
                               ctx->opt.pdl != 0);
        else
            launch_with_window(k_sweep<D, LPC, 2, 0>, dim3(std::max(nb, 1)), dim3(128), s, a, win, win_bytes,
                               ctx->opt.pdl != 0);
        return;
    }
    const int cap = FF ? ctx->sweep_grid_cap_ff : ctx->sweep_grid_cap;
    if (cap > 0) nb = std::min(nb, cap);
    if (a.Wout)   // the last backward phase also writes W
        launch_with_window(k_sweep<D, LPC, FF ? 1 : 0, 1>, dim3(std::max(nb, 1)), dim3(128), s, a, win, win_bytes,
                           ctx->opt.pdl != 0);
    else
        launch_with_window(k_sweep<D, LPC, FF ? 1 : 0, 0>, dim3(std::max(nb, 1)), dim3(128), s, a, win, win_bytes,
                           ctx->opt.pdl != 0);
}

template <int D, bool FF>
void launch_sweep(const gmg_ctx *ctx, const SweepArgs &a, int lpc, cudaStream_t s, const void *win, size_t win_bytes)
{
    switch (lpc) {
        case 1: launch_sweep_lpc<D, 1, FF>(ctx, a, s, win, win_bytes); break;
        case 4: launch_sweep_lpc<D, 4, FF>(ctx, a, s, win, win_bytes); break;
        case 8: launch_sweep_lpc<D, 8, FF>(ctx, a, s, win, win_bytes); break;
        case 16: launch_sweep_lpc<D, 16, FF>(ctx, a, s, win, win_bytes); break;
        default: launch_sweep_lpc<D, 2, FF>(ctx, a, s, win, win_bytes); break;
    }
}

SweepArgs sweep_args(const gmg_ctx *ctx, DevLevel &L, const DomLevel &H, int c, int b0, int b1, const double *rhs,
                     double *Wout)
{
    SweepArgs a;
    a.cbeg = b0;
    a.cend = b1;
    a.lo = c >= 0 ? (int)H.blk[c] : 0;
    a.n_own = (int)H.n_own;
    a.n_loc = (int)H.n_loc;
    a.gm1 = ctx->opt.gamma - 1.0;
    a.sinfo = L.sinfo;
    a.sJe = L.sJe;
    a.sRe = L.sRe;
    a.wp = L.wp;
    a.xr = L.xr;
    a.wlin = L.wlin;
    a.rhs = rhs;
    a.dc = L.dc;
    a.Wout = Wout;
    a.rev = 0;
    return a;
}

// one color block of one domain (Eq.(gpu-forward-relaxation) / (gpu-backward-relaxation))
// part: 0 = whole block, 1 = its boundary cells (ghost neighbours), 2 = its interior cells
// ff: a phase of the first forward half-sweep of a smoothing step (k_sweep<.., FF>)
template <int D>
void enqueue_sweep_color(Launcher &Lc, Domain &dm, int l, int c, const double *rhs, double *Wout, int part, bool ff,
                         bool rev = false)
{
    gmg_ctx *ctx = Lc.ctx;
    DevLevel &L = dm.dv[l];
    const DomLevel &H = dm.lv[l];
    int b0 = (int)H.blk[c], b1 = (int)H.blk[c + 1];
    double frac = 1.0;
    if (part) {
        const int mid = b0 + (int)H.nbnd[c];
        frac = b1 > b0 ? (double)(part == 1 ? mid - b0 : b1 - mid) / (b1 - b0) : 0.0;
        if (part == 1) b1 = mid;
        else b0 = mid;
    }
    if (b1 <= b0) return;
    SweepArgs a = sweep_args(ctx, L, H, c, b0, b1, rhs, Wout);
    a.rev = rev ? 1 : 0;   // backward half-sweeps from the block's end: the cells swept last in the
                           // previous visit of this color come first, while their records are still in L2
    const void *win = ctx->l2_window ? (const void *)L.wp : nullptr;
    const size_t wb = ctx->l2_window ? std::min<size_t>(ctx->l2_window, (size_t)L.n_loc * (D + 2) * 8) : 0;
    const int lpc = part ? ctx->lpc : sweep_lpc(ctx, b1 - b0);
    Lc.pre(GMG_K_SWEEP);
    if (ff) launch_sweep<D, true>(ctx, a, lpc, Lc.s, win, wb);
    else launch_sweep<D, false>(ctx, a, lpc, Lc.s, win, wb);
    Lc.post(GMG_K_SWEEP, frac * ((ff ? dm.lbytes[l].sweep_ff[c] : dm.lbytes[l].sweep[c]) +
                                 (Wout ? dm.lbytes[l].sweep_out[c] : 0.0)));
    ctx->visits += (int64_t)(b1 - b0);
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
        const SweepArgs a = sweep_args(ctx, L, H, c, b0, b1, rhs(L), last ? wout(L) : nullptr);
        P2PArgs p{L.p2p_off, L.p2p_k, L.p2p_g, L.peer_wp, L.peer_nloc, L.npeer, L.p2p_wait, L.p2p_sig, L.p2p_flags, L.p2p_ctl};
        const int lpc = sweep_lpc(ctx, b1 - b0);
        int nb = nblk((int64_t)(b1 - b0) * lpc);
        if (ctx->sweep_grid_cap > 0) nb = std::min(nb, ctx->sweep_grid_cap / 2);
        const dim3 g(std::max(nb, 1)), b(256);
        Lc.pre(GMG_K_SWEEP);
#define GMG_P2P_LAUNCH(LP)                                                          \
    (ff ? k_sweep_p2p<D, LP, true><<<g, b, 0, Lc.s>>>(a, p)                         \
        : k_sweep_p2p<D, LP, false><<<g, b, 0, Lc.s>>>(a, p))
        switch (lpc) {
            case 1: GMG_P2P_LAUNCH(1); break;
            case 4: GMG_P2P_LAUNCH(4); break;
            case 8: GMG_P2P_LAUNCH(8); break;
            case 16: GMG_P2P_LAUNCH(16); break;
            default: GMG_P2P_LAUNCH(2); break;
        }
#undef GMG_P2P_LAUNCH
        Lc.post(GMG_K_SWEEP, c < 0 ? 0.0 : (ff ? dm.lbytes[l].sweep_ff[c] : dm.lbytes[l].sweep[c]) +
                                              (last ? dm.lbytes[l].sweep_out[c] : 0.0));
        ctx->visits += (int64_t)(b1 - b0);
    }
}

// Algorithm 2's phase list of one smoothing step: n_sweeps x
// (forward colors 1..Nc, backward Nc..1).  With skip_repeat a color phase
// that directly follows a phase of the SAME color (the turn of every forward
// -> backward and backward -> forward pass: c_N then c_N, c_1 then c_1) is
// dropped: a cell's update reads only other-colored neighbours, none of which
// changed in between, and never its own state -- so it would recompute
// identical values (its W write, if any, moves to the kept phase).  Exact,
// not an approximation: the oracle runs every phase.
struct Phase { int c; bool last; bool ff; bool rev; };
std::vector<Phase> phase_list(const gmg_ctx *ctx, int l, int n_sweeps)
{
    const int nc = ctx->lv[l].ncolor;
    std::vector<Phase> seq;
    for (int s = 0; s < n_sweeps; ++s)
        for (int half = 0; half < 2; ++half)
            for (int cc = 0; cc < nc; ++cc) {
                const Phase ph{half == 0 ? cc : nc - 1 - cc, (s == n_sweeps - 1) && half == 1, s == 0 && half == 0,
                               half == 1};
                if (ctx->opt.skip_repeat && !seq.empty() && seq.back().c == ph.c) seq.back().last |= ph.last;
                else seq.push_back(ph);
            }
    return seq;
}

// one smoothing step's sweeps; after every color its W' goes to the
// ranks/domains that ghost it.  rhs/wout select the domain's arrays: the first
// forward half-sweep reads rhs (with W_lin and 1/D, c) and the last backward
// half-sweep writes W = W' into wout.
template <int D>
void enqueue_sweeps(Launcher &Lc, int l, int n_sweeps, std::function<const double *(DevLevel &)> rhs,
                    std::function<double *(DevLevel &)> wout)
{
    gmg_ctx *ctx = Lc.ctx;
    const std::vector<Phase> seq = phase_list(ctx, l, n_sweeps);
    // fused P2P halo: states go to the ghosts from the sweep epilogue; a
    // synchronisation phase before (the ghosts' local initialisation is done)
    // and after (the peers' last states have landed) the step
    if (ctx->opt.p2p && ctx->p2p_ready && ctx->nparts > 1) {
        enqueue_p2p_phase<D>(Lc, l, -1, false, false, rhs, wout);
        for (const Phase &ph : seq) enqueue_p2p_phase<D>(Lc, l, ph.c, ph.last, ph.ff, rhs, wout);
        enqueue_p2p_phase<D>(Lc, l, -1, false, false, rhs, wout);
        return;
    }
    const bool overlap = (ctx->opt.overlap < 0 ? ctx->opt.nranks > 1 : ctx->opt.overlap != 0) && ctx->nparts > 1 && ctx->side;
    for (const Phase &ph : seq) {
        const int c = ph.c;
        if (overlap) {
            // boundary cells of color c first; their states travel on the side
            // stream while the interior cells of c (no ghost neighbours) are
            // swept; the next color waits for the ghosts (fork / join)
            for (Domain &dm : ctx->dom)
                enqueue_sweep_color<D>(Lc, dm, l, c, rhs(dm.dv[l]), ph.last ? wout(dm.dv[l]) : nullptr, 1, ph.ff);
            cudaEventRecord(ctx->ev_fork, Lc.s);
            cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0);
            Launcher Ls{ctx, ctx->side};
            enqueue_exchange<D>(Ls, l, EX_WP, c);
            cudaEventRecord(ctx->ev_join, ctx->side);
            for (Domain &dm : ctx->dom)
                enqueue_sweep_color<D>(Lc, dm, l, c, rhs(dm.dv[l]), ph.last ? wout(dm.dv[l]) : nullptr, 2, ph.ff);
            cudaStreamWaitEvent(Lc.s, ctx->ev_join, 0);
        } else {
            for (Domain &dm : ctx->dom)
                enqueue_sweep_color<D>(Lc, dm, l, c, rhs(dm.dv[l]), ph.last ? wout(dm.dv[l]) : nullptr, 0, ph.ff,
                                       ph.rev);
            enqueue_exchange<D>(Lc, l, EX_WP, c);
        }
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
            Lc.pre(GMG_K_HALO);
            klaunch(ctx, k_pack, dim3(nblk(s1)), dim3(256), Lc.s, (int)s1, L.send_idx, (const double *)(L.ho.*arr), ncomp, 0,
                    ncomp, dm.ho.sendbuf, 0);
            Lc.post(GMG_K_HALO, (double)s1 * ncomp * 16);
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
            Lc.pre(GMG_K_HALO);
            klaunch(ctx, k_unpack, dim3(nblk(r1)), dim3(256), Lc.s, (int)r1, L.recv_idx, (const double *)dm.ho.recvbuf,
                    L.ho.*arr, ncomp, 0, ncomp, (double *)nullptr, 0);
            Lc.post(GMG_K_HALO, (double)r1 * ncomp * 16);
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
            klaunch(Lc.ctx, k_norm_sum, dim3(1), dim3(1024), Lc.s, L.partial, nblk(L.n), L.nv, ctx->d_sumsq + di * L.nv,
                    ctx->d_hist, ctx->hist_cap, ctx->d_flag, (int)norm_fused(ctx));
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
                              G_FLUX | G_NORM | G_WRITE_RT | G_PREPARE | G_COPY_W | (df0 ? G_ALPHA : 0),
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
        enqueue_face<D>(Lc, doms[d], 0, doms[d].dv[0].W, true, false, df0, false, false);
        enqueue_gather<D>(Lc, doms[d], (int)d, 0, G_FLUX | G_WRITE_RT | (df0 ? G_ALPHA : 0), nullptr);
    }
    }
    // 4. coarse levels
    for (int l = 1; l < nl; ++l) {
        const bool last = (l == nl - 1);
        for (Domain &dm : doms) enqueue_restrict<D>(Lc, dm, l);                // W0, Res*, alpha, dW = 0
        enqueue_exchange<D>(Lc, l, EX_WLIN, -1);                                // ghosts' W0, dW = 0
        for (size_t d = 0; d < doms.size(); ++d) {
            enqueue_face<D>(Lc, doms[d], l, doms[d].dv[l].wlin, !last, true, false, true);   // R(W0) only if F is needed later
            enqueue_gather<D>(Lc, doms[d], (int)d, l, (last ? 0 : (G_FLUX | G_SET_F)) | G_PREPARE, nullptr);
        }
        enqueue_sweeps<D>(Lc, l, ctx->opt.n_sweeps, [](DevLevel &L) { return (const double *)L.Rs; },
                          [](DevLevel &L) { return L.W; });                      // RHS = Res* (A8)
        if (!last) {
            enqueue_ghost_w<D>(Lc, l);
            for (size_t d = 0; d < doms.size(); ++d) {
                enqueue_face<D>(Lc, doms[d], l, doms[d].dv[l].W, true, false, false, false, false);
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
        enqueue_face<D>(Lc, ctx->dom[d], 0, ctx->dom[d].dv[0].W, true, false, false, false, false);
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

// every domain's owned dW = W' - W_lin (or W_lin itself) -> natural SoA (gmg_smooth, gmg_get_level_field)
gmg_status get_dw_natural(gmg_ctx *ctx, int l, double *dst, bool wlin_only = false)
{
    const int64_t N = ctx->lv[l].n;
    const int ncomp = ctx->opt.dim + 2;
    if (ctx->opt.nranks > 1)
        CK(cudaMemcpyAsync(ctx->d_stage, dst, sizeof(double) * ncomp * N, cudaMemcpyDefault, ctx->stream));
    for (Domain &dm : ctx->dom) {
        DevLevel &L = dm.dv[l];
        k_state_to_natural<<<nblk(L.n), 256, 0, ctx->stream>>>(L.n, (int)N, ncomp, L.perm, wlin_only ? L.wlin : L.wp,
                                                               wlin_only ? nullptr : L.wlin, L.n_loc, ctx->d_stage);
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(dst, ctx->d_stage, sizeof(double) * ncomp * N, cudaMemcpyDefault, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return GMG_OK;
}
