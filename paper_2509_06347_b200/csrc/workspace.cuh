// workspace.cuh -- internal to api.cu (included once, inside its anonymous
// namespace): carving of the single device workspace per domain and level,
// the algorithmic byte counts of every launch, the host ->
// device upload of the setup, and the V-cycle dispatch.
#pragma once
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
            L.wlin = b.take<double>((size_t)nv * nloc);   // state arrays, Wp<D> layout
            L.wp = b.take<double>((size_t)nv * nloc);
            L.xr = b.take<double>((size_t)kXr * n);
            L.dc = b.take<double>((size_t)2 * n);
            L.tmp = b.take<double>(n);
            L.Rs = b.take<double>((size_t)nv * n); L.F = b.take<double>((size_t)nv * n);
            L.alpha = b.take<double>(n); L.sigma = b.take<double>(n);
            L.deg_int = b.take<uint8_t>(n); L.deg_all = b.take<uint8_t>(n);
            L.gord = b.take<int>(n);
            L.gface = b.take<int>(H.ng_entries);
            L.sinfo = b.take<int2>(n);
            L.fslot = b.take<int2>(nf);
            L.npeer = (int)H.peers.size();
            L.p2p_off = b.take<int>(H.p2p_off.size());
            L.p2p_k = b.take<int>(H.p2p_k.size());
            L.p2p_g = b.take<int>(H.p2p_g.size());
            L.peer_wp = b.take<double *>(H.peers.size());
            L.peer_nloc = b.take<int>(H.peers.size());
            L.p2p_sig = b.take<int *>(H.peers.size());
            L.p2p_wait = b.take<int>(H.peers.size());
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
            V.nlane = (int)(H.glane.size() / 2);
            V.glane = b.take<int2>(V.nlane);
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
            // face data (A, S r) once per face + 4 B per slot.  First forward half-sweep: only the
            // neighbours of earlier colors (and ghosts of earlier colors) carry an increment, so only
            // their slots and their share of the neighbour term are charged
            B.sweep.assign(ncolor, 0.0);
            B.sweep_ff.assign(ncolor, 0.0);
            B.sweep_out.assign(ncolor, 0.0);
            B.visits.assign(ncolor, 0);
            const std::vector<int32_t> &gcol = ctx->lv[l].color;
            for (int c = 0; c < ncolor; ++c) {
                double s = 0, sf = 0;
                for (int64_t i = H.blk[c]; i < H.blk[c + 1]; ++i) {
                    s += (2 * nv * 8 + 16) + 2 * nv * 8 + H.deg_int[i] * ((d + 1) * 8 / 2.0 + 4);
                    int lower = 0;
                    for (int32_t e = H.soffc[i]; e < H.soffc[i + 1]; ++e) {
                        const int32_t j = H.sJe[e];
                        lower += j < H.n_own ? (j < H.blk[c]) : (gcol[H.l2n[j]] - 1 < c);
                    }
                    sf += (2 * nv * 8 + 16) + (H.deg_int[i] ? 2 * nv * 8 * (double)lower / H.deg_int[i] : 0.0) +
                          lower * ((d + 1) * 8 / 2.0 + 4);
                }
                B.sweep[c] = s;
                B.sweep_ff[c] = sf;
                B.sweep_out[c] = (double)(H.blk[c + 1] - H.blk[c]) * 2 * nv * 8;
                B.visits[c] = H.blk[c + 1] - H.blk[c];
            }
            B.restrict_ = l > 0 ? (double)dm.lv[l - 1].n_own * (2 * nv * 8 + 16) + (double)H.n_own * (3 * nv * 8 + 16) : 0;
            B.prolong = (double)H.n_own * (2 * nv * 8 + 8 + 4) + (nl > 1 ? (double)dm.lv[1].n_own * (2 * nv * 8 + 12) : 0) +
                        (nl > 2 ? (double)dm.lv[2].n_own * 2 * nv * 8 : 0);
            B.update = (double)H.n_own * 3 * nv * 8;
        }
    }
}

template <int D>
void vcycle_dispatch(Launcher &Lc) { enqueue_vcycle<D>(Lc); }
