// api.cu -- the C ABI of libgmg (include/gmg.h): context, options, workspace,
// data movement and the CUDA-graph capture of one V-cycle.  The kernel
// orchestration (residual / smoothing / halo exchange / V-cycle, run-time
// NCCL) is launch.cuh, the workspace carving and byte counts workspace.cuh --
// both internal fragments included once, below.
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
#include "p2p_emulate.cuh"

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

#include "launch.cuh"
#include "workspace.cuh"

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
    o->skip_repeat = 1;
    o->p2p = 0;
    o->overlap = -1;
    o->l2_persist_mb = 0;
    o->sweep_lanes = 2;
    o->pdl = 1;
    o->ho_p2min = 0;
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
        opt->setup_device < 0 || opt->setup_device > 1 || opt->skip_repeat < 0 || opt->skip_repeat > 1 ||
        opt->p2p < 0 || opt->p2p > 1 || opt->overlap < -1 || opt->overlap > 1 || opt->l2_persist_mb < 0 ||
        !(opt->sweep_lanes == 0 || opt->sweep_lanes == 1 || opt->sweep_lanes == 2 || opt->sweep_lanes == 4) ||
        opt->pdl < 0 || opt->pdl > 1 || opt->ho_p2min < 0)
        return GMG_EINVAL;
    gmg_ctx *ctx = new (std::nothrow) gmg_ctx();
    if (!ctx) return GMG_ENOMEM;
    ctx->opt = *opt;
    ctx->stream = (cudaStream_t)opt->stream;
    ctx->nparts = std::max(opt->nranks, opt->local_domains);
    ctx->lpc = opt->sweep_lanes ? opt->sweep_lanes : 2;
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
                build_domain_level(ctx->lv[l], dm.rank, dm.lv[l], ctx->nparts == 1);
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
        if (ctx->opt.p2p && ctx->nparts > 1) {   // fused P2P halo targets
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
            CK(up_raw(L.gord, H.gord.data(), H.gord.size() * sizeof(int)));
            CK(up_raw(L.gface, H.gface.data(), H.gface.size() * sizeof(int)));
            CK(up_raw(L.fslot, H.fslot.data(), H.fslot.size() * sizeof(int)));
            CK(up_raw(L.p2p_off, H.p2p_off.data(), H.p2p_off.size() * sizeof(int)));
            CK(up_raw(L.p2p_k, H.p2p_k.data(), H.p2p_k.size() * sizeof(int)));
            CK(up_raw(L.p2p_g, H.p2p_g.data(), H.p2p_g.size() * sizeof(int)));
            CK(up_raw(L.p2p_wait, H.peers.data(), H.peers.size() * sizeof(int)));
            {
                std::vector<int> si(2 * H.n_own);
                for (int64_t i = 0; i < H.n_own; ++i) { si[2 * i] = H.soffc[i]; si[2 * i + 1] = H.deg_int[i]; }
                CK(up_i((const int *)L.sinfo, std::move(si)));
                std::vector<int> gi(4 * H.n_own);
                for (int64_t t = 0; t < H.n_own; ++t) {
                    const int i = H.gord[t];
                    gi[4 * t] = H.gbase[i];
                    gi[4 * t + 1] = (int)H.deg_all[i] | ((int)H.deg_int[i] << 16);
                    gi[4 * t + 2] = i;
                    gi[4 * t + 3] = 0;
                }
                CK(up_i((const int *)L.ginfo, std::move(gi)));
            }
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
            CK(cudaMemsetAsync(L.wlin, 0, sizeof(double) * L.nv * H.n_loc, ctx->stream));
            CK(cudaMemsetAsync(L.wp, 0, sizeof(double) * L.nv * H.n_loc, ctx->stream));
            CK(cudaMemsetAsync(L.xr, 0, sizeof(double) * kXr * H.n_own, ctx->stream));
            CK(cudaMemsetAsync(L.dc, 0, sizeof(double) * 2 * H.n_own, ctx->stream));
        }
    }
    CK(cudaMemsetAsync(ctx->d_flag, 0, 4 * sizeof(int), ctx->stream));
    for (Domain &dm : ctx->dom) {   // P2P phase counts / control
        CK(cudaMemsetAsync(dm.dv[0].p2p_flags, 0, sizeof(int) * std::max(ctx->nparts, 1), ctx->stream));
        CK(cudaMemsetAsync(dm.dv[0].p2p_ctl, 0, sizeof(int) * 4, ctx->stream));
    }
    ctx->p2p_ready = false;
    if (ctx->opt.p2p && ctx->nparts > 1 && ctx->opt.nranks == 1) {   // local domains: peers are in this process
        CK(cudaStreamSynchronize(ctx->stream));
        for (Domain &dm : ctx->dom)
            for (int l = 0; l < nl; ++l) {
                const DomLevel &H = dm.lv[l];
                std::vector<double *> pr(H.peers.size());
                std::vector<int *> sg(H.peers.size());
                std::vector<int> pn(H.peers.size());
                for (size_t k = 0; k < H.peers.size(); ++k) {
                    DevLevel &Q = ctx->dom[H.peers[k]].dv[l];
                    pr[k] = Q.wp;
                    sg[k] = Q.p2p_flags + dm.rank;
                    pn[k] = Q.n_loc;
                }
                if (!pr.empty()) {
                    CK(cudaMemcpy(dm.dv[l].peer_nloc, pn.data(), pn.size() * sizeof(int), cudaMemcpyHostToDevice));
                    CK(cudaMemcpy(dm.dv[l].peer_wp, pr.data(), pr.size() * sizeof(double *), cudaMemcpyHostToDevice));
                    CK(cudaMemcpy(dm.dv[l].p2p_sig, sg.data(), sg.size() * sizeof(int *), cudaMemcpyHostToDevice));
                }
            }
        ctx->p2p_ready = true;
    }
    if (!ctx->copy) {                      // copy stream + events of the pipelined host I/O
        CK(cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&ctx->copy_out, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ctx->ev_call, cudaEventDisableTiming));
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
    if (ctx->opt.l2_persist_mb > 0 && !ctx->l2_changed) {
        // persisting-L2 window over the gathered W' records, attached to the sweep launches only (opt-in,
        // gmg_options.l2_persist_mb).  The limit is device-wide: the previous value is restored and the
        // persisting lines are reset by gmg_destroy
        int maxp = 0, maxw = 0;
        cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, ctx->opt.device);
        cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, ctx->opt.device);
        const size_t setaside = std::min<size_t>((size_t)maxp, (size_t)ctx->opt.l2_persist_mb << 20);
        CK(cudaDeviceGetLimit(&ctx->l2_prev_limit, cudaLimitPersistingL2CacheSize));
        CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, setaside));
        ctx->l2_changed = true;
        ctx->l2_window = std::min<size_t>((size_t)maxw, setaside);
    }
    {   // sweep grid: exactly one resident wave (grid-stride kernel, DESIGN.md §6 v5)
        int nsm = 0, per_sm = 0, per_ff = 0, per_ff1 = 0;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->opt.device);
        if (ctx->opt.dim == 3) {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sweep<3, 2, 0, 0>, 128, 0);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_ff, k_sweep<3, 2, 1, 0>, 128, 0);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_ff1, k_sweep<3, 2, 2, 0>, 128, 0);
        } else {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sweep<2, 2, 0, 0>, 128, 0);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_ff, k_sweep<2, 2, 1, 0>, 128, 0);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_ff1, k_sweep<2, 2, 2, 0>, 128, 0);
        }
        ctx->sweep_grid_cap = nsm * std::max(per_sm, 1);
        ctx->sweep_grid_cap_ff = nsm * std::max(per_ff, 1);
        ctx->sweep_grid_cap_ff1 = nsm * std::max(per_ff1, 1);
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
            CK(cudaMemcpyAsync((void *)V.glane, H.glane.data(), H.glane.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
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
    if (!ctx->opt.p2p || !ctx->p2p_ready || ctx->opt.nranks != 1 || P < 2 || P > kEmuMaxDom ||
        ctx->lv[level].ncolor > kEmuMaxCol) {
        ctx->err = "P2P emulation needs p2p = 1, 2..16 local domains, <= 24 colors";
        return GMG_ESTATE;
    }
    Launcher Lc{ctx, ctx->stream};
    const int gf = G_PREPARE | G_SIGMA | G_COPY_W;
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
    for (const Phase &ph : phase_list(ctx, level, n_sweeps)) seq.push_back(ph.c | (ph.ff ? 1 << 9 : 0));
    seq.push_back(255);
    if ((int)seq.size() > kEmuMaxPh) { ctx->err = "too many phases"; return GMG_EINVAL; }
    e.ndom = P;
    e.nph = (int)seq.size();
    for (size_t k = 0; k < seq.size(); ++k) e.ph[k] = (unsigned short)seq[k];
    std::vector<EmuDom> ed(P);
    for (int d = 0; d < P; ++d) {
        DevLevel &L = ctx->dom[d].dv[level];
        const DomLevel &H = ctx->dom[d].lv[level];
        ed[d].a = sweep_args(ctx, L, H, -1, 0, 0, L.Rt, nullptr);
        ed[d].p = P2PArgs{L.p2p_off, L.p2p_k, L.p2p_g, L.peer_wp, L.peer_nloc, L.npeer, L.p2p_wait, L.p2p_sig, L.p2p_flags, L.p2p_ctl};
        for (int c = 0; c <= nc; ++c) ed[d].blk[c] = (int)H.blk[c];
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
    if (dW_out) return get_dw_natural(ctx, level, dW_out);
    return GMG_OK;
}

gmg_status gmg_smooth(gmg_ctx *ctx, int level, int n_sweeps, double *dW_out)
{
    if (!ctx) return GMG_EINVAL;
    gmg_status st = check_ready(ctx, false);
    if (st) return st;
    if (level < 0 || level >= (int)ctx->lv.size() || n_sweeps < 1) { ctx->err = "bad level / n_sweeps"; return GMG_EINVAL; }
    Launcher Lc{ctx, ctx->stream};
    const int gf = G_PREPARE | G_SIGMA | G_COPY_W;
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
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->opt.p2p) {
        for (Domain &dm : ctx->dom) {
            int c2 = 0;
            CK(cudaMemcpy(&c2, dm.dv[0].p2p_ctl + 2, sizeof(int), cudaMemcpyDeviceToHost));
            if (c2) { ctx->err = "P2P halo: peer phase wait timed out"; return GMG_ECUDA; }
        }
    }
    if (dW_out) {
        st = get_dw_natural(ctx, level, dW_out);
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
    ctx->visits = 0;
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
    ctx->graph_visits = ctx->visits;
    return GMG_OK;
}

// GMG_ENONFINITE: the history went non-finite; name the first level (fine first) and the first
// natural cell whose state or fine residual holds a NaN / Inf
static gmg_status report_nonfinite(gmg_ctx *ctx)
{
    const int nv = ctx->opt.dim + 2;
    ctx->err = "non-finite residual history";
    for (int l = 0; l < (int)ctx->lv.size(); ++l) {
        for (int which = 0; which < 2; ++which) {
            if (which == 1 && l > 0) break;
            std::vector<double> h((size_t)nv * ctx->lv[l].n, 0.0);
            const gmg_status st = which == 0 ? get_natural(ctx, l, [](DevLevel &L) { return (const double *)L.W; }, nv, h.data())
                                             : get_natural(ctx, l, [](DevLevel &L) { return (const double *)L.Rt; }, nv, h.data());
            if (st) return st;
            const int64_t N = ctx->lv[l].n;
            for (int64_t i = 0; i < N; ++i)
                for (int q = 0; q < nv; ++q)
                    if (!std::isfinite(h[(size_t)q * N + i])) {
                        ctx->err = std::string("non-finite ") + (which == 0 ? "state" : "fine residual") + " at level " +
                                   std::to_string(l) + ", cell " + std::to_string(i) + " (natural id), component " +
                                   std::to_string(q);
                        return GMG_ENONFINITE;
                    }
        }
    }
    return GMG_ENONFINITE;
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
    if (ctx->opt.p2p) {
        for (Domain &dm : ctx->dom) {
            int c2 = 0;
            CK(cudaMemcpy(&c2, dm.dv[0].p2p_ctl + 2, sizeof(int), cudaMemcpyDeviceToHost));
            if (c2) { ctx->err = "P2P halo: peer phase wait timed out"; return GMG_ECUDA; }
        }
    }
    if (flags[1]) return report_nonfinite(ctx);
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

// a device pointer passed to the async host-I/O calls may be produced by work on the compute stream: order
// the copy stream after it (host buffers need no GPU ordering; waiting for them would serialise the pipeline)
static cudaError_t order_device_source(gmg_ctx *ctx, const void *p)
{
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return cudaSuccess; }
    if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged) return cudaSuccess;
    cudaError_t e = cudaEventRecord(ctx->ev_call, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->copy, ctx->ev_call, 0);
    return e;
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
    // copy stream: wait until the compute stream has consumed this slot, then H2D; a device source is
    // ordered after everything already enqueued on the compute stream (it may be produced there)
    CK(cudaStreamWaitEvent(ctx->copy, ctx->ev_in_free[k], 0));
    CK(order_device_source(ctx, W));
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
    CK(order_device_source(ctx, W_owned));
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
    if (flags[1]) return report_nonfinite(ctx);
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

int64_t gmg_vcycle_visits(gmg_ctx *ctx)
{
    if (!ctx) return -1;
    if (!ctx->graph && check_ready(ctx) == GMG_OK) build_graph(ctx);
    return ctx->graph_visits;
}

gmg_status gmg_get_level_field(gmg_ctx *ctx, int level, int field, double *out)
{
    if (!ctx) return GMG_EINVAL;
    gmg_status st = check_ready(ctx, false);
    if (st) return st;
    if (level < 0 || level >= (int)ctx->lv.size() || !out || field < GMG_FIELD_W || field > GMG_FIELD_ALPHA) {
        ctx->err = "bad level / field / null";
        return GMG_EINVAL;
    }
    const int nv = ctx->opt.dim + 2;
    switch (field) {
        case GMG_FIELD_W: return get_natural(ctx, level, [](DevLevel &L) { return (const double *)L.W; }, nv, out);
        case GMG_FIELD_W0: return get_dw_natural(ctx, level, out, true);
        case GMG_FIELD_DW: return get_dw_natural(ctx, level, out);
        case GMG_FIELD_RS: return get_natural(ctx, level, [](DevLevel &L) { return (const double *)L.Rs; }, nv, out);
        case GMG_FIELD_F: return get_natural(ctx, level, [](DevLevel &L) { return (const double *)L.F; }, nv, out);
        case GMG_FIELD_RT: return get_natural(ctx, level, [](DevLevel &L) { return (const double *)L.Rt; }, nv, out);
        default: return get_natural(ctx, level, [](DevLevel &L) { return (const double *)L.alpha; }, 1, out);
    }
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
    for (int l = 0; l < nl; ++l) out[l] = (int64_t)((const char *)dm.dv[l].wp - (const char *)ctx->ws);
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
    if (!ctx->opt.p2p || ctx->nparts < 2 || H.p2p_off.empty()) { ctx->err = "no P2P targets (p2p = 1, > 1 partition)"; return GMG_ESTATE; }
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
    if (ctx->opt.nranks < 2 || !ctx->opt.p2p) { ctx->err = "P2P import needs nranks > 1 and p2p = 1"; return GMG_ESTATE; }
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
            // the peers' state-array sizes (owned + ghost cells of their domain on this level), from the setup
            CK(cudaMemcpy(dm.dv[l].peer_nloc, H.p2p_peer_nloc.data(), H.p2p_peer_nloc.size() * sizeof(int),
                          cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dm.dv[l].peer_wp, pr.data(), pr.size() * sizeof(double *), cudaMemcpyHostToDevice));
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
        if (ctx->ev_call) cudaEventDestroy(ctx->ev_call);
        for (int k = 0; k < 2; ++k) {
            cudaEventDestroy(ctx->ev_in_ready[k]);
            cudaEventDestroy(ctx->ev_in_free[k]);
            cudaEventDestroy(ctx->ev_out_ready[k]);
            cudaEventDestroy(ctx->ev_out_free[k]);
        }
    }
    if (ctx->nccl_comm && nccl().CommDestroy) nccl().CommDestroy((ncclComm_t)ctx->nccl_comm);
    if (ctx->l2_changed) {   // the persisting-L2 set-aside is device-wide: give it back
        if (ctx->stream) cudaStreamSynchronize(ctx->stream);
        cudaCtxResetPersistingL2Cache();
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, ctx->l2_prev_limit);
    }
    for (void *p : ctx->p2p_opened) cudaIpcCloseMemHandle(p);
    delete ctx->ho;
    delete ctx;
}

}  // extern "C"
