// gmg_internal.h -- private structures of libgmg (host setup + device layout).
// Not part of the ABI.  Nothing here is shared with oracle/.
//
// Data model
//  * HostLevel: one GLOBAL level in natural numbering (geometry, Algorithm-1
//    colors, global renumbering, parent map, partition ids).  Every rank
//    builds the identical global hierarchy (deterministic host code).
//  * DomLevel: the part of a level one domain (rank) works on: its owned
//    cells in color blocks (boundary cells first when partitioned; Morton key
//    of the centroid inside), then one layer of ghost cells in (owner, color,
//    natural id) order; the local faces (those touching an
//    owned cell); slot layouts over owned cells; multigrid links; the halo
//    plan grouped by (color, peer).
//  * DevLevel: device pointers of a DomLevel (inside the workspace).
// A single-GPU run is one domain owning everything (no ghosts, no peers).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/gmg.h"

namespace gmg {

constexpr int kChunk = 32;  // SELL chunk height = one warp of cells

struct HostLevel {
    int dim = 3;
    int64_t n = 0, nf = 0;
    std::vector<double> vol, ctr;          // [n], [dim][n]
    std::vector<int64_t> left, right;      // [nf]
    std::vector<double> avec, fctr;        // [dim][nf]
    std::vector<int8_t> ngauss;            // [nf]
    std::vector<int32_t> part;             // [n] partition id (empty: one partition)
    // coloring and renumbering (a2, a3)
    std::vector<int32_t> color;            // [n] natural order, 1..ncolor
    int ncolor = 0;
    std::vector<int64_t> perm;             // global renumbering: position -> natural (stable by color)
    // agglomeration to the next level (a4)
    std::vector<int64_t> parent;           // [n] natural -> natural coarse id (empty: coarsest)
    int64_t n_coarse = 0;
    int part_of(int64_t i) const { return part.empty() ? 0 : part[i]; }
};

struct DomLevel {
    int64_t n_own = 0, n_loc = 0, nf = 0;
    std::vector<int64_t> l2n;              // [n_loc] local -> natural
    std::vector<int64_t> blk;              // [ncolor+1] color blocks over owned cells
    std::vector<int64_t> nbnd;             // [ncolor] boundary cells (ghost neighbour) at the start of each block
    std::vector<int64_t> fnat;             // [nf] natural ids of the local faces (ascending)
    std::vector<int32_t> fl, fr;           // [nf] local left / right, fr < 0: -(patch+1)
    std::vector<double> vol;               // [n_own]
    // gather slots (SELL-32 over owned cells in the gather order: chunks of 32 cells, entries [slot][lane])
    std::vector<int32_t> gord;             // [n_own] gather position -> owned cell (Morton across colors)
    int64_t nchunks = 0, ng_entries = 0, ns_entries = 0;
    std::vector<int32_t> goff, gbase;      // [nchunks], [n_own]
    std::vector<uint8_t> deg_int, deg_all; // [n_own]
    std::vector<int32_t> gface;            // [ng_entries] +(f+1) left, -(f+1) right (local face f), 0 pad
    // sweep slots (CSR over owned cells, same order as their interior gather slots)
    std::vector<int32_t> soffc;            // [n_own+1]
    std::vector<int32_t> sJe;              // [ns] local neighbour (owned or ghost)
    std::vector<double> sRe;               // [ns][4] (A outward | S r)
    std::vector<int32_t> fslot;            // [nf][2] sweep entry of the face in its left / right cell's slots (-1: none)
    // multigrid links (local indices)
    std::vector<int32_t> child;            // [2][n_own] coarse levels: fine children, -1 = none
    std::vector<int32_t> parent;           // [n_own] levels with a coarser one: coarse parent
    // halo plan: groups (color c, peer k) at [off[c*npeers+k], off[c*npeers+k+1])
    std::vector<int> peers;                // peer ranks, ascending
    std::vector<int32_t> send_idx, recv_idx;   // local cells (owned / ghost)
    std::vector<int64_t> send_off, recv_off;   // [ncolor*npeers + 1]
    // fused P2P halo: per owned cell, the ghost copies it must update (peer slot, peer-local ghost index)
    std::vector<int32_t> p2p_off, p2p_k, p2p_g;
    std::vector<int32_t> p2p_peer_nloc;    // [npeers] the peers' owned + ghost cells on this level
};

// NEXT-1: third-order compact GKS fine operator, fine level.
// Device arrays live in the workspace (carve); [n] = owned cells, [nl] = owned + ghosts.
struct HoDev {
    int G = 0, nk = 0, nc = 0, nq = 0;   // Gauss slots per face, p2 unknowns, poly coefficients, m2 components
    const double *ctr = nullptr;         // [nl][D] centroids (local order)
    const double *m2 = nullptr;          // [nl][nq] central second moments
    const double *gp = nullptr;          // [nf][G][D] Gauss points (local faces)
    const double *gw = nullptr;          // [nf][G] weights (0 = padding)
    const int *hfoff = nullptr;          // [n+1] cell -> faces
    const int *hface = nullptr;          // signed local faces: +(f+1) cell is left, -(f+1) right; ascending natural id
    const double *hrec = nullptr;        // [slots][4] per (cell, face) slot: A outward (D doubles) | (neighbour or
                                         //   -(patch+1), local face) as two int32 in the last double
    const int *poff = nullptr;           // [n+1] offset (doubles) of the cell's p2 operator; empty = p1 only
    const double *P = nullptr;           // per interior neighbour m: (D+1) columns of nk: d a / d(Q_m - Q_i), d a / d(Q_e)_m,
                                         // padded to a multiple of 4 doubles (32-byte aligned blocks)
    double *G_ = nullptr;                // [nl][nv][D] cell-averaged slopes (carried; ghosts by halo)
    double *alpha = nullptr;             // [n] DF carried between evaluations (p1 factor, C4/C14)
    double *poly = nullptr;              // [nl][nv][nc] final polynomials (c0, lin[D], quad[nq]) about the centroid
    int *flags = nullptr;                // [n] bit 0 p2 used
    double *sr = nullptr;                // [nf] S r_f (first-order spectral radius, A5)
    double *dt = nullptr;                // [nl] Dt_i = CFL_exp V_i / Sigma_i (C8)
    const int2 *glane = nullptr;         // [nlane] packed Gauss-point lanes of the flux kernel (HoLocal::glane)
    int nlane = 0;
    double *frec = nullptr;              // [nf][12] S sum_k w F_k / Dt_f [nv] | sum_k w W_k(Dt_f) [nv] | prod alpha_fk
    double *Gout = nullptr;              // [n][nv][D] slopes of a non-updating evaluation
};

struct DevLevel {
    int dim, nv, ncolor;
    int n, n_loc, nf;            // owned cells, owned + ghost cells, local faces
    // faces (local)
    const int *fl, *fr;
    const double *fA;            // [dim][nf]
    const int8_t *fM;            // [nf]
    double *Frec;                // [nf][8] (S_f F_f (left -> right) | S_f r_f | alpha_f^{M_f} | 0)
    // cells (AoS, local order; [n_loc] where ghosts are needed)
    const double *vol;           // [n]
    double *W;                   // [n_loc][nv] state
    double *Rt, *Rs, *F;         // [n][nv] RHS / restricted residual / forcing
    double *alpha, *sigma, *tmp; // [n]
    // smoother state (W' formulation; strides Wp<D>::STRIDE, kXr)
    double *wlin;                // state array (Wp<D> layout, n_loc cells): W_lin (coarse: the restricted W0)
    double *wp;                  // state array: W' = W_lin + dW of the current half-sweep
    double *xr;                  // [n][kXr] X = W_lin - Rt/D + c P, c = alpha/(2D) (own-cell record)
    double *dc;                  // [n][2] 1/D, alpha/(2D) of the hybrid diagonal (gather G_PREPARE)
    const uint8_t *deg_int, *deg_all;    // [n]
    const int *gord;             // [n] gather position -> owned cell (Morton across colors)
    const int *gface;
    const int2 *sinfo;           // [n] (first sweep slot, interior slots) packed for one 8-byte load
    const int2 *fslot;           // [nf] sweep entries of the face (left cell, right cell), -1 = none
    const int4 *ginfo;           // [n] per gather position t: (gbase, deg_all | deg_int << 16, cell, 0)
    const int *sJe;              // [ne] neighbour, -1 = padding
    double *sRe;                 // [ne][4] A outward + S r
    const int *perm;             // [n_loc] local -> natural
    const int *child;            // [2][n]
    const int *parent;           // [n]
    double *partial;             // [nblocks][nv] norm partials
    // fused P2P halo (gmg_options.p2p)
    const int *p2p_off, *p2p_k, *p2p_g;
    double **peer_wp;                 // [npeer] peers' W' arrays (this level)
    int *peer_nloc;                   // [npeer] their state-array sizes (owned + ghost cells)
    int **p2p_sig;                    // [npeer] &peer.flags[my rank]
    int *p2p_wait;                    // [npeer] peer ranks
    int *p2p_flags, *p2p_ctl;         // per domain: [nparts] published phase counts, [4] control
    int npeer;
    // halo
    int n_send, n_recv;
    const int *send_idx, *recv_idx;
    double *sendbuf, *recvbuf;   // [n_send][nv], [n_recv][nv]
    HoDev ho;                    // NEXT-1 (level 0 only)
};

struct Profile {
    bool on = false;
    std::vector<cudaEvent_t> ev;
    std::vector<std::pair<int, int>> marks;  // (kernel class, event index of start)
    std::vector<double> bytes;               // algorithmic bytes of each mark
};

// algorithmic bytes bookkeeping
struct LevelBytes {
    double face_flux = 0, face_prep = 0, face_slots = 0, gather = 0, restrict_ = 0, prolong = 0, update = 0;
    std::vector<double> sweep;     // per color, SURVEY §8(d) compulsory bytes of one half-sweep phase
    std::vector<double> sweep_ff;  // per color, the same for the first forward half-sweep (only the lower-color
                                   // neighbours carry an increment: their slots and records are charged)
    std::vector<double> sweep_out; // per color, extra bytes when the launch also writes W = W0 + dW
    std::vector<int64_t> visits;   // per color: owned cells (one cell-update each)
};

// modes of the NEXT-1 gather (ho.cu k_ho_gather)
enum : int {
    HO_NORM = 1,     // per-block partial sums of R_q^2 (history)
    HO_UPDATE = 2,   // W -= CFL_exp R / Sigma (C12), G = new slopes, alpha carried = alpha
    HO_RT = 4,       // Rt = R, level alpha = alpha (restriction inputs), alpha carried = alpha
    HO_OUT = 8,      // R -> Rout (AoS), new slopes -> Gout, alpha -> alpha_out (ABI)
};
// NEXT-1 geometry as loaded (natural order) -- ctx->ho
struct HoHost {
    int G = 0;
    std::vector<double> m2, gp, gw;      // [nq][N], [D][G][NF], [G][NF]
    bool prepared = false;
};
// NEXT-1 per domain, level 0, local order (ho_setup.cpp)
struct HoLocal {
    std::vector<double> ctr, m2l, gpl, gwl, P, hrec;   // ctr / m2l over owned + ghost cells
    std::vector<int> hfoff, hface, poff;               // owned cells
    std::vector<int32_t> glane;          // [nlane][2] flux lanes: (f G + k | -1, Gauss points of f on its first lane, else 0)
    int64_t n_p2 = 0;                    // cells with a p2 operator
    int64_t n_gauss_pts = 0;             // Gauss points of the local faces (flux work units)
    double bytes_sr = 0, bytes_recon = 0, bytes_flux = 0, bytes_gather = 0;   // algorithmic bytes per launch
    double *sendbuf = nullptr, *recvbuf = nullptr;     // halo of slopes / polynomials / Dt (partitioned)
};

struct Domain {
    int rank = 0;
    HoLocal ho;                  // NEXT-1 (level 0)
    std::vector<DomLevel> lv;
    std::vector<DevLevel> dv;
    std::vector<LevelBytes> lbytes;
};

}  // namespace gmg

struct gmg_ctx {
    gmg_options opt;
    std::string err;
    std::vector<gmg::HostLevel> lv;          // global hierarchy
    std::vector<gmg::Domain> dom;            // domains driven by this process
    int nparts = 1;                          // partitions of the global mesh
    std::vector<int32_t> user_color0;
    int n_patches = 0;
    std::vector<int32_t> patch_kind;
    bool mesh_loaded = false, built = false, ws_ready = false, state_set = false;
    // device
    void *ws = nullptr;
    size_t ws_bytes = 0;
    double *d_hist = nullptr;     // [hist_cap][nv]
    int hist_cap = 0;
    int *d_flag = nullptr;        // [0] history index, [1] non-finite flag
    double *d_sumsq = nullptr;    // [ndom][nv] per-domain residual sums of squares
    double *d_stage = nullptr;    // natural-order staging [nv][Nmax]
    double winf[5] = {0, 0, 0, 0, 0};
    cudaStream_t stream = nullptr;
    cudaGraphExec_t graph = nullptr;  // one V-cycle
    int64_t graph_launches = 0;
    int64_t graph_visits = 0;         // sweep cell-updates executed per captured V-cycle
    void *nccl_comm = nullptr;        // ncclComm_t (multi-rank)
    gmg::Profile prof;
    double kbytes[GMG_K_COUNT] = {0}; // algorithmic bytes accumulated by the recorded sequence
    int64_t launches = 0;             // kernels launched by the last recorded sequence
    int64_t exchanges = 0;            // halo exchanges in the last recorded sequence
    int sweep_grid_cap = 0;           // sweep grid = one resident wave: SMs x blocks/SM (set with the workspace)
    int sweep_grid_cap_ff = 0;        // the same for the first-forward variant (more registers)
    int sweep_grid_cap_ff1 = 0;       // ... and for the first-forward phase of the first color (no W' gathers)
    int64_t visits = 0;               // cell-updates executed by the last recorded sequence
    int lpc = 2;                      // sweep lanes per cell of the large color blocks (gmg_options.sweep_lanes)
    int adapt_lpc = 1;                // blocks that fit one wave at 2x lanes get up to 16 lanes per cell
    bool p2p_ready = false;           // peer pointers known (local domains: at workspace; ranks: after import)
    std::vector<void *> p2p_opened;   // IPC mappings of the peers' workspaces (ranks)
    char *d_emu = nullptr;            // test only: EmuDom[16] of k_p2p_emulate
    int *d_emu_bar = nullptr;         // test only: group barriers of k_p2p_emulate
    size_t l2_window = 0;             // persisting-L2 window over the W' records (gmg_options.l2_persist_mb)
    size_t l2_prev_limit = 0;         // the device's persisting-L2 limit before this context changed it
    bool l2_changed = false;
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    gmg::HoHost *ho = nullptr;        // NEXT-1 geometry + setup (gmg_load_ho_geometry)
    // pipelined host I/O (gmg_*_async): copy stream, double-buffered staging, events
    cudaStream_t copy = nullptr, copy_out = nullptr;   // host->device / device->host copy streams
    double *stage_in[2] = {nullptr, nullptr}, *stage_out[2] = {nullptr, nullptr};   // [nv][N0] natural order
    cudaEvent_t ev_in_ready[2] = {}, ev_in_free[2] = {}, ev_out_ready[2] = {}, ev_out_free[2] = {};
    cudaEvent_t ev_call = nullptr;    // compute-stream position when an async call reads a device source
    int in_slot = 0, out_slot = 0;
    bool async_flag_reset = false;    // d_flag cleared for the current async epoch
};

namespace gmg {
struct SetupStats {                 // device setup diagnostics
    int64_t color_levels = 0, color_rounds = 0, match_rounds = 0;
};
// setup_dev.cu (device-side Algorithm 1 / Algorithm 3, results identical to the host versions)
int color_level_dev(HostLevel &L, cudaStream_t s, SetupStats *st);
int64_t agglomerate_dev(const HostLevel &L, double theta, std::vector<int64_t> &parent, int64_t &nc, cudaStream_t s,
                        SetupStats *st);
// setup.cpp
gmg_status load_mesh(gmg_ctx *ctx, int64_t n, const double *vol, const double *ctr, int64_t nf,
                     const int64_t *left, const int64_t *right, const double *avec, const double *fctr,
                     const int8_t *ng, const int32_t *part);
int color_level(HostLevel &L);                          // Algorithm 1
bool validate_coloring(const HostLevel &L, const std::vector<int32_t> &col);
int64_t agglomerate(const HostLevel &L, double theta, std::vector<int64_t> &parent, int64_t &nc);
void build_coarse(const HostLevel &fine, HostLevel &coarse);
void renumber(HostLevel &L);
void build_domain_level(const HostLevel &G, int rank, DomLevel &D, bool morton = false);
void link_domain_levels(const HostLevel &Gf, const HostLevel &Gc, DomLevel &Df, DomLevel &Dc);
void build_p2p_targets(DomLevel &D, int me, int ncolor, const std::vector<const DomLevel *> &peer_dom);
void partition_rcb(int64_t n, int dim, const double *ctr, int nparts, int32_t *part);
// ho_setup.cpp (NEXT-1): local geometry, cell -> face lists and the per-cell p2 operators
gmg_status ho_prepare(gmg_ctx *ctx);
}  // namespace gmg
