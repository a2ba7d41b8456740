// gmg_internal.h -- private structures of libgmg (host setup + device layout).
// Not part of the ABI.  Nothing here is shared with oracle/.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/gmg.h"

namespace gmg {

constexpr int kChunk = 32;  // SELL chunk height = one warp of cells

// ---------------------------------------------------------------------------
// Host description of one level (natural numbering) + its internal layout.
// ---------------------------------------------------------------------------
struct HostLevel {
    int dim = 3;
    int64_t n = 0, nf = 0;
    std::vector<double> vol, ctr;          // [n], [dim][n]
    std::vector<int64_t> left, right;      // [nf]
    std::vector<double> avec, fctr;        // [dim][nf]
    std::vector<int8_t> ngauss;            // [nf]
    std::vector<int32_t> part;             // [n] partition id (empty: single rank)

    // coloring and renumbering (a2, a3)
    std::vector<int32_t> color;            // [n] natural order, 1..ncolor
    int ncolor = 0;
    std::vector<int64_t> perm;             // internal -> natural
    std::vector<int64_t> iperm;            // natural -> internal
    std::vector<int64_t> blk;              // [ncolor+1] color block offsets (internal)

    // agglomeration to the next level (a4)
    std::vector<int64_t> parent;           // [n] natural -> natural coarse id (empty: coarsest)
    int64_t n_coarse = 0;

    // layouts (internal order), see build_layout
    int64_t nchunks = 0;
    std::vector<int32_t> chunk_base;       // [ncolor+1] first gather chunk of each color
    std::vector<int32_t> goff;             // [nchunks] gather entry offset of each chunk
    int64_t ng_entries = 0, ns_entries = 0;
    std::vector<int32_t> gbase;            // [n] gather entry of slot 0 (slot s at gbase + 32 s)
    std::vector<uint8_t> deg_int, deg_all; // [n] interior / all face slots
    std::vector<int32_t> gface;            // [ng_entries] signed face slot: +(f+1) left, -(f+1) right, 0 pad
    std::vector<int32_t> soffc;            // [n+1] sweep slots of cell i: [soffc[i], soffc[i+1])
    std::vector<int32_t> sJ;               // [ns_entries] neighbour (internal)
    std::vector<double> sRec;              // [ns_entries][4] (A_x, A_y, A_z | S r) 3D, (A_x, A_y, S r, 0) 2D
    std::vector<int32_t> sface;            // [ns_entries] face id of the slot (host bookkeeping)
};

// ---------------------------------------------------------------------------
// Device view of one level (pointers into the workspace).
// Cell arrays are AoS [n][nv] in internal (color-contiguous) order.
// ---------------------------------------------------------------------------
struct DevLevel {
    int dim, nv, ncolor;
    int n, nf, nchunks;
    // faces (natural face order; cells as internal indices)
    const int *fl, *fr;          // fr < 0: -(patch+1)
    const double *fA;            // [dim][nf]
    const int8_t *fM;            // [nf]
    double *Fs;                  // [nf][nv]  S_f F_f (left -> right)
    double *Srf;                 // [nf]      S_f r_f
    double *aM;                  // [nf]      alpha_f^{M_f}
    // cells (AoS [n][nv], internal order)
    const double *vol;           // [n]
    double *W;                   // [n][nv] state
    double *Rt, *Rs, *F;         // [n][nv] RHS / restricted residual / forcing
    double *alpha, *sigma, *tmp; // [n]
    double *rec;                 // [n][REC] sweep record: W_lin | 1/D | dW | alpha/2 (kernels.cuh Rec<D>)
    const uint8_t *deg_int, *deg_all;    // [n]
    const int *gbase;            // [n] gather entry of slot 0; slot s at gbase + 32 s
    const int *gface;            // gather entries
    const int *soff;             // [n+1] sweep slot range per cell
    const int *sJ;               // [ns] neighbour
    double *sRec;                // [ns][4] A (outward) + S r
    const int *perm;             // [n] internal -> natural
    // multigrid links
    const int *child;            // [2][n] fine children (internal idx in level-1), -1 = none (coarse levels)
    const int *parent;           // [n] coarse parent (internal idx in level+1), fine levels
    double *partial;             // [nblocks_max][nv] norm partials
};

struct Profile {
    bool on = false;
    std::vector<cudaEvent_t> ev;
    std::vector<std::pair<int, int>> marks;  // (kernel class, event index of start)
};

// algorithmic bytes bookkeeping
struct LevelBytes {
    double face_flux = 0, face_prep = 0, gather = 0, restrict_ = 0, prolong = 0, update = 0;
    int max_slots64 = 1, max_slots128 = 1;   // staged sweep: max slots per 64 / 128-cell chunk
    std::vector<double> sweep;     // per color
    std::vector<double> sweep_out; // per color, extra bytes when the launch also writes W = W0 + dW
};

}  // namespace gmg

struct gmg_ctx {
    gmg_options opt;
    std::string err;
    std::vector<gmg::HostLevel> lv;
    std::vector<int32_t> user_color0;
    int n_patches = 0;
    std::vector<int32_t> patch_kind;
    bool mesh_loaded = false, built = false, ws_ready = false, state_set = false;
    // device
    void *ws = nullptr;
    size_t ws_bytes = 0;
    std::vector<gmg::DevLevel> dv;
    double *d_hist = nullptr;     // [hist_cap][nv]
    int hist_cap = 0;
    int *d_flag = nullptr;
    double winf[5] = {0, 0, 0, 0, 0};
    cudaStream_t stream = nullptr;
    cudaGraphExec_t graph = nullptr;  // one V-cycle
    int64_t graph_launches = 0;
    gmg::Profile prof;
    std::vector<gmg::LevelBytes> lbytes;
    double kbytes[GMG_K_COUNT] = {0};   // algorithmic bytes accumulated by the recorded sequence
    int64_t launches = 0;          // kernels launched by the last recorded sequence
    int lpc = 2;                   // sweep lanes per cell (1, 2, 4)
    int minb = 4;                  // sweep __launch_bounds__ min blocks per SM (4, 6, 8)
    int prefetch = 0;              // sweep: L2-prefetch neighbour records before gathering (slower; kept for experiments)
    int sweep_mode = 0;            // 0 = register gather (lpc lanes/cell), 1/2 = smem-staged 64/128-cell chunks
    size_t l2_window = 0;          // bytes of the persisting-L2 window over a level's records (0 = off)
    double *d_stage = nullptr;     // natural-order staging buffer [nv][nmax]
    std::vector<int> host_keep_alive;
};

namespace gmg {
// setup.cpp
gmg_status load_mesh(gmg_ctx *ctx, int64_t n, const double *vol, const double *ctr, int64_t nf,
                     const int64_t *left, const int64_t *right, const double *avec, const double *fctr,
                     const int8_t *ng, const int32_t *part);
int color_level(HostLevel &L);                          // Algorithm 1
bool validate_coloring(const HostLevel &L, const std::vector<int32_t> &col);
int64_t agglomerate(const HostLevel &L, double theta, std::vector<int64_t> &parent, int64_t &nc);
void build_coarse(const HostLevel &fine, HostLevel &coarse);
void renumber(HostLevel &L);
void build_layout(HostLevel &L);
}  // namespace gmg
