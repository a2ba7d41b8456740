/*
 * gmg.h -- C ABI of libgmg: the B200 (sm_100a) hot path of arXiv 2509.06347,
 * "A Geometric Multigrid-Accelerated Compact Gas-Kinetic Scheme ..." :
 * multi-color matrix-free LU-SGS (MC-LU-SGS) smoothing inside a 3-level
 * geometric V-cycle on unstructured 2D/3D meshes, with hash/skewness
 * agglomeration, volume-weighted restriction, forcing and DF-limited
 * prolongation.
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n (the reference
 * texts), readings A1..A30.
 *
 * ---------------------------------------------------------------------------
 * Conventions (apply to every call)
 *  - Ownership: the caller owns every pointer it passes; the library copies
 *    what it needs during the call and never retains caller pointers.
 *  - Arrays at the boundary are in NATURAL order (the mesh generator's cell /
 *    face numbering, or the natural numbering of a coarse level, O1), SoA
 *    [component][item], float64 unless stated.  The library permutes
 *    internally (color-contiguous renumbering).
 *  - Pointers may be host or device memory (classified with
 *    cudaPointerGetAttributes) wherever "host/device" is written.
 *  - Device memory: ONE caller-allocated workspace (gmg_set_workspace); the
 *    library sub-allocates it.  The only other device allocations are the
 *    temporaries of the optional device-side setup (setup_device = 1:
 *    stream-ordered cudaMallocAsync, freed before gmg_build_hierarchy
 *    returns).  Host-side setup (coloring, agglomeration, layouts) uses host
 *    heap memory.
 *  - Threads: a context is not thread-safe; use it from one thread at a time.
 *  - Stream: every call is asynchronous on gmg_options.stream; a call that
 *    returns host data synchronizes that stream first.
 *  - Errors: return codes only; no exceptions cross the ABI.  A failing
 *    call leaves a message in gmg_last_error(ctx).
 *  - Multi-rank (nranks > 1): collective semantics, every rank
 *    makes the same sequence of calls with the same global mesh and the same
 *    part[] array.  Every rank builds the identical global hierarchy (colors
 *    are global, agglomeration never crosses a partition face) and
 *    works on its owned cells plus one ghost layer; increments are exchanged
 *    after every color (NCCL send/recv), states after state changes, norms
 *    are all-reduced.  Natural-order outputs of multi-rank calls write only
 *    the caller rank's owned entries.
 * ---------------------------------------------------------------------------
 */
#ifndef GMG_H
#define GMG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gmg_ctx gmg_ctx; /* opaque; one per rank */

typedef enum {
    GMG_OK = 0,
    GMG_EINVAL = 1,      /* bad argument / option                                  */
    GMG_ETOPO = 2,       /* mesh topology: bad cell index, non-manifold, open cell   */
    GMG_ECOLOR = 3,      /* user coloring invalid (same-color face neighbours)      */
    GMG_ESTALL = 4,      /* hierarchy truncated: a level merged nothing     */
    GMG_ENOMEM = 5,      /* workspace too small / host allocation failed            */
    GMG_ECUDA = 6,       /* CUDA runtime error                                      */
    GMG_ENCCL = 7,       /* NCCL error (multi-rank)                                 */
    GMG_ENONFINITE = 8,  /* NaN/Inf detected; level and cell in gmg_last_error      */
    GMG_ESTATE = 9       /* call out of order (e.g. smooth before workspace)        */
} gmg_status;

/* boundary patch kinds (ghost states, SURVEY O4 / reading A25) */
enum { GMG_FARFIELD = 0, GMG_SLIP = 1, GMG_NOSLIP = 2, GMG_EXTRAP = 3 };

typedef struct {
    int dim;                /* 2 or 3; nv = dim + 2 conserved variables W = (rho, m, rho E) */
    double gamma;           /* ratio of specific heats, 1.4                                 */
    double cfl_imp;         /* implicit CFL, Dt_imp = cfl_imp V / Sigma (A2, A3); 10  */
    double cfl_exp;         /* explicit CFL, Dt_exp = cfl_exp V / Sigma; 0.5          */
    int n_sweeps;           /* MC-LU-SGS sweeps per smoothing step; 6          */
    int n_levels;           /* V-cycle levels; 3                                      */
    int pre_smooth;         /* 1; only 1 is supported                                 */
    int post_smooth;        /* 0; only 0 is supported                                 */
    double skew_limit;      /* agglomeration skewness threshold theta (A21); 0.5              */
    double r_factor;        /* omega in r_ij = omega (|U.n| + a) >= Lambda; 1.0       */
    int fine_smoother;      /* 0 = explicit Eq.(smo) (paper); 1 = MC-LU-SGS        */
    int df_mode;            /* 0 = first-order DF helper (O5); 1 = user alpha; 2 = alpha == 1
                               (DF off); 3 = fixed relaxation factor beta in the smoother      */
    int rank, nranks;       /* this rank / world size (1 = single GPU)                        */
    const void *nccl_id;    /* 128-byte ncclUniqueId (nranks > 1), else NULL                  */
    int device;             /* CUDA device ordinal                                            */
    void *stream;           /* cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream)    */
    double beta;            /* df_mode 3 only: the fixed relaxation factor of the "traditional
                               relaxation" used in place of the per-cell DF alpha in
                               the smoother's diagonal and off-diagonal; prolongation keeps the
                               DF limiter (reading B3).  Default 0.5.                         */
    int local_domains;      /* nranks == 1 only: drive this many partitions (part[] values
                               0..local_domains-1) as separate domains in this process, their
                               halo exchanged by device copies on the stream.  Same layouts,
                               plans, pack/unpack kernels and exchange points as the NCCL path;
                               used to test the partitioned path on one GPU.  Default 1.      */
    int setup_device;       /* 1: gmg_build_hierarchy runs Algorithm 1 (coloring) and
                               Algorithm 3 (agglomeration) on `device`.
                               The results are identical to the host setup (0, default):
                               same colors, renumbering and parent maps, bit for bit.         */
    int fine_operator;      /* fine-level residual of the V-cycle:
                               0 = first-order KFVS (O4, default); 1 = third-order compact GKS
                               (§2.3-§3; readings C1-C14 of DESIGN.md §12):
                               p2/p1 WENO + DF reconstruction from the cell averages and the
                               cell-averaged slopes, BGK flux at the face Gauss points, direct
                               slope evolution.  Needs gmg_load_ho_geometry, a single domain
                               (nranks = local_domains = 1), fine_smoother = 0, df_mode = 0.  */
    double ho_c1, ho_c2;    /* C9 collision time tau = c1 Dt + c2 Dt |pl - pr| / (pl + pr);
                               defaults 0.05, 1.0                                              */
    double ho_gam0;         /* C5 linear weight of the large (p2) stencil; default 0.95        */
    double ho_eps;          /* C5 WENO-Z epsilon; default 1e-14                                */
    /* execution choices (no effect on the results beyond rounding) */
    int skip_repeat;        /* 1 (default): the color phase that directly repeats the previous
                               one at every sweep turn of Algorithm 2 (c_N forward then c_N
                               backward, c_1 backward then c_1 forward) is not run -- it reads
                               only other-colored neighbours, none of which changed, so it
                               recomputes identical values (exact); 0 runs every phase.        */
    int p2p;                /* partitioned runs: 1 = fused halo, the sweep epilogue stores a
                               boundary cell's new state into the peers' ghost records over
                               peer memory (CUDA IPC between ranks, gmg_p2p_layout/_import);
                               0 (default) = pack / NCCL send-recv (device copies between local
                               domains) / unpack after every color.                           */
    int overlap;            /* partitioned runs: 1 = sweep a color's boundary cells, exchange
                               them on a side stream while its interior cells are swept; 0 =
                               sweep, then exchange; -1 (default) = 1 for NCCL ranks, 0 for
                               local domains.                                                 */
    int l2_persist_mb;      /* > 0: set aside this many MB of L2 as persisting and attach an
                               access-policy window over the gathered W' records to the sweep
                               launches (the previous device limit is restored and the
                               persisting lines reset by gmg_destroy); 0 (default) = off.      */
    int sweep_lanes;        /* lanes per cell of the sweep kernel for the large color blocks:
                               1, 2 (default; 0 = default) or 4                                */
    int pdl;                /* 1 (default): programmatic dependent launch between the kernels
                               of a V-cycle; 0 = plain stream order                            */
    int ho_p2min;           /* fine_operator 1, readings C3 / C3b: a cell uses
                               the p2 reconstruction only with at least this many interior
                               von Neumann neighbours; 0 (default) = d + 1 (C3); d + 2 keeps the
                               simplices (triangles / tets) on p1 (C3b)                       */
} gmg_options;

/* Fill *o with the defaults above (dim = 3, single rank, device 0, stream 0). */
void gmg_default_options(gmg_options *o);

/* Create a context.  Validates options (GMG_EINVAL). */
gmg_status gmg_create(const gmg_options *opt, gmg_ctx **out);

/* a1: load the fine mesh (host pointers, natural order):
 *   vol[n], centroid[dim][n]; faces: left[nf] (owner cell), right[nf] (other
 *   cell, or -(patch+1) for a boundary face), area_vec[dim][nf] = S_f n_f
 *   pointing left -> right, face_ctr[dim][nf], n_gauss[nf] = M_f (DF exponent,
 *   P:174; 2 per 2D segment, 3 per triangle, 4 per quad), patch_kind[n_patches]
 *   (GMG_FARFIELD ...).  part[n] = global cell -> rank (NULL if nranks == 1).
 * Validates indices, manifoldness and per-cell closure |sum sigma A| <=
 * 1e-10 sum S -> GMG_ETOPO. */
gmg_status gmg_load_mesh(gmg_ctx *ctx, int64_t n_cells, const double *vol, const double *centroid,
                         int64_t n_faces, const int64_t *left, const int64_t *right,
                         const double *area_vec, const double *face_ctr, const int8_t *n_gauss,
                         int n_patches, const int32_t *patch_kind, const int32_t *part);

/* a2: optional user coloring of the FINE level (host, natural order, colors
 * 1..Nc).  NULL = Algorithm 1.  Must precede
 * gmg_build_hierarchy.  GMG_ECOLOR if two face neighbours share a color. */
gmg_status gmg_set_coloring(gmg_ctx *ctx, int level, const int32_t *color);

/* a2-a5: build up to n_levels levels: per level Algorithm-1 coloring
 * (reading A24), color-contiguous renumbering (stable sort by
 * (color, natural id)), then hash/skewness agglomeration (Algorithm 3,
 * P:577-627, readings A18-A23) to the next level.  *n_levels_built = levels
 * built.  Returns GMG_ESTALL (hierarchy usable, truncated) if a level merged
 * nothing.  Host-only; deterministic, bit-identical to the oracle's maps. */
gmg_status gmg_build_hierarchy(gmg_ctx *ctx, int n_levels, int *n_levels_built);

gmg_status gmg_get_level_info(gmg_ctx *ctx, int level, int64_t *n_cells, int *n_colors, int64_t *n_faces);

/* Host outputs (any may be NULL): color[n] (1..Nc, natural order),
 * perm[n] (internal position -> natural id), parent[n] (natural id of the
 * coarse cell on level+1, natural numbering of that level; -1 on the
 * coarsest level). */
gmg_status gmg_get_maps(gmg_ctx *ctx, int level, int32_t *color, int64_t *perm, int64_t *parent);

/* Coarse-level geometry as built (host, natural order of that level):
 * vol[n], left/right[nf], area_vec[dim][nf], face_ctr[dim][nf], n_gauss[nf];
 * any may be NULL. */
gmg_status gmg_get_level_geometry(gmg_ctx *ctx, int level, double *vol, double *centroid, int64_t *left,
                                  int64_t *right, double *area_vec, double *face_ctr, int8_t *n_gauss);

/* Device workspace: query bytes after gmg_build_hierarchy, then hand over a
 * device buffer of at least that size (16-byte aligned).  Uploads the
 * static level data (asynchronous on the stream). */
size_t gmg_workspace_bytes(gmg_ctx *ctx);
gmg_status gmg_set_workspace(gmg_ctx *ctx, void *dptr, size_t bytes);

/* Fine state W[nv][n] (natural order, host/device) and the free-stream /
 * farfield state W_inf[nv] (host). */
gmg_status gmg_set_state(gmg_ctx *ctx, const double *W, const double *W_inf);
/* State of any level (tests): W[nv][n_level] natural order, host/device. */
gmg_status gmg_set_level_state(gmg_ctx *ctx, int level, const double *W);
/* W_out[nv][n_level] natural order (host/device).  For a coarse level after
 * a V-cycle this is W0 + dW before prolongation. */
gmg_status gmg_get_state(gmg_ctx *ctx, int level, double *W_out);

/* Tests / inspection: one per-cell field of a level after the last call that
 * produced it, natural order, out[ncomp][n_level] (host/device):
 *   GMG_FIELD_W     the level's state W (nv comps; coarse: W0 + dW after a V-cycle)
 *   GMG_FIELD_W0    the linearisation state of the level's last smoothing step
 *                   (coarse: the restricted W0 of P:643-647)            (nv)
 *   GMG_FIELD_DW    the increment dW of the last smoothing step         (nv)
 *   GMG_FIELD_RS    the restricted residual Res*             (nv)
 *   GMG_FIELD_F     the forcing F = Res* - R(W0)            (nv)
 *   GMG_FIELD_RT    the level's last right-hand side / residual buffer  (nv)
 *   GMG_FIELD_ALPHA the level's DF alpha (coarse: min over children)    (1) */
enum { GMG_FIELD_W = 0, GMG_FIELD_W0 = 1, GMG_FIELD_DW = 2, GMG_FIELD_RS = 3, GMG_FIELD_F = 4, GMG_FIELD_RT = 5,
       GMG_FIELD_ALPHA = 6 };
gmg_status gmg_get_level_field(gmg_ctx *ctx, int level, int field, double *out);

/* df_mode 1: fine-level DF alpha[n] (natural order, host/device). */
gmg_status gmg_set_alpha(gmg_ctx *ctx, const double *alpha);

/* a6 + a10: residual R_l(W_l) = sum_f sigma S_f F_f (first-order KFVS, O4;
 * flux sum, reading A4) with BC ghosts, the DF helper alpha_i = prod
 * alpha_f^{M_f} (O5), r_f and Sigma_i (O6).  Outputs natural order,
 * nullable: R_out[nv][n], alpha_out[n], sigma_out[n]. */
gmg_status gmg_residual(gmg_ctx *ctx, int level, double *R_out, double *alpha_out, double *sigma_out);

/* Tests: set the right-hand side Rt[nv][n] and alpha[n] of a level
 * (natural order, host/device) used by the next gmg_smooth. */
gmg_status gmg_set_level_inputs(gmg_ctx *ctx, int level, const double *Rt, const double *alpha);

/* a10-a12: one smoothing step on `level` (O7): prepare r_f, Sigma, D at the
 * level's current W with its alpha (readings A2, A3, A5, A6), then n_sweeps
 * x (forward colors 1..Nc, backward Nc..1) of Eq.(gpu-forward-relaxation) /
 * Eq.(gpu-backward-relaxation) (Algorithm 2, readings
 * A1, A7), RHS = the level's Rt.  dW_out[nv][n] (natural order,
 * host/device, nullable).  W is NOT updated. */
gmg_status gmg_smooth(gmg_ctx *ctx, int level, int n_sweeps, double *dW_out);

/* a6-a16: n_cycles V-cycles (O8: fine explicit pre-smooth P:638-641,
 * restriction P:643-652, forcing P:662-665, coarse MC-LU-SGS, DF-limited
 * prolongation P:672-678; pre = 1, post = 0).  res_hist (host,
 * nullable) receives [n_cycles+1][nv] L2 norms of the fine residual
 * components at each cycle start plus one final entry (reading A26).
 * Captured once as a CUDA graph and replayed.  GMG_ENONFINITE if the
 * history is not finite. */
gmg_status gmg_vcycle(gmg_ctx *ctx, int n_cycles, double *res_hist);

/* Instrumentation for bench.py: run n_cycles V-cycles launching kernels
 * individually with CUDA events around every launch; ms_out[k] / count_out[k]
 * receive the summed device time and launch count of kernel class k
 * (GMG_K_* below).  bytes_out[k] = algorithmic bytes moved by class k over
 * the run.  Arrays of length GMG_K_COUNT. */
enum { GMG_K_FACE = 0, GMG_K_GATHER = 1, GMG_K_SWEEP = 2, GMG_K_RESTRICT = 3, GMG_K_PROLONG = 4,
       GMG_K_NORM = 5, GMG_K_HO_RECON = 6, GMG_K_HO_FLUX = 7, GMG_K_HALO = 8, GMG_K_COUNT = 9 };
/* (GMG_K_HALO: halo pack / unpack and ghost-record kernels of partitioned runs) */
gmg_status gmg_profile_vcycle(gmg_ctx *ctx, int n_cycles, double *ms_out, int64_t *count_out, double *bytes_out);

/* Sweep-only instrumentation: time one smoothing step's sweeps on `level`
 * (graph-replayed `reps` times) -- the same launches as the V-cycle's step,
 * including the W = W_lin + dW write of the last backward half-sweep, so the
 * level's W is overwritten; *ms = total device ms, *cell_updates =
 * N_l * 2 * n_sweeps * reps, *bytes = algorithmic bytes. */
gmg_status gmg_time_smooth(gmg_ctx *ctx, int level, int n_sweeps, int reps, double *ms, double *cell_updates,
                           double *bytes);

/* Pipelined host I/O (single rank): the same operations as gmg_set_state /
 * gmg_vcycle / gmg_get_state, enqueued without host synchronisation so that
 * the host<->device copies of consecutive calls overlap the V-cycles of the
 * others.  Copies run on two library-owned copy streams (one per direction)
 * through two device staging buffers per direction; the compute stream
 * orders everything else.
 *   gmg_set_state_async: W[nv][n] natural order; the host buffer (pinned for
 *     real overlap) must stay valid and unmodified until gmg_sync, and must be
 *     fully written by the host when the call is made (the call does not wait
 *     for GPU work that might still be filling a host buffer).  A DEVICE
 *     pointer is read after all work already enqueued on gmg_options.stream
 *     (the copy waits for it), so a tensor produced on that stream is safe.
 *   gmg_vcycle_async: n_cycles V-cycles + the residual norm (history kept on
 *     the device; no host read).
 *   gmg_get_state_async: W_out[nv][n] natural order, written by gmg_sync.
 *   gmg_sync: waits for everything enqueued; GMG_ENONFINITE if any cycle
 *     since the last sync produced a non-finite residual.
 * Results are bit-identical to the synchronous calls in the same order.
 * GMG_EINVAL for nranks > 1 (the synchronous calls serve ranks). */
gmg_status gmg_set_state_async(gmg_ctx *ctx, const double *W, const double *W_inf);
gmg_status gmg_vcycle_async(gmg_ctx *ctx, int n_cycles);
gmg_status gmg_get_state_async(gmg_ctx *ctx, double *W_out);
gmg_status gmg_sync(gmg_ctx *ctx);

/* Rank-local variants (any nranks, one domain per rank): W_owned[nv][n_own]
 * holds only this rank's owned fine cells, column p = owned cell p in the
 * order gmg_get_halo(level 0) lists them ("owned"); ghosts are refreshed by
 * the V-cycle's own halo exchange.  Same buffer-lifetime rules as above. */
gmg_status gmg_set_state_owned_async(gmg_ctx *ctx, const double *W_owned, const double *W_inf);
gmg_status gmg_get_state_owned_async(gmg_ctx *ctx, double *W_owned_out);

/* Number of kernels one V-cycle launches (graph nodes). */
int64_t gmg_vcycle_launches(gmg_ctx *ctx);
/* Sweep cell-updates (one cell's increment solved once) EXECUTED per V-cycle
 * (the repeated phases dropped by skip_repeat are not counted). */
int64_t gmg_vcycle_visits(gmg_ctx *ctx);

/* a5: recursive coordinate bisection of the cell centroids (host, natural
 * order; centroid[dim][n]) into nparts partitions -> part_out[n] in
 * 0..nparts-1.  Deterministic (ties broken by natural id), so every rank
 * computes the same partition.  Pure host function, no context needed. */
gmg_status gmg_partition_rcb(int64_t n_cells, int dim, const double *centroid, int nparts, int32_t *part_out);

/* a5/a13: halo plan of local domain `dom` (0 when nranks > 1) on `level`,
 * for tests.  Sizes first (any pointer NULL): *n_owned, *n_ghost, *n_peers,
 * *n_send, *n_recv.  Then (all non-NULL) the natural ids of the owned cells
 * (local order), of the ghosts, the peer ranks, and the send / recv lists as
 * natural ids with their group offsets send_off/recv_off[n_colors*n_peers+1]
 * (groups ordered (color, peer), natural id ascending inside a group). */
gmg_status gmg_get_halo(gmg_ctx *ctx, int level, int dom, int64_t *n_owned, int64_t *n_ghost, int *n_peers,
                        int64_t *n_send, int64_t *n_recv, int64_t *owned, int64_t *ghost, int32_t *peers,
                        int64_t *send_nat, int64_t *send_off, int64_t *recv_nat, int64_t *recv_off);

/* NEXT-3, fused P2P halo between ranks (environment GMG_P2P=1, nranks > 1;
 * SURVEY §8(f)).  The sweep that computes a boundary cell's increment stores
 * it straight into the ghost record on every peer GPU that holds a copy
 * (NVLink peer memory) and publishes its phase count into the peer's flags --
 * no pack / ncclSend / ncclRecv / unpack per color.  Setup, after
 * gmg_set_workspace on every rank:
 *   gmg_p2p_layout(ctx, out): out[0 .. n_levels-1] = byte offsets of this
 *     rank's record arrays inside its workspace, out[n_levels] = offset of its
 *     flag array; (n_levels + 1) int64.
 *   gmg_p2p_import(ctx, handles, base_off, layouts): for every rank r
 *     (nranks entries; this rank's own entry is ignored): handles + 64 r = its
 *     cudaIpcMemHandle_t of the allocation holding its workspace, base_off[r]
 *     = byte offset of that workspace inside the allocation, layouts +
 *     (n_levels + 1) r = its gmg_p2p_layout output.  Opens the peers'
 *     allocations (cudaIpcOpenMemHandle) and stores their record / flag
 *     addresses; GMG_ECUDA if a peer cannot be mapped.  Until it succeeds the
 *     NCCL exchange is used.  The binding (gmg.Solver) does this exchange with
 *     torch.distributed.all_gather_object.  (Untested in this build on more
 *     than one GPU; the same kernels run between the local domains of one
 *     process -- tests/test_gpu_partitioned.py.) */
gmg_status gmg_p2p_layout(gmg_ctx *ctx, int64_t *out);
/* Host view of the fused-halo targets of domain `dom` on `level` (tests):
 * *n_targets first (other pointers NULL), then off[n_owned+1] (CSR over the
 * owned cells in local order), peer_slot[n_targets] (index into the domain's
 * ascending peer list), ghost_local[n_targets] (the peer's local index of its
 * ghost copy).  GMG_ESTATE unless built with GMG_P2P=1 and > 1 partition. */
gmg_status gmg_get_p2p_targets(gmg_ctx *ctx, int level, int dom, int64_t *n_targets, int32_t *off,
                               int32_t *peer_slot, int32_t *ghost_local);
gmg_status gmg_p2p_import(gmg_ctx *ctx, const void *handles, const int64_t *base_off, const int64_t *layouts);
/* ---------------------------------------------------------------------------
 * NEXT-1: third-order compact GKS fine operator (fine_operator = 1,
 * DESIGN.md §12).  Single domain only (GMG_EINVAL otherwise).
 * ------------------------------------------------------------------------- */

/* High-order fine-level geometry (host, natural order; after gmg_load_mesh,
 * before gmg_workspace_bytes): m2[nq][n] central second moments
 * (1/|Omega|) int (x - x_c)_a (x - x_c)_b dV, components a <= b row major
 * (2D xx, xy, yy; 3D xx, xy, xz, yy, yz, zz) -- the p2 moments of P:318-322;
 * gp[dim][G][nf] face Gauss points and gw[G][nf] weights summing to 1 per
 * face (3 per triangle, 4 per quad, 2 per 2D segment; G = 4 in
 * 3D, 2 in 2D; unused slots weight 0).  Copied; the caller keeps ownership.
 * GMG_EINVAL on a bad G / NULL pointer, GMG_ESTATE before gmg_load_mesh. */
gmg_status gmg_load_ho_geometry(gmg_ctx *ctx, const double *m2, int G, const double *gp, const double *gw);

/* Cell-averaged slopes G[nv][dim][n] (component q, direction e at (q*dim+e)*n
 * + i) and the carried DF alpha[n] (host/device, natural order); NULL = the
 * initial values of reading C1 (G = 0, alpha = 1).  gmg_set_state does not
 * touch them. */
gmg_status gmg_set_ho_state(gmg_ctx *ctx, const double *G, const double *alpha);
gmg_status gmg_get_ho_state(gmg_ctx *ctx, double *G_out, double *alpha_out);

/* One evaluation of the operator at the current (W, G, alpha), no state
 * change (readings C2-C13): R_out[nv][n] time-averaged flux sum (C11),
 * G_out[nv][dim][n] the evolved slopes times DF (C13), alpha_out[n] (C7),
 * sigma_out[n] (C8); any may be NULL.  Natural order, host/device. */
gmg_status gmg_ho_residual(gmg_ctx *ctx, double *R_out, double *G_out, double *alpha_out, double *sigma_out);

/* The reconstruction alone (C2-C6): poly_out[nv*nc][n] with nc = 1 + dim + nq,
 * per component (c0, lin[dim], quad[nq]) of p(x) = c0 + lin . y + sum_k quad_k
 * y_a y_b, y = x - x_cell (natural order); flags_out[n] bit 0 = p2 used
 * (positivity, C6b, is applied per Gauss point in the flux).  Either may be
 * NULL. */
gmg_status gmg_ho_recon(gmg_ctx *ctx, double *poly_out, int32_t *flags_out);

/* Test only: one smoothing step (as gmg_smooth) of ALL local domains
 * (local_domains >= 2, GMG_P2P=1) in ONE cooperative launch with one block
 * group per domain, so that the fused-P2P-halo protocol (wait for the peers'
 * phase counts, sweep + peer stores, publish) runs with the domains truly
 * concurrent -- the single-GPU stand-in for ranks that wait on one another.
 * dW_out as gmg_smooth (nullable). */
gmg_status gmg_p2p_emulate_smooth(gmg_ctx *ctx, int level, int n_sweeps, double *dW_out);

const char *gmg_last_error(gmg_ctx *ctx); /* valid until the next call on ctx */
void gmg_destroy(gmg_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* GMG_H */
