// device_common.cuh -- structures and inline device helpers shared by the
// kernels of libgmg (kernels.cuh) and of the NEXT-1 operator (ho.cu): record
// layouts, Phys / BCs, vector loads and stores, pressure, ghost states, the
// per-side primitive view.  Header-only, no __global__ functions (each .cu
// translation unit defines its own kernels).
#pragma once
#include <cuda_runtime.h>

#include "gmg_internal.h"

namespace gmg {

// Sweep state layout (doubles).  The smoother works on W' = W_lin + dW (the
// linearisation state plus the current increment), DESIGN.md §6 "W'
// formulation".  A state array (W' and W_lin) of n_loc cells holds nv * n_loc
// doubles: 2D [n_loc][4] = (rho, m, rho E), one 32-byte sector per cell; 3D
// split [n_loc][4] = (rho, m) followed by [n_loc] = rho E -- a neighbour
// gather is one 256-bit load plus one 64-bit load (40 B, no padding; the
// rho E words of neighbouring cells share sectors), round 2 v24.
//  * kXr -- own-cell record [X_0..X_{nv-1}, c (, pad)], X = W_lin - Rt/D + c P,
//    c = alpha/(2D), written by the first forward half-sweep of a smoothing step.
template <int D> struct Wp;
template <> struct Wp<3> { static constexpr bool SPLIT = true; };
template <> struct Wp<2> { static constexpr bool SPLIT = false; };
constexpr int kXr = 6;
// per-slot record: A_0..A_{D-1}, S r at [D]
constexpr int kSlotRec = 4;

struct Phys {
    double gamma, gm1, K, omega;
};
struct BCs {
    double winf[5];
    int kind[16];
};

enum : int {
    G_FLUX = 1,       // accumulate R = sum sigma S F and alpha = prod alpha_f^M from the face buffers
    G_NORM = 2,       // per-block partial sums of R_q^2
    G_EXPLICIT = 4,   // W -= (cfl_exp / Sigma) R            (Eq.(smo), reading A9)
    G_WRITE_RT = 8,   // Rt = R (+ F if G_ADD_F)
    G_ADD_F = 16,
    G_SET_F = 32,     // F = Rs - R
    G_ALPHA = 64,     // alpha = prod alpha_f^{M_f}          (O5)
    G_PREPARE = 128,  // dc = (1/D, alpha/(2D)) of the hybrid diagonal (O6)
    G_SIGMA = 256,    // store Sigma
    G_COPY_W = 1024,  // W_lin = W (fine-level smoothing)
    G_BETA = 2048,    // prepare with the fixed relaxation factor beta instead of alpha (df_mode 3)
};

struct GArgs {
    int flags;
    double cfl_imp, cfl_exp;
    double *Wexp;
    double *partial;
    double beta;
};

// Programmatic dependent launch (sm_90+): every V-cycle kernel may be
// launched while its predecessor drains; it waits here until the predecessor
// grid has completed and its writes are visible, and immediately lets its
// own successor be scheduled.  No-ops when launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter()
{
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <int NV>
__device__ __forceinline__ void ld_vec(const double *__restrict__ q, double *w)
{
#pragma unroll
    for (int k = 0; k < NV; ++k) w[k] = __ldg(q + k);
}

// 256-bit global accesses (sm_100: LDG.E.ENL2.256 / STG.E.ENL2.256); p 32-byte aligned
__device__ __forceinline__ void ld4nc(const double *p, double *v)
{
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}
// L1 policy hints of the sweep: slot records and the own (X, c) record are
// read once (no L1 allocation), the gathered neighbour records are the ones
// worth keeping (evict last)
__device__ __forceinline__ void ld4na(const double *p, double *v)
{
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}
__device__ __forceinline__ void ld4el(const double *p, double *v)
{
    asm volatile("ld.global.nc.L1::evict_last.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}
__device__ __forceinline__ void ld2na(const double *p, double *v)
{
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v[0]), "=d"(v[1]) : "l"(p));
}
__device__ __forceinline__ void ld4cg(const double *p, double *v)
{
    asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p) : "memory");
}
// 128-bit accesses (p 16-byte aligned)
__device__ __forceinline__ void ld2nc(const double *p, double *v)
{
    asm volatile("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(v[0]), "=d"(v[1]) : "l"(p));
}
__device__ __forceinline__ void ld2cg(const double *p, double *v)
{
    asm volatile("ld.global.cg.v2.f64 {%0,%1}, [%2];" : "=d"(v[0]), "=d"(v[1]) : "l"(p) : "memory");
}
__device__ __forceinline__ void st2(double *p, const double *v)
{
    asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(v[0]), "d"(v[1]) : "memory");
}
__device__ __forceinline__ void st4(double *p, const double *v)
{
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
                 : "memory");
}

// Cell record i of an AoS array [n][NV] (base 256-B aligned).  NV = 4: one
// 256-bit access.  NV = 5 (40 B): three accesses instead of five -- a 128-bit
// pair starting at the first 16-B boundary of the record (element 0 for even
// i, element 1 for odd i), a second pair after it and the remaining scalar;
// every lane issues the same three instructions (no divergence on parity).
// NC: the read-only path (the array is not written by the kernel).
template <int NV, bool NC = false>
__device__ __forceinline__ void ld_rec(const double *base, size_t i, double *w)
{
    const double *p = base + (size_t)NV * i;
    if constexpr (NV == 4) {
        if constexpr (NC) ld4nc(p, w);
        else {
            asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                         : "=d"(w[0]), "=d"(w[1]), "=d"(w[2]), "=d"(w[3]) : "l"(p) : "memory");
        }
    } else {
        static_assert(NV == 5, "records of 4 or 5 doubles");
        const int o = (int)(i & 1);
        double a[2], b[2], s;
        if constexpr (NC) {
            ld2nc(p + o, a);
            ld2nc(p + o + 2, b);
            s = __ldg(p + (o ? 0 : 4));
        } else {
            const double2 va = *reinterpret_cast<const double2 *>(p + o);
            const double2 vb = *reinterpret_cast<const double2 *>(p + o + 2);
            a[0] = va.x; a[1] = va.y; b[0] = vb.x; b[1] = vb.y;
            s = p[o ? 0 : 4];
        }
        w[0] = o ? s : a[0];
        w[1] = o ? a[0] : a[1];
        w[2] = o ? a[1] : b[0];
        w[3] = o ? b[0] : b[1];
        w[4] = o ? b[1] : s;
    }
}
template <int NV>
__device__ __forceinline__ void st_rec(double *base, size_t i, const double *w)
{
    double *p = base + (size_t)NV * i;
    if constexpr (NV == 4) {
        st4(p, w);
    } else {
        static_assert(NV == 5, "records of 4 or 5 doubles");
        const int o = (int)(i & 1);
        const double a[2] = {o ? w[1] : w[0], o ? w[2] : w[1]};
        const double b[2] = {o ? w[3] : w[2], o ? w[4] : w[3]};
        st2(p + o, a);
        st2(p + o + 2, b);
        p[o ? 0 : 4] = o ? w[0] : w[4];
    }
}

// one state into cell i of a state array of nloc cells (layout above)
template <int D>
__device__ __forceinline__ void st_state(double *base, size_t nloc, size_t i, const double *w)
{
    st4(base + 4 * i, w);
    if constexpr (D == 3) base[4 * nloc + i] = w[4];
}

// cell i of a state array of nloc cells -> w[nv] (one 256-bit load, plus one
// 64-bit load in 3D); CG: L2-coherent (states written by other blocks of the
// same launch), else the non-coherent path (EL: L1 evict-last)
template <int D, bool CG = false, bool EL = false>
__device__ __forceinline__ void ld_state(const double *base, size_t nloc, size_t i, double *w)
{
    if constexpr (CG) ld4cg(base + 4 * i, w);
    else if constexpr (EL) ld4el(base + 4 * i, w);
    else ld4nc(base + 4 * i, w);
    if constexpr (D == 3) w[4] = CG ? __ldcg(base + 4 * nloc + i) : __ldg(base + 4 * nloc + i);
}

template <int D>
__device__ __forceinline__ double pressure(const double *w, double gm1)
{
    double m2 = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) m2 += w[1 + k] * w[1 + k];
    return gm1 * (w[D + 1] - 0.5 * m2 / w[0]);
}

// ghost state of a boundary face (O4, reading A25); n = unit outward normal
template <int D>
__device__ __forceinline__ void ghost(int kind, const double *wi, const BCs &bc, const double *n, double *wg)
{
    if (kind == GMG_FARFIELD) {
#pragma unroll
        for (int q = 0; q < D + 2; ++q) wg[q] = bc.winf[q];
        return;
    }
#pragma unroll
    for (int q = 0; q < D + 2; ++q) wg[q] = wi[q];
    if (kind == GMG_SLIP) {
        double mn = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) mn += wi[1 + k] * n[k];
#pragma unroll
        for (int k = 0; k < D; ++k) wg[1 + k] = wi[1 + k] - 2.0 * mn * n[k];
    } else if (kind == GMG_NOSLIP) {
#pragma unroll
        for (int k = 0; k < D; ++k) wg[1 + k] = -wi[1 + k];
    }
}

// primitive view of one face side, shared by the KFVS flux, the DF helper
// and nothing else recomputes it (one 1/rho, one 1/p, one rsqrt per side)
template <int D>
struct Side {
    double rho, ir, u[D], U, u2, p, ip;
};
template <int D>
__device__ __forceinline__ Side<D> side_of(const double *w, const double *n, double gm1)
{
    Side<D> s;
    s.rho = w[0];
    s.ir = 1.0 / s.rho;
    s.U = 0.0;
    s.u2 = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) { s.u[k] = w[1 + k] * s.ir; s.U += s.u[k] * n[k]; s.u2 += s.u[k] * s.u[k]; }
    s.p = gm1 * (w[D + 1] - 0.5 * s.rho * s.u2);
    s.ip = 1.0 / s.p;
    return s;
}

}  // namespace gmg
