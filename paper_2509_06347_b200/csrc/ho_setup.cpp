// ho_setup.cpp -- host setup of the third-order compact GKS fine operator
// (DESIGN.md §12): local-order geometry, per-cell face
// lists, and the per-cell p2 operator of the constrained least squares of
// P:312-346 (reading C2).  Geometry only -- computed once per hierarchy.
//
// The p2 coefficients of cell i are a linear function of its stencil data,
//   a = sum_m [ Pq_m (Q_m - Q_i) + sum_e Pg_{m,e} (Q_e)_m ],
// so the KKT system [[2 L^T L, C^T], [C, 0]] is factored here once and its
// solution columns stored; the device reconstruction is then one small
// matrix-vector product per neighbour (ho.cu k_ho_recon).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "gmg_internal.h"

namespace gmg {

namespace {

// LU with partial pivoting of A [m][m] (row major, in place); piv [m].
bool lu_factor(int m, std::vector<double> &A, std::vector<int> &piv)
{
    piv.resize(m);
    for (int k = 0; k < m; ++k) {
        int p = k;
        for (int r = k + 1; r < m; ++r)
            if (std::fabs(A[r * m + k]) > std::fabs(A[p * m + k])) p = r;
        piv[k] = p;
        if (A[p * m + k] == 0.0) return false;
        if (p != k)
            for (int c = 0; c < m; ++c) std::swap(A[k * m + c], A[p * m + c]);
        const double inv = 1.0 / A[k * m + k];
        for (int r = k + 1; r < m; ++r) {
            const double f = A[r * m + k] * inv;
            A[r * m + k] = f;
            for (int c = k + 1; c < m; ++c) A[r * m + c] -= f * A[k * m + c];
        }
    }
    return true;
}

void lu_solve(int m, const std::vector<double> &A, const std::vector<int> &piv, double *b)
{
    for (int k = 0; k < m; ++k) std::swap(b[k], b[piv[k]]);
    for (int r = 1; r < m; ++r)
        for (int c = 0; c < r; ++c) b[r] -= A[r * m + c] * b[c];
    for (int r = m - 1; r >= 0; --r) {
        for (int c = r + 1; c < m; ++c) b[r] -= A[r * m + c] * b[c];
        b[r] /= A[r * m + r];
    }
}

}  // namespace

// one domain: local geometry over owned + ghost cells, face slots of the
// owned cells, their p2 operators
static gmg_status ho_prepare_domain(gmg_ctx *ctx, const HoHost &HH, Domain &dm)
{
    HoLocal &H = dm.ho;
    const HostLevel &G = ctx->lv[0];
    const DomLevel &D0 = dm.lv[0];
    const int d = G.dim, nq = d * (d + 1) / 2, nk = d + nq, Gs = HH.G;
    const int64_t n = D0.n_own, nl = D0.n_loc, nf = D0.nf, N = G.n, NF = G.nf;
    // local geometry (AoS), owned + ghosts
    H.ctr.assign((size_t)nl * d, 0.0);
    H.m2l.assign((size_t)nl * nq, 0.0);
    for (int64_t i = 0; i < nl; ++i) {
        const int64_t g = D0.l2n[i];
        for (int e = 0; e < d; ++e) H.ctr[i * d + e] = G.ctr[(size_t)e * N + g];
        for (int k = 0; k < nq; ++k) H.m2l[i * nq + k] = HH.m2[(size_t)k * N + g];
    }
    H.gpl.assign((size_t)nf * Gs * d, 0.0);
    H.gwl.assign((size_t)nf * Gs, 0.0);
    for (int64_t f = 0; f < nf; ++f) {
        const int64_t g = D0.fnat[f];
        for (int k = 0; k < Gs; ++k) {
            H.gwl[f * Gs + k] = HH.gw[(size_t)k * NF + g];
            for (int e = 0; e < d; ++e) H.gpl[(f * Gs + k) * d + e] = HH.gp[((size_t)e * Gs + k) * NF + g];
        }
    }
    // flux lanes: one lane per Gauss point (no idle padding lanes of triangles), a face's points on
    // consecutive lanes of one warp (its first lane reduces them), faces in local order
    H.glane.clear();
    for (int64_t f = 0; f < nf; ++f) {
        int c = 0;
        for (int k = 0; k < Gs; ++k) c += H.gwl[f * Gs + k] != 0.0;
        if (c == 0) continue;
        const int64_t pos = (int64_t)H.glane.size() / 2;
        if (pos % 32 + c > 32)
            for (int64_t p = pos; p % 32 != 0; ++p) { H.glane.push_back(-1); H.glane.push_back(0); }
        bool first = true;
        for (int k = 0; k < Gs; ++k) {
            if (H.gwl[f * Gs + k] == 0.0) continue;
            H.glane.push_back((int32_t)(f * Gs + k));
            H.glane.push_back(first ? c : 0);
            first = false;
        }
    }
    // owned cell -> faces, ascending natural face id (the oracle's order)
    H.hfoff.assign(n + 1, 0);
    for (int64_t f = 0; f < nf; ++f) {
        if (D0.fl[f] < n) H.hfoff[D0.fl[f] + 1]++;
        if (D0.fr[f] >= 0 && D0.fr[f] < n) H.hfoff[D0.fr[f] + 1]++;
    }
    for (int64_t i = 0; i < n; ++i) H.hfoff[i + 1] += H.hfoff[i];
    H.hface.assign(H.hfoff[n], 0);
    {
        std::vector<int> fill(H.hfoff.begin(), H.hfoff.end() - 1);
        for (int64_t f = 0; f < nf; ++f) {
            if (D0.fl[f] < n) H.hface[fill[D0.fl[f]]++] = (int)(f + 1);
            if (D0.fr[f] >= 0 && D0.fr[f] < n) H.hface[fill[D0.fr[f]]++] = -(int)(f + 1);
        }
        for (int64_t i = 0; i < n; ++i)
            std::sort(H.hface.begin() + H.hfoff[i], H.hface.begin() + H.hfoff[i + 1], [&](int a, int b) {
                return D0.fnat[std::abs(a) - 1] < D0.fnat[std::abs(b) - 1];
            });
    }
    // per-slot records: A outward from the cell, (neighbour | -(patch+1), local face)
    H.hrec.assign((size_t)H.hfoff[n] * 4, 0.0);
    for (int64_t i = 0; i < n; ++i)
        for (int s = H.hfoff[i]; s < H.hfoff[i + 1]; ++s) {
            const int f = std::abs(H.hface[s]) - 1;
            const double sg = H.hface[s] > 0 ? 1.0 : -1.0;
            const int64_t g = D0.fnat[f];
            for (int e = 0; e < d; ++e) H.hrec[(size_t)s * 4 + e] = sg * G.avec[(size_t)e * NF + g];
            int32_t jf[2] = {D0.fr[f] < 0 ? D0.fr[f] : (D0.fl[f] == i ? D0.fr[f] : D0.fl[f]), (int32_t)f};
            std::memcpy(&H.hrec[(size_t)s * 4 + 3], jf, sizeof jf);
        }
    // p2 operators (C2, C3: >= d + 1 interior neighbours)
    std::vector<int> nnb(n, 0);
    for (int64_t i = 0; i < n; ++i)
        for (int s = H.hfoff[i]; s < H.hfoff[i + 1]; ++s) nnb[i] += D0.fr[std::abs(H.hface[s]) - 1] >= 0;
    // per neighbour (d + 1) columns of nk, padded to a multiple of 4 doubles (32-byte loads)
    const int pst = ((d + 1) * nk + 3) & ~3;
    H.poff.assign(n + 1, 0);
    const int p2min = ctx->opt.ho_p2min > 0 ? ctx->opt.ho_p2min : d + 1;   // C3 / C3b
    for (int64_t i = 0; i < n; ++i) H.poff[i + 1] = H.poff[i] + (nnb[i] >= p2min ? nnb[i] * pst : 0);
    H.P.assign((size_t)H.poff[n], 0.0);
    std::vector<char> ok(n, 1);
    auto m2at = [&](int64_t c, int a, int b) {
        if (a > b) std::swap(a, b);
        int k = 0;
        for (int x = 0; x < d; ++x)
            for (int y = x; y < d; ++y) {
                if (x == a && y == b) return H.m2l[c * nq + k];
                ++k;
            }
        return 0.0;
    };
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i) {
        if (H.poff[i + 1] == H.poff[i]) continue;
        const int nb = nnb[i], m = nk + nb, nlsq = d * nb;
        std::vector<double> Cm((size_t)nb * nk, 0.0), L((size_t)nlsq * nk, 0.0);
        int r = 0;
        for (int s = H.hfoff[i]; s < H.hfoff[i + 1]; ++s) {
            const int f = std::abs(H.hface[s]) - 1;
            if (D0.fr[f] < 0) continue;
            const int64_t j = D0.fl[f] == i ? D0.fr[f] : D0.fl[f];
            double dl[3] = {0, 0, 0};
            for (int e = 0; e < d; ++e) dl[e] = H.ctr[j * d + e] - H.ctr[i * d + e];
            int k = 0;
            for (int e = 0; e < d; ++e) Cm[r * nk + e] = dl[e];
            for (int a = 0; a < d; ++a)
                for (int b = a; b < d; ++b, ++k) Cm[r * nk + d + k] = (m2at(j, a, b) + dl[a] * dl[b]) - m2at(i, a, b);
            for (int e = 0; e < d; ++e) {
                double *row = &L[(size_t)(r * d + e) * nk];
                row[e] = 1.0;
                int kk = 0;
                for (int a = 0; a < d; ++a)
                    for (int b = a; b < d; ++b, ++kk) row[d + kk] = (a == e ? dl[b] : 0.0) + (b == e ? dl[a] : 0.0);
            }
            ++r;
        }
        std::vector<double> K((size_t)m * m, 0.0);
        for (int x = 0; x < nk; ++x) {
            for (int y = 0; y < nk; ++y) {
                double sum = 0.0;
                for (int q = 0; q < nlsq; ++q) sum += L[(size_t)q * nk + x] * L[(size_t)q * nk + y];
                K[x * m + y] = 2.0 * sum;
            }
            for (int q = 0; q < nb; ++q) {
                K[x * m + nk + q] = Cm[q * nk + x];
                K[(nk + q) * m + x] = Cm[q * nk + x];
            }
        }
        std::vector<int> piv;
        if (!lu_factor(m, K, piv)) { ok[i] = 0; continue; }
        double *out = &H.P[H.poff[i]];
        std::vector<double> rhs(m);
        for (int q = 0; q < nb; ++q) {
            // column of (Q_m - Q_i): unit right-hand side in constraint row q
            std::fill(rhs.begin(), rhs.end(), 0.0);
            rhs[nk + q] = 1.0;
            lu_solve(m, K, piv, rhs.data());
            double *col = out + (size_t)q * pst;
            for (int k = 0; k < nk; ++k) col[k] = rhs[k];
            // columns of the neighbour's averaged slopes: 2 L^T e_(q,e)
            for (int e = 0; e < d; ++e) {
                std::fill(rhs.begin(), rhs.end(), 0.0);
                for (int k = 0; k < nk; ++k) rhs[k] = 2.0 * L[(size_t)(q * d + e) * nk + k];
                lu_solve(m, K, piv, rhs.data());
                for (int k = 0; k < nk; ++k) col[(1 + e) * nk + k] = rhs[k];
            }
        }
    }
    // a singular system (not expected with >= d + 1 neighbours) -> p1 only
    std::vector<int> poff2(n + 1, 0);
    for (int64_t i = 0; i < n; ++i) poff2[i + 1] = poff2[i] + ((H.poff[i + 1] > H.poff[i] && ok[i]) ? H.poff[i + 1] - H.poff[i] : 0);
    if (poff2[n] != H.poff[n]) {
        std::vector<double> P2((size_t)poff2[n]);
        for (int64_t i = 0; i < n; ++i)
            if (poff2[i + 1] > poff2[i]) std::memcpy(&P2[poff2[i]], &H.P[H.poff[i]], sizeof(double) * (poff2[i + 1] - poff2[i]));
        H.P.swap(P2);
        H.poff.swap(poff2);
    }
    H.n_p2 = 0;
    for (int64_t i = 0; i < n; ++i) H.n_p2 += H.poff[i + 1] > H.poff[i];
    // algorithmic bytes per launch: each datum moved once
    const int nv = d + 2, nc = 1 + nk;
    int64_t nint = 0, nslots = H.hfoff[n], gpts = 0;
    for (int64_t f = 0; f < nf; ++f) {
        nint += D0.fr[f] >= 0;
        for (int k = 0; k < Gs; ++k) gpts += H.gwl[f * Gs + k] != 0.0;
    }
    H.n_gauss_pts = gpts;
    H.bytes_sr = (double)nf * (d * 8 + 8 + 8) + (double)(nint + nf) * nv * 8;
    H.bytes_recon = (double)n * (nv * 8 + 8 + 8 + nq * 8 + 4 * 2 + nv * nc * 8 + 8 + 8) +
                    (double)nslots * (32 + 8) + (double)nint * 2 * (nv * 8 + nv * d * 8) + (double)H.P.size() * 8;
    H.bytes_flux = (double)nf * (8 + d * 8 + Gs * (d + 1) * 8 + 12 * 8) + (double)(nint + nf) * (nv * nc * 8 + d * 8 + 8);
    H.bytes_gather = (double)nslots * (4 + 32 + (2 * nv + 1) * 8) + (double)n * (8 + 8 + 4 * 2 + nv * 8 * 2 + nv * d * 8 + 8);
    return GMG_OK;
}

gmg_status ho_prepare(gmg_ctx *ctx)
{
    HoHost &HH = *ctx->ho;
    if (HH.prepared) return GMG_OK;
    for (Domain &dm : ctx->dom) {
        const gmg_status st = ho_prepare_domain(ctx, HH, dm);
        if (st) return st;
    }
    HH.prepared = true;
    return GMG_OK;
}

}  // namespace gmg
