// setup.cpp -- host-side setup of libgmg:
// mesh ingest + validation, Algorithm-1 coloring, color-contiguous
// renumbering, hash/skewness agglomeration, coarse geometry and the SELL-32
// slot layouts the kernels consume.
//
// Deterministic and bit-identical to the oracle's maps by construction of
// the *specification* (SURVEY §8(c) O1-O3): every floating-point expression
// that decides an integer (skewness test) or feeds the next level's decision
// (coarse geometry) is evaluated in the order the spec writes it, compiled
// with -ffp-contract=off.  This is an independent implementation: it shares
// no code with oracle/.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <deque>
#include <numeric>
#include <stdexcept>
#include <tuple>

#include "gmg_internal.h"

namespace gmg {

namespace {
struct Csr {
    std::vector<int64_t> off, idx;
};

// interior-face adjacency (neighbour cells), each list sorted by id
Csr neighbours(const HostLevel &L)
{
    Csr g;
    g.off.assign(L.n + 1, 0);
    for (int64_t f = 0; f < L.nf; ++f)
        if (L.right[f] >= 0) { g.off[L.left[f] + 1]++; g.off[L.right[f] + 1]++; }
    std::partial_sum(g.off.begin(), g.off.end(), g.off.begin());
    g.idx.resize(g.off[L.n]);
    std::vector<int64_t> pos(g.off.begin(), g.off.end() - 1);
    for (int64_t f = 0; f < L.nf; ++f)
        if (L.right[f] >= 0) { g.idx[pos[L.left[f]]++] = L.right[f]; g.idx[pos[L.right[f]]++] = L.left[f]; }
    for (int64_t i = 0; i < L.n; ++i) std::sort(g.idx.begin() + g.off[i], g.idx.begin() + g.off[i + 1]);
    return g;
}

// cell -> incident faces, ascending face id
Csr incident_faces(const HostLevel &L)
{
    Csr g;
    g.off.assign(L.n + 1, 0);
    for (int64_t f = 0; f < L.nf; ++f) {
        g.off[L.left[f] + 1]++;
        if (L.right[f] >= 0) g.off[L.right[f] + 1]++;
    }
    std::partial_sum(g.off.begin(), g.off.end(), g.off.begin());
    g.idx.resize(g.off[L.n]);
    std::vector<int64_t> pos(g.off.begin(), g.off.end() - 1);
    for (int64_t f = 0; f < L.nf; ++f) {
        g.idx[pos[L.left[f]]++] = f;
        if (L.right[f] >= 0) g.idx[pos[L.right[f]]++] = f;
    }
    return g;
}

inline double norm_area(int dim, const double *A)
{
    // |A| with the sum order fixed by O3 step 5: ((a0 a0) + a1 a1) + a2 a2
    double s = A[0] * A[0];
    s = s + A[1] * A[1];
    if (dim == 3) s = s + A[2] * A[2];
    return std::sqrt(s);
}
}  // namespace

// ------------------------------------------------------------------ a1
gmg_status load_mesh(gmg_ctx *ctx, int64_t n, const double *vol, const double *ctr, int64_t nf,
                     const int64_t *left, const int64_t *right, const double *avec, const double *fctr,
                     const int8_t *ng, const int32_t *part)
{
    const int d = ctx->opt.dim;
    HostLevel L;
    L.dim = d;
    L.n = n;
    L.nf = nf;
    L.vol.assign(vol, vol + n);
    L.ctr.assign(ctr, ctr + (size_t)d * n);
    L.left.assign(left, left + nf);
    L.right.assign(right, right + nf);
    L.avec.assign(avec, avec + (size_t)d * nf);
    L.fctr.assign(fctr, fctr + (size_t)d * nf);
    L.ngauss.assign(ng, ng + nf);
    if (part) L.part.assign(part, part + n);
    for (int64_t i = 0; i < n; ++i)
        if (!(L.vol[i] > 0.0)) { ctx->err = "cell " + std::to_string(i) + " has non-positive volume"; return GMG_ETOPO; }
    for (int64_t f = 0; f < nf; ++f) {
        int64_t l = L.left[f], r = L.right[f];
        if (l < 0 || l >= n) { ctx->err = "face " + std::to_string(f) + ": left cell out of range"; return GMG_ETOPO; }
        if (r >= n || r == l) { ctx->err = "face " + std::to_string(f) + ": bad right cell"; return GMG_ETOPO; }
        if (r < 0 && (-r - 1) >= ctx->n_patches) { ctx->err = "face " + std::to_string(f) + ": bad patch"; return GMG_ETOPO; }
        if (L.ngauss[f] < 1) { ctx->err = "face " + std::to_string(f) + ": n_gauss < 1"; return GMG_ETOPO; }
    }
    // closure sum_f sigma A_f = 0 per cell
    std::vector<double> acc((size_t)d * n, 0.0), sarea(n, 0.0);
    for (int64_t f = 0; f < nf; ++f) {
        double S = norm_area(d, std::vector<double>{L.avec[f], L.avec[nf + f], d == 3 ? L.avec[2 * nf + f] : 0.0}.data());
        for (int k = 0; k < d; ++k) acc[(size_t)k * n + L.left[f]] += L.avec[(size_t)k * nf + f];
        sarea[L.left[f]] += S;
        if (L.right[f] >= 0) {
            for (int k = 0; k < d; ++k) acc[(size_t)k * n + L.right[f]] -= L.avec[(size_t)k * nf + f];
            sarea[L.right[f]] += S;
        }
    }
    for (int64_t i = 0; i < n; ++i) {
        double e = 0.0;
        for (int k = 0; k < d; ++k) e += acc[(size_t)k * n + i] * acc[(size_t)k * n + i];
        if (std::sqrt(e) > 1e-10 * sarea[i]) { ctx->err = "cell " + std::to_string(i) + " is not closed"; return GMG_ETOPO; }
    }
    ctx->lv.clear();
    ctx->lv.push_back(std::move(L));
    return GMG_OK;
}

// ------------------------------------------------------------------ a2
// Algorithm 1, reading A24: FIFO waves from cell 0, neighbours in
// ascending id, a newly reached cell takes the least positive color no
// neighbour already has; restart at the least uncolored id.
int color_level(HostLevel &L)
{
    Csr g = neighbours(L);
    L.color.assign(L.n, 0);
    int nc = 0;
    std::deque<int64_t> wave;
    std::vector<int32_t> stamp;   // stamp[k] == w+1 <=> color k taken around w
    for (int64_t seed = 0; seed < L.n; ++seed) {
        if (L.color[seed]) continue;
        L.color[seed] = 1;
        nc = std::max(nc, 1);
        wave.push_back(seed);
        while (!wave.empty()) {
            const int64_t v = wave.front();
            wave.pop_front();
            for (int64_t a = g.off[v]; a < g.off[v + 1]; ++a) {
                const int64_t w = g.idx[a];
                if (L.color[w]) continue;
                const int64_t deg = g.off[w + 1] - g.off[w];
                if ((int64_t)stamp.size() < deg + 2) stamp.resize(deg + 2, 0);
                std::fill(stamp.begin(), stamp.begin() + deg + 2, 0);
                for (int64_t b = g.off[w]; b < g.off[w + 1]; ++b) {
                    const int32_t c = L.color[g.idx[b]];
                    if (c > 0 && c <= deg + 1) stamp[c] = 1;
                }
                int32_t k = 1;
                while (stamp[k]) ++k;
                L.color[w] = k;
                nc = std::max<int>(nc, k);
                wave.push_back(w);
            }
        }
    }
    L.ncolor = nc;
    return nc;
}

bool validate_coloring(const HostLevel &L, const std::vector<int32_t> &col)
{
    if ((int64_t)col.size() != L.n) return false;
    for (int64_t i = 0; i < L.n; ++i)
        if (col[i] < 1) return false;
    for (int64_t f = 0; f < L.nf; ++f)
        if (L.right[f] >= 0 && col[L.left[f]] == col[L.right[f]]) return false;
    return true;
}

// ------------------------------------------------------------------ a3
// stable sort by (color, natural id) -> color-contiguous internal order
void renumber(HostLevel &L)
{
    L.blk.assign(L.ncolor + 1, 0);
    for (int64_t i = 0; i < L.n; ++i) L.blk[L.color[i]]++;        // blk[c] = count of color c (c >= 1)
    // blk as offsets: [blk[c-1], blk[c]) holds color c
    std::vector<int64_t> cnt(L.blk);
    L.blk[0] = 0;
    for (int c = 1; c <= L.ncolor; ++c) L.blk[c] = L.blk[c - 1] + cnt[c];
    L.perm.assign(L.n, 0);
    L.iperm.assign(L.n, 0);
    std::vector<int64_t> fill(L.blk.begin(), L.blk.end() - 1);
    for (int64_t i = 0; i < L.n; ++i) {               // ascending natural id = stable
        const int64_t p = fill[L.color[i] - 1]++;
        L.perm[p] = i;
        L.iperm[i] = p;
    }
}

// ------------------------------------------------------------------ a4
// Algorithm 3 with readings A18-A22.
int64_t agglomerate(const HostLevel &L, double theta, std::vector<int64_t> &parent, int64_t &nc)
{
    const int d = L.dim;
    uint64_t n_int = 0;
    for (int64_t f = 0; f < L.nf; ++f) n_int += (L.right[f] >= 0);
    std::vector<int64_t> partner(L.n, -1);
    int64_t merged = 0;
    if (n_int) {
        // first loop: faces whose hash value is new enter the collection V_d
        std::vector<uint8_t> taken(n_int, 0);
        std::vector<int64_t> cand;
        for (int64_t f = 0; f < L.nf; ++f) {
            const int64_t l = L.left[f], r = L.right[f];
            if (r < 0) continue;                                     // boundary face
            if (!L.part.empty() && L.part[l] != L.part[r]) continue; // parallel interface
            const uint64_t ul = (uint64_t)l, ur = (uint64_t)r;
            const uint64_t h = (23ull * (ul + ur) + ul * ur) % n_int; // Eq.(hash value), uint64 (A19)
            if (taken[h]) continue;
            taken[h] = 1;
            cand.push_back(f);
        }
        const Csr inc = incident_faces(L);
        // second loop: merge pairs that pass the skewness test (A21, A22)
        for (const int64_t f : cand) {
            const int64_t l = L.left[f], r = L.right[f];
            if (partner[l] >= 0 || partner[r] >= 0) continue;
            const double Vl = L.vol[l], Vr = L.vol[r];
            double Cv[3] = {0.0, 0.0, 0.0};
            for (int k = 0; k < d; ++k)
                Cv[k] = (Vl * L.ctr[(size_t)k * L.n + l] + Vr * L.ctr[(size_t)k * L.n + r]) / (Vl + Vr);
            double smin = 2.0;
            for (const int64_t c : {l, r}) {
                for (int64_t a = inc.off[c]; a < inc.off[c + 1]; ++a) {
                    const int64_t g = inc.idx[a];
                    const int64_t gl = L.left[g], gr = L.right[g];
                    if ((gl == l && gr == r) || (gl == r && gr == l)) continue;
                    const double sg = (gl == c) ? 1.0 : -1.0;
                    double A[3] = {0.0, 0.0, 0.0}, dv[3] = {0.0, 0.0, 0.0}, nv[3] = {0.0, 0.0, 0.0};
                    for (int k = 0; k < d; ++k) A[k] = L.avec[(size_t)k * L.nf + g];
                    const double S = norm_area(d, A);
                    for (int k = 0; k < d; ++k) {
                        nv[k] = (sg * A[k]) / S;
                        dv[k] = L.fctr[(size_t)k * L.nf + g] - Cv[k];
                    }
                    double dn = dv[0] * nv[0];
                    dn = dn + dv[1] * nv[1];
                    double dd = dv[0] * dv[0];
                    dd = dd + dv[1] * dv[1];
                    if (d == 3) { dn = dn + dv[2] * nv[2]; dd = dd + dv[2] * dv[2]; }
                    const double s = (dd == 0.0) ? 1.0 : dn / std::sqrt(dd);
                    if (s < smin) smin = s;
                }
            }
            if (smin >= theta) {                      // merge iff min_g s_g >= theta
                partner[l] = r;
                partner[r] = l;
                ++merged;
            }
        }
    }
    parent.assign(L.n, -1);
    nc = 0;
    for (int64_t i = 0; i < L.n; ++i)
        parent[i] = (partner[i] >= 0 && partner[i] < i) ? parent[partner[i]] : nc++;
    return merged;
}

// O1: coarse cells (V_c = V_a + V_b, C_c = (V_a C_a + V_b C_b)/V_c, children
// ascending) and coarse faces (one per coarse pair a < b aggregated in
// ascending fine-face order, then boundary faces in fine-face order).
void build_coarse(const HostLevel &fine, HostLevel &C)
{
    const int d = fine.dim;
    const int64_t nc = fine.n_coarse;
    C.dim = d;
    C.n = nc;
    C.vol.assign(nc, 0.0);
    C.ctr.assign((size_t)d * nc, 0.0);
    std::vector<double> wsum((size_t)d * nc, 0.0);
    std::vector<uint8_t> seen(nc, 0);
    for (int64_t i = 0; i < fine.n; ++i) {
        const int64_t c = fine.parent[i];
        if (!seen[c]) {
            seen[c] = 1;
            C.vol[c] = fine.vol[i];
            for (int k = 0; k < d; ++k) wsum[(size_t)k * nc + c] = fine.vol[i] * fine.ctr[(size_t)k * fine.n + i];
        } else {
            C.vol[c] = C.vol[c] + fine.vol[i];
            for (int k = 0; k < d; ++k)
                wsum[(size_t)k * nc + c] = wsum[(size_t)k * nc + c] + fine.vol[i] * fine.ctr[(size_t)k * fine.n + i];
        }
    }
    for (int k = 0; k < d; ++k)
        for (int64_t c = 0; c < nc; ++c) C.ctr[(size_t)k * nc + c] = wsum[(size_t)k * nc + c] / C.vol[c];
    if (!fine.part.empty()) {
        C.part.assign(nc, 0);
        for (int64_t i = 0; i < fine.n; ++i) C.part[fine.parent[i]] = fine.part[i];
    }

    std::vector<std::tuple<int64_t, int64_t, int64_t>> pairs;
    int64_t nb = 0;
    for (int64_t f = 0; f < fine.nf; ++f) {
        if (fine.right[f] < 0) { ++nb; continue; }
        const int64_t a = fine.parent[fine.left[f]], b = fine.parent[fine.right[f]];
        if (a == b) continue;
        pairs.emplace_back(std::min(a, b), std::max(a, b), f);
    }
    std::sort(pairs.begin(), pairs.end());
    int64_t ni = 0;
    for (size_t k = 0; k < pairs.size(); ++k)
        if (k == 0 || std::get<0>(pairs[k]) != std::get<0>(pairs[k - 1]) || std::get<1>(pairs[k]) != std::get<1>(pairs[k - 1])) ++ni;
    const int64_t nfc = ni + nb;
    C.nf = nfc;
    C.left.assign(nfc, 0);
    C.right.assign(nfc, 0);
    C.avec.assign((size_t)d * nfc, 0.0);
    C.fctr.assign((size_t)d * nfc, 0.0);
    C.ngauss.assign(nfc, 0);
    int64_t fo = -1;
    double wa = 0.0, wx[3] = {0, 0, 0};
    auto close_face = [&]() {
        if (fo >= 0) for (int k = 0; k < d; ++k) C.fctr[(size_t)k * nfc + fo] = wx[k] / wa;
    };
    for (size_t k = 0; k < pairs.size(); ++k) {
        const int64_t a = std::get<0>(pairs[k]), b = std::get<1>(pairs[k]), f = std::get<2>(pairs[k]);
        if (k == 0 || a != std::get<0>(pairs[k - 1]) || b != std::get<1>(pairs[k - 1])) {
            close_face();
            ++fo;
            C.left[fo] = a;
            C.right[fo] = b;
            wa = 0.0;
            wx[0] = wx[1] = wx[2] = 0.0;
        }
        const double sg = (fine.parent[fine.left[f]] == a) ? 1.0 : -1.0;
        double A[3] = {0.0, 0.0, 0.0};
        for (int q = 0; q < d; ++q) A[q] = fine.avec[(size_t)q * fine.nf + f];
        const double S = norm_area(d, A);
        for (int q = 0; q < d; ++q) {
            C.avec[(size_t)q * nfc + fo] = C.avec[(size_t)q * nfc + fo] + sg * A[q];
            wx[q] = wx[q] + S * fine.fctr[(size_t)q * fine.nf + f];
        }
        wa = wa + S;
        C.ngauss[fo] = std::max(C.ngauss[fo], fine.ngauss[f]);
    }
    close_face();
    for (int64_t f = 0; f < fine.nf; ++f) {
        if (fine.right[f] >= 0) continue;
        ++fo;
        C.left[fo] = fine.parent[fine.left[f]];
        C.right[fo] = fine.right[f];
        C.ngauss[fo] = fine.ngauss[f];
        for (int q = 0; q < d; ++q) {
            C.avec[(size_t)q * nfc + fo] = fine.avec[(size_t)q * fine.nf + f];
            C.fctr[(size_t)q * nfc + fo] = fine.fctr[(size_t)q * fine.nf + f];
        }
    }
}

// Layouts (internal order).
//  * gather slots (residual/prepare, thread per cell): SELL-32 -- per color,
//    chunks of 32 consecutive cells, entries [slot][lane], chunk padded to its
//    max degree.  Slots: interior faces (ascending id) then boundary faces.
//  * sweep slots (lanes per cell): CSR -- cell i's interior slots are
//    contiguous at [soffc[i], soffc[i+1]), same order as its gather slots;
//    per slot the neighbour sJ and a 32-byte record (A_x, A_y, [A_z,] S r)
//    with A = sigma S n oriented outward from the cell.
void build_layout(HostLevel &L)
{
    const int d = L.dim;
    const Csr inc = incident_faces(L);
    L.chunk_base.assign(L.ncolor + 1, 0);
    for (int c = 0; c < L.ncolor; ++c) {
        const int64_t cnt = L.blk[c + 1] - L.blk[c];
        L.chunk_base[c + 1] = L.chunk_base[c] + (int32_t)((cnt + kChunk - 1) / kChunk);
    }
    L.nchunks = L.chunk_base[L.ncolor];
    L.gbase.assign(L.n, 0);
    L.deg_int.assign(L.n, 0);
    L.deg_all.assign(L.n, 0);
    std::vector<int32_t> cchunk(L.n, 0);
    std::vector<std::vector<int64_t>> slots(L.n);
    for (int c = 0; c < L.ncolor; ++c) {
        for (int64_t i = L.blk[c]; i < L.blk[c + 1]; ++i) {
            const int64_t t = i - L.blk[c];
            cchunk[i] = L.chunk_base[c] + (int32_t)(t / kChunk);
            const int64_t nat = L.perm[i];
            auto &s = slots[i];
            for (int64_t a = inc.off[nat]; a < inc.off[nat + 1]; ++a)
                if (L.right[inc.idx[a]] >= 0) s.push_back(inc.idx[a]);
            const size_t ni = s.size();
            for (int64_t a = inc.off[nat]; a < inc.off[nat + 1]; ++a)
                if (L.right[inc.idx[a]] < 0) s.push_back(inc.idx[a]);
            if (s.size() > 255) throw std::runtime_error("cell with more than 255 faces");
            L.deg_int[i] = (uint8_t)ni;
            L.deg_all[i] = (uint8_t)s.size();
        }
    }
    L.goff.assign(L.nchunks, 0);
    int64_t go = 0;
    for (int c = 0; c < L.ncolor; ++c) {
        for (int32_t k = L.chunk_base[c]; k < L.chunk_base[c + 1]; ++k) {
            const int64_t i0 = L.blk[c] + (int64_t)(k - L.chunk_base[c]) * kChunk;
            const int64_t i1 = std::min<int64_t>(i0 + kChunk, L.blk[c + 1]);
            int mg = 0;
            for (int64_t i = i0; i < i1; ++i) mg = std::max<int>(mg, L.deg_all[i]);
            L.goff[k] = (int32_t)go;
            go += (int64_t)mg * kChunk;
        }
    }
    L.soffc.assign(L.n + 1, 0);
    for (int64_t i = 0; i < L.n; ++i) L.soffc[i + 1] = L.soffc[i] + L.deg_int[i];
    const int64_t so = L.soffc[L.n];
    if (go >= INT32_MAX || so >= INT32_MAX / 4) throw std::runtime_error("slot table exceeds int32");
    L.ng_entries = go;
    L.ns_entries = so;
    L.gface.assign(go, 0);
    L.sJ.assign(so, -1);
    L.sface.assign(so, -1);
    L.sRec.assign((size_t)4 * so, 0.0);
    for (int c = 0; c < L.ncolor; ++c)
    for (int64_t i = L.blk[c]; i < L.blk[c + 1]; ++i) {
        const int32_t k = cchunk[i];
        const int64_t lane = (i - L.blk[c]) % kChunk;
        L.gbase[i] = (int32_t)(L.goff[k] + lane);
        const int64_t nat = L.perm[i];
        for (size_t s = 0; s < slots[i].size(); ++s) {
            const int64_t f = slots[i][s];
            const bool is_left = (L.left[f] == nat);
            L.gface[L.goff[k] + s * kChunk + lane] = is_left ? (int32_t)(f + 1) : -(int32_t)(f + 1);
            if (s < L.deg_int[i]) {
                const int64_t e = L.soffc[i] + (int64_t)s;
                const int64_t other = is_left ? L.right[f] : L.left[f];
                L.sJ[e] = (int32_t)L.iperm[other];
                L.sface[e] = (int32_t)f;
                const double sg = is_left ? 1.0 : -1.0;
                for (int q = 0; q < d; ++q) L.sRec[(size_t)4 * e + q] = sg * L.avec[(size_t)q * L.nf + f];
            }
        }
    }
}

}  // namespace gmg
