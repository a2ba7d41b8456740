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
    std::vector<int64_t> cnt(L.ncolor + 1, 0), pos(L.ncolor + 1, 0);
    for (int64_t i = 0; i < L.n; ++i) cnt[L.color[i]]++;
    int64_t acc = 0;
    for (int c = 1; c <= L.ncolor; ++c) { pos[c] = acc; acc += cnt[c]; }
    L.perm.assign(L.n, 0);
    for (int64_t i = 0; i < L.n; ++i) L.perm[pos[L.color[i]]++] = i;   // ascending natural id = stable
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
    {   // (a, b, f) order: counting sort by a (stable, f ascending), then each small bucket by (b, f)
        std::vector<int64_t> cnt(nc + 1, 0);
        for (const auto &t : pairs) cnt[std::get<0>(t) + 1]++;
        std::partial_sum(cnt.begin(), cnt.end(), cnt.begin());
        std::vector<std::tuple<int64_t, int64_t, int64_t>> out(pairs.size());
        std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
        for (const auto &t : pairs) out[pos[std::get<0>(t)]++] = t;
        for (int64_t a = 0; a < nc; ++a)
            if (cnt[a + 1] - cnt[a] > 1) std::sort(out.begin() + cnt[a], out.begin() + cnt[a + 1]);
        pairs.swap(out);
    }
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

// ------------------------------------------------------------------ a5
// Recursive coordinate bisection of the cell centroids: split the longest
// extent so that each side gets cells in proportion to its partition count,
// order (coordinate, natural id) -- deterministic on every rank.
void partition_rcb(int64_t n, int dim, const double *ctr, int nparts, int32_t *part)
{
    std::vector<int64_t> ids(n);
    std::iota(ids.begin(), ids.end(), (int64_t)0);
    struct Job { int64_t b, e; int p0, np; };
    std::vector<Job> st{{0, n, 0, nparts}};
    while (!st.empty()) {
        const Job j = st.back();
        st.pop_back();
        if (j.np <= 1 || j.e - j.b <= 1) {
            for (int64_t k = j.b; k < j.e; ++k) part[ids[k]] = j.p0;
            continue;
        }
        int axis = 0;
        double best = -1.0;
        for (int k = 0; k < dim; ++k) {
            double lo = 1e300, hi = -1e300;
            for (int64_t t = j.b; t < j.e; ++t) {
                const double x = ctr[(size_t)k * n + ids[t]];
                lo = std::min(lo, x);
                hi = std::max(hi, x);
            }
            if (hi - lo > best) { best = hi - lo; axis = k; }
        }
        const int nl = j.np / 2, nr = j.np - nl;
        const int64_t m = j.b + (j.e - j.b) * nl / j.np;
        auto less = [&](int64_t a, int64_t b) {
            const double xa = ctr[(size_t)axis * n + a], xb = ctr[(size_t)axis * n + b];
            return xa < xb || (xa == xb && a < b);
        };
        std::nth_element(ids.begin() + j.b, ids.begin() + m, ids.begin() + j.e, less);
        st.push_back({m, j.e, j.p0 + nl, nr});
        st.push_back({j.b, m, j.p0, nl});
    }
}

// Domain of `rank` on a global level: owned cells in color
// blocks (boundary cells -- a face neighbour on another rank -- first), inside
// a block by the Morton key of the centroid when `morton` (natural id
// otherwise), then one layer of ghosts in (owner, color, natural id) order;
// local faces = faces touching an owned cell, ordered by their first local
// cell; layouts over owned cells:
//  * gather slots (residual/prepare, thread per cell, cells in the gather
//    order gord -- Morton across colors): SELL-32 -- chunks of 32 consecutive
//    cells of that order, entries [slot][lane], chunk padded to its max
//    degree.  Slots: interior faces (by neighbour local index: lower colors first) then boundary faces.
//  * sweep slots (lanes per cell): CSR -- cell i's interior slots are
//    contiguous at [soffc[i], soffc[i+1]), same order as its gather slots;
//    per slot the neighbour sJe and a 32-byte record (A_x, A_y, [A_z,] S r)
//    with A = sigma S n oriented outward from the cell.
//  * halo plan grouped (color, peer), natural id ascending within a group, so
//    a sender's group equals the receiver's group element by element.
void build_domain_level(const HostLevel &G, int rank, DomLevel &D, bool morton)
{
    const int d = G.dim;
    const int64_t N = G.n;
    D = DomLevel();
    auto owned = [&](int64_t c) { return G.part_of(c) == rank; };
    std::vector<int32_t> n2l(N, -1);
    D.blk.assign(G.ncolor + 1, 0);
    // owned cells with a face neighbour on another rank ("boundary" cells) go
    // first inside their color block, so their increments can be sent while
    // the interior cells of the same color are swept (exchange overlap)
    std::vector<uint8_t> bnd(N, 0);
    for (int64_t f = 0; f < G.nf; ++f) {
        const int64_t l = G.left[f], r = G.right[f];
        if (r < 0) continue;
        if (owned(l) && !owned(r)) bnd[l] = 1;
        if (owned(r) && !owned(l)) bnd[r] = 1;
    }
    for (int64_t p = 0; p < N; ++p) {
        const int64_t nat = G.perm[p];
        if (!owned(nat)) continue;
        D.l2n.push_back(nat);
        D.blk[G.color[nat]]++;
    }
    D.n_own = (int64_t)D.l2n.size();
    for (int c = 1; c <= G.ncolor; ++c) D.blk[c] += D.blk[c - 1];
    D.nbnd.assign(G.ncolor, 0);
    for (int c = 0; c < G.ncolor; ++c) {
        auto b0 = D.l2n.begin() + D.blk[c], b1 = D.l2n.begin() + D.blk[c + 1];
        auto mid = std::stable_partition(b0, b1, [&](int64_t nat) { return bnd[nat] != 0; });
        D.nbnd[c] = (int64_t)(mid - b0);
    }
    // single domain: inside each color block the cells are ordered by the
    // Morton (Z-order) key of their centroid -- neighbours of consecutive cells
    // are then close in memory (L2 reuse of the gathered records, DESIGN.md §6 v13)
    std::vector<uint64_t> key;
    if (morton) {
        // Morton (Z-order) key of the centroid: the same spatial grouping as
        // fine RCB chunks at a fraction of the setup cost
        double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
        for (int k = 0; k < d; ++k)
            for (int64_t i = 0; i < N; ++i) {
                lo[k] = std::min(lo[k], G.ctr[(size_t)k * N + i]);
                hi[k] = std::max(hi[k], G.ctr[(size_t)k * N + i]);
            }
        const int bits = d == 3 ? 21 : 31;
        const double scale = (double)((1u << bits) - 1);
        auto spread = [&](uint64_t v) {
            uint64_t r = 0;
            for (int b = 0; b < bits; ++b) r |= ((v >> b) & 1ull) << (b * d);
            return r;
        };
        key.assign(N, 0);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < N; ++i) {
            uint64_t code = 0;
            for (int k = 0; k < d; ++k) {
                const double ext = hi[k] > lo[k] ? hi[k] - lo[k] : 1.0;
                const uint64_t q = (uint64_t)((G.ctr[(size_t)k * N + i] - lo[k]) / ext * scale);
                code |= spread(q) << k;
            }
            key[i] = code;
        }
        // boundary cells stay first inside their block (exchange overlap): sort each part
        auto cmp = [&](int64_t a, int64_t b) { return key[a] < key[b] || (key[a] == key[b] && a < b); };
        for (int c = 0; c < G.ncolor; ++c) {
            std::sort(D.l2n.begin() + D.blk[c], D.l2n.begin() + D.blk[c] + D.nbnd[c], cmp);
            std::sort(D.l2n.begin() + D.blk[c] + D.nbnd[c], D.l2n.begin() + D.blk[c + 1], cmp);
        }
    }
    for (int64_t i = 0; i < D.n_own; ++i) n2l[D.l2n[i]] = (int32_t)i;
    // gather order (the residual / prepare kernels have no color dependency): the
    // owned cells by Morton key across all colors, so the two cells of a face --
    // which read its face record -- are visited close in time (the second read
    // hits L2); without Morton keys the internal order
    D.gord.resize(D.n_own);
    for (int64_t i = 0; i < D.n_own; ++i) D.gord[i] = (int32_t)i;
    if (!key.empty())
        std::sort(D.gord.begin(), D.gord.end(), [&](int32_t a, int32_t b) {
            const uint64_t ka = key[D.l2n[a]], kb = key[D.l2n[b]];
            return ka < kb || (ka == kb && D.l2n[a] < D.l2n[b]);
        });
    std::vector<int64_t> ghosts;
    for (int64_t f = 0; f < G.nf; ++f) {
        const int64_t l = G.left[f], r = G.right[f];
        const bool ol = owned(l), orr = r >= 0 && owned(r);
        if (!ol && !orr) continue;
        D.fnat.push_back(f);
        if (r >= 0 && !ol) ghosts.push_back(l);
        if (r >= 0 && !orr) ghosts.push_back(r);
    }
    std::sort(ghosts.begin(), ghosts.end(), [&](int64_t a, int64_t b) {
        const int pa = G.part_of(a), pb = G.part_of(b);
        if (pa != pb) return pa < pb;
        if (G.color[a] != G.color[b]) return G.color[a] < G.color[b];
        return a < b;
    });
    ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
    for (const int64_t g : ghosts) {
        n2l[g] = (int32_t)D.l2n.size();
        D.l2n.push_back(g);
    }
    D.n_loc = (int64_t)D.l2n.size();
    // local face order: by the first local cell of the face, then natural id --
    // the face kernel's state gathers and the gather kernel's face reads then
    // walk memory roughly in cell order
    {
        // counting sort by key (stable: fnat is in ascending natural order), the
        // same order as sorting (key, natural id) pairs
        auto key = [&](int64_t f) {
            int32_t k = n2l[G.left[f]];
            if (G.right[f] >= 0) k = std::min(k, n2l[G.right[f]]);
            return k;
        };
        std::vector<int64_t> cnt(D.n_loc + 1, 0), out(D.fnat.size());
        std::vector<int32_t> kk(D.fnat.size());
        for (size_t t = 0; t < D.fnat.size(); ++t) { kk[t] = key(D.fnat[t]); cnt[kk[t] + 1]++; }
        std::partial_sum(cnt.begin(), cnt.end(), cnt.begin());
        for (size_t t = 0; t < D.fnat.size(); ++t) out[cnt[kk[t]]++] = D.fnat[t];
        D.fnat.swap(out);
    }
    D.nf = (int64_t)D.fnat.size();
    D.fl.resize(D.nf);
    D.fr.resize(D.nf);
    for (int64_t k = 0; k < D.nf; ++k) {
        const int64_t f = D.fnat[k];
        D.fl[k] = n2l[G.left[f]];
        D.fr[k] = G.right[f] >= 0 ? n2l[G.right[f]] : (int32_t)G.right[f];
    }
    D.vol.resize(D.n_own);
    for (int64_t i = 0; i < D.n_own; ++i) D.vol[i] = G.vol[D.l2n[i]];

    // incident local faces of owned cells, ascending local face id
    std::vector<int64_t> ioff(D.n_own + 1, 0), iidx;
    for (int64_t k = 0; k < D.nf; ++k) {
        if (D.fl[k] < D.n_own) ioff[D.fl[k] + 1]++;
        if (D.fr[k] >= 0 && D.fr[k] < D.n_own) ioff[D.fr[k] + 1]++;
    }
    std::partial_sum(ioff.begin(), ioff.end(), ioff.begin());
    iidx.resize(ioff[D.n_own]);
    {
        std::vector<int64_t> pos(ioff.begin(), ioff.end() - 1);
        for (int64_t k = 0; k < D.nf; ++k) {
            if (D.fl[k] < D.n_own) iidx[pos[D.fl[k]]++] = k;
            if (D.fr[k] >= 0 && D.fr[k] < D.n_own) iidx[pos[D.fr[k]]++] = k;
        }
    }
    // slots of cell i = its incident faces, interior ones first (by neighbour), in place in iidx
    D.deg_int.assign(D.n_own, 0);
    D.deg_all.assign(D.n_own, 0);
    for (int64_t i = 0; i < D.n_own; ++i)
        if (ioff[i + 1] - ioff[i] > 255) throw std::runtime_error("cell with more than 255 faces");
#pragma omp parallel
    {
        std::vector<int64_t> tmp;
#pragma omp for schedule(static)
        for (int64_t i = 0; i < D.n_own; ++i) {
            const int64_t a0 = ioff[i], a1 = ioff[i + 1];
            tmp.clear();
            for (int64_t a = a0; a < a1; ++a)
                if (D.fr[iidx[a]] >= 0) tmp.push_back(iidx[a]);
            const size_t ni = tmp.size();
            // interior slots by neighbour (local index: color-major, so lower-color neighbours first --
            // which keeps the two lanes of a cell on the same side of the first-forward
            // "earlier color" branch more often, and a cell's neighbour loads in address order)
            std::stable_sort(tmp.begin(), tmp.end(), [&](int64_t x, int64_t y) {
                const int32_t jx = D.fl[x] == i ? D.fr[x] : D.fl[x], jy = D.fl[y] == i ? D.fr[y] : D.fl[y];
                return jx < jy;
            });
            for (int64_t a = a0; a < a1; ++a)
                if (D.fr[iidx[a]] < 0) tmp.push_back(iidx[a]);
            std::copy(tmp.begin(), tmp.end(), iidx.begin() + a0);
            D.deg_int[i] = (uint8_t)ni;
            D.deg_all[i] = (uint8_t)(a1 - a0);
        }
    }
    // SELL-32 gather chunks: 32 consecutive cells of the gather order
    std::vector<int32_t> cchunk(D.n_own, 0), lane(D.n_own, 0);
    int64_t go = 0;
    for (int64_t t0 = 0; t0 < D.n_own; t0 += kChunk) {
        const int64_t t1 = std::min<int64_t>(t0 + kChunk, D.n_own);
        int mg = 0;
        for (int64_t t = t0; t < t1; ++t) {
            const int32_t i = D.gord[t];
            mg = std::max<int>(mg, D.deg_all[i]);
            cchunk[i] = (int32_t)D.goff.size();
            lane[i] = (int32_t)(t - t0);
        }
        D.goff.push_back((int32_t)go);
        go += (int64_t)mg * kChunk;
    }
    D.nchunks = (int64_t)D.goff.size();
    D.soffc.assign(D.n_own + 1, 0);
    for (int64_t i = 0; i < D.n_own; ++i) D.soffc[i + 1] = D.soffc[i] + D.deg_int[i];
    const int64_t so = D.soffc[D.n_own];
    if (go >= INT32_MAX || so >= INT32_MAX / 4) throw std::runtime_error("slot table exceeds int32");
    D.ng_entries = go;
    D.ns_entries = so;
    D.gface.assign(go, 0);
    D.gbase.assign(D.n_own, 0);
    D.sJe.assign(so, -1);
    D.sRe.assign((size_t)4 * so, 0.0);
    D.fslot.assign((size_t)2 * D.nf, -1);
    // every cell writes only its own gather / sweep slots and its (face, side) fslot entries
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < D.n_own; ++i) {
        D.gbase[i] = D.goff[cchunk[i]] + lane[i];
        for (int64_t s = 0; s < ioff[i + 1] - ioff[i]; ++s) {
            const int64_t k = iidx[ioff[i] + s];
            const bool is_left = (D.fl[k] == i);
            D.gface[D.gbase[i] + s * kChunk] = is_left ? (int32_t)(k + 1) : -(int32_t)(k + 1);
            if (s < D.deg_int[i]) {
                const int64_t e = D.soffc[i] + (int64_t)s;
                D.sJe[e] = is_left ? D.fr[k] : D.fl[k];
                D.fslot[(size_t)2 * k + (is_left ? 0 : 1)] = (int32_t)e;
                const double sg = is_left ? 1.0 : -1.0;
                const int64_t f = D.fnat[k];
                for (int q = 0; q < d; ++q) D.sRe[(size_t)4 * e + q] = sg * G.avec[(size_t)q * G.nf + f];
            }
        }
    }
    // halo plan
    for (int64_t g = D.n_own; g < D.n_loc; ++g) D.peers.push_back(G.part_of(D.l2n[g]));
    std::sort(D.peers.begin(), D.peers.end());
    D.peers.erase(std::unique(D.peers.begin(), D.peers.end()), D.peers.end());
    const int np = (int)D.peers.size();
    auto peer_index = [&](int p) { return (int)(std::lower_bound(D.peers.begin(), D.peers.end(), p) - D.peers.begin()); };
    const int ng = G.ncolor * np;
    std::vector<std::vector<int32_t>> sg(ng), rg(ng);
    for (int64_t g = D.n_own; g < D.n_loc; ++g) {                 // ghosts: (owner, color, id) order
        const int64_t nat = D.l2n[g];
        rg[(G.color[nat] - 1) * np + peer_index(G.part_of(nat))].push_back((int32_t)g);
    }
    std::vector<int> ps;
    for (int64_t i = 0; i < D.n_own; ++i) {                       // owned: (color, boundary first, id) order
        if (!bnd[D.l2n[i]]) continue;                             // no ghost neighbour
        ps.clear();
        for (int32_t e = D.soffc[i]; e < D.soffc[i + 1]; ++e) {
            const int32_t j = D.sJe[e];
            if (j >= D.n_own) ps.push_back(G.part_of(D.l2n[j]));
        }
        std::sort(ps.begin(), ps.end());
        ps.erase(std::unique(ps.begin(), ps.end()), ps.end());
        for (const int p : ps) sg[(G.color[D.l2n[i]] - 1) * np + peer_index(p)].push_back((int32_t)i);
    }
    for (auto &g : sg)   // natural id ascending: element-wise equal to the receiver's ghost group
        std::sort(g.begin(), g.end(), [&](int32_t a, int32_t b) { return D.l2n[a] < D.l2n[b]; });
    D.send_off.assign(ng + 1, 0);
    D.recv_off.assign(ng + 1, 0);
    for (int k = 0; k < ng; ++k) {
        D.send_off[k + 1] = D.send_off[k] + (int64_t)sg[k].size();
        D.recv_off[k + 1] = D.recv_off[k] + (int64_t)rg[k].size();
        D.send_idx.insert(D.send_idx.end(), sg[k].begin(), sg[k].end());
        D.recv_idx.insert(D.recv_idx.end(), rg[k].begin(), rg[k].end());
    }
}

// fused P2P halo: for every send entry (color c, peer k, position t) the
// receiving rank's ghost at the same position of ITS group (c, my rank) --
// the groups are element-wise identical (natural id ascending) by construction
void build_p2p_targets(DomLevel &D, int me, int ncolor, const std::vector<const DomLevel *> &peer_dom)
{
    const int np = (int)D.peers.size();
    std::vector<std::vector<std::pair<int32_t, int32_t>>> tg(D.n_own);
    for (int k = 0; k < np; ++k) {
        const DomLevel &Q = *peer_dom[k];
        const int npq = (int)Q.peers.size();
        const int kq = (int)(std::lower_bound(Q.peers.begin(), Q.peers.end(), me) - Q.peers.begin());
        if (kq >= npq || Q.peers[kq] != me) throw std::runtime_error("p2p: asymmetric halo plan");
        for (int c = 0; c < ncolor; ++c) {
            const int64_t s0 = D.send_off[(size_t)c * np + k], s1 = D.send_off[(size_t)c * np + k + 1];
            const int64_t r0 = Q.recv_off[(size_t)c * npq + kq], r1 = Q.recv_off[(size_t)c * npq + kq + 1];
            if (s1 - s0 != r1 - r0) throw std::runtime_error("p2p: halo group size mismatch");
            for (int64_t t = 0; t < s1 - s0; ++t)
                tg[D.send_idx[s0 + t]].push_back({(int32_t)k, Q.recv_idx[r0 + t]});
        }
    }
    D.p2p_peer_nloc.assign(np, 0);
    for (int k = 0; k < np; ++k) D.p2p_peer_nloc[k] = (int32_t)peer_dom[k]->n_loc;
    D.p2p_off.assign(D.n_own + 1, 0);
    D.p2p_k.clear();
    D.p2p_g.clear();
    for (int64_t i = 0; i < D.n_own; ++i) {
        for (const auto &e : tg[i]) { D.p2p_k.push_back(e.first); D.p2p_g.push_back(e.second); }
        D.p2p_off[i + 1] = (int32_t)D.p2p_k.size();
    }
}

// fine <-> coarse links inside one domain (agglomeration never crosses a
// partition face, so both ends are owned by the same rank)
void link_domain_levels(const HostLevel &Gf, const HostLevel &Gc, DomLevel &Df, DomLevel &Dc)
{
    std::vector<int32_t> c2l(Gc.n, -1);
    for (int64_t i = 0; i < Dc.n_own; ++i) c2l[Dc.l2n[i]] = (int32_t)i;
    Df.parent.assign(Df.n_own, -1);
    std::vector<int32_t> f2l(Gf.n, -1);                 // natural -> local (owned) fine index
    for (int64_t i = 0; i < Df.n_own; ++i) {
        const int32_t pc = c2l[Gf.parent[Df.l2n[i]]];
        if (pc < 0) throw std::runtime_error("coarse parent not owned by the fine cell's rank");
        Df.parent[i] = pc;
        f2l[Df.l2n[i]] = (int32_t)i;
    }
    Dc.child.assign(2 * Dc.n_own, -1);
    for (int64_t nat = 0; nat < Gf.n; ++nat) {          // ascending natural id of the fine cell
        const int32_t i = f2l[nat];
        if (i < 0) continue;
        const int32_t c = Df.parent[i];
        if (Dc.child[c] < 0) Dc.child[c] = i;
        else Dc.child[Dc.n_own + c] = i;
    }
}

}  // namespace gmg
