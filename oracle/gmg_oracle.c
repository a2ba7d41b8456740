/*
 * gmg_oracle.c -- plain, slow, obviously-correct CPU oracle for the hot path
 * of arXiv 2509.06347 (GMG + MC-LU-SGS).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_2509_06347_b200/csrc); the two never include or link each other.
 *
 * Conventions: natural cell/face order, fp64, SoA [component][item] arrays,
 * no blocking, no fusion, no reordering beyond what the cited passage states.
 * Built with -O2 -ffp-contract=off (no FMA contraction), so that the
 * floating-point decisions of the agglomeration (skewness test) are exactly
 * the expressions written below.
 *
 * Timing build (bench.py cpu_baseline / --impl reference only): the same
 * source with -O3 -march=native -fopenmp -ffp-contract=off.  The OpenMP
 * pragmas below parallelise only loops whose iterations are independent
 * (cells of ONE color in the sweep, per-face flux evaluations, per-cell
 * updates); every sum keeps its sequential order, so the timing build
 * returns the same bits as the parity build (tests/test_oracle_timing.py).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n; "S:n" = SPEC.md line
 * n; "O#" / "A#" = the SURVEY.md §8(c) oracle step / reading adopted (also
 * listed in DESIGN.md "Readings").
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"): see the header comment of each
 * function; functions without a pin say "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* --------------------------------------------------------------------- */
/* mesh level (natural order), passed from Python via ctypes              */
/* --------------------------------------------------------------------- */
typedef struct {
    int dim;                 /* 2 or 3 */
    int n_patches;
    int64_t n;               /* cells */
    int64_t nf;              /* faces (interior + boundary) */
    const double *vol;       /* [n] */
    const double *ctr;       /* [dim][n] */
    const int64_t *left;     /* [nf] */
    const int64_t *right;    /* [nf]  <0 : -(patch+1) */
    const double *avec;      /* [dim][nf] area vector S_f n_f, left -> right */
    const double *fctr;      /* [dim][nf] */
    const int8_t *ngauss;    /* [nf] M_f */
    const int32_t *patch_kind; /* [n_patches] */
} orc_level;

enum { ORC_FARFIELD = 0, ORC_SLIP = 1, ORC_NOSLIP = 2, ORC_EXTRAP = 3 };

/* cell -> faces CSR, ascending face id (built on the fly; tiny helper) */
static void cell_faces(const orc_level *L, int64_t **off_out, int64_t **idx_out)
{
    int64_t *off = calloc((size_t)L->n + 1, sizeof(int64_t));
    for (int64_t f = 0; f < L->nf; ++f) {
        off[L->left[f] + 1]++;
        if (L->right[f] >= 0) off[L->right[f] + 1]++;
    }
    for (int64_t i = 0; i < L->n; ++i) off[i + 1] += off[i];
    int64_t *fill = malloc(sizeof(int64_t) * (size_t)(L->n + 1));
    memcpy(fill, off, sizeof(int64_t) * (size_t)(L->n + 1));
    int64_t *idx = malloc(sizeof(int64_t) * (size_t)(off[L->n] + 1));
    for (int64_t f = 0; f < L->nf; ++f) {     /* ascending f => sorted lists */
        idx[fill[L->left[f]]++] = f;
        if (L->right[f] >= 0) idx[fill[L->right[f]]++] = f;
    }
    free(fill);
    *off_out = off;
    *idx_out = idx;
}

/* ===================================================================== */
/* O2. Coloring: Algorithm 1, start cell 0,       */
/*     FIFO BFS, neighbours in ascending natural id, restart at the       */
/*     smallest uncolored id (reading A24).                               */
/* Pins: validity + greedy bound, exact 2-color checkerboard  */
/* on quad grids and uniform-diagonal triangulations, brute-  */
/* force replay in pure Python (tests/brute.py).                          */
/* ===================================================================== */
int orc_color(int64_t n, int64_t nf, const int64_t *left, const int64_t *right, int32_t *color)
{
    /* adjacency: neighbours of each cell sorted by natural id */
    int64_t *off = calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t f = 0; f < nf; ++f)
        if (right[f] >= 0) { off[left[f] + 1]++; off[right[f] + 1]++; }
    for (int64_t i = 0; i < n; ++i) off[i + 1] += off[i];
    int64_t *fill = malloc(sizeof(int64_t) * (size_t)(n + 1));
    memcpy(fill, off, sizeof(int64_t) * (size_t)(n + 1));
    int64_t *adj = malloc(sizeof(int64_t) * (size_t)(off[n] + 1));
    for (int64_t f = 0; f < nf; ++f)
        if (right[f] >= 0) { adj[fill[left[f]]++] = right[f]; adj[fill[right[f]]++] = left[f]; }
    for (int64_t i = 0; i < n; ++i) {           /* insertion sort each list */
        for (int64_t a = off[i] + 1; a < off[i + 1]; ++a) {
            int64_t v = adj[a], b = a - 1;
            while (b >= off[i] && adj[b] > v) { adj[b + 1] = adj[b]; --b; }
            adj[b + 1] = v;
        }
    }
    free(fill);

    for (int64_t i = 0; i < n; ++i) color[i] = 0;          /* colorArray(:) = 0 */
    int64_t *queue = malloc(sizeof(int64_t) * (size_t)(n + 1));
    int64_t head = 0, tail = 0, next_start = 0;
    int ncolor = 0;
    char *used = NULL;
    size_t used_cap = 0;
    while (1) {
        while (next_start < n && color[next_start] != 0) next_start++;
        if (next_start >= n) break;                          /* all cells painted */
        color[next_start] = 1;                               /* color(v0) = 1 */
        if (ncolor < 1) ncolor = 1;
        queue[tail++] = next_start;
        while (head < tail) {
            int64_t v = queue[head++];
            for (int64_t a = off[v]; a < off[v + 1]; ++a) {
                int64_t w = adj[a];
                if (color[w] != 0) continue;
                /* color(w) = min{k > 0 | k != color(j), j in C_w} */
                size_t deg = (size_t)(off[w + 1] - off[w]);
                if (deg + 2 > used_cap) { used_cap = deg + 2; used = realloc(used, used_cap); }
                memset(used, 0, deg + 2);
                for (int64_t b = off[w]; b < off[w + 1]; ++b) {
                    int32_t cj = color[adj[b]];
                    if (cj > 0 && (size_t)cj <= deg + 1) used[cj] = 1;
                }
                int32_t k = 1;
                while (used[k]) k++;
                color[w] = k;
                if (k > ncolor) ncolor = k;
                queue[tail++] = w;
            }
        }
    }
    free(used); free(queue); free(adj); free(off);
    return ncolor;
}

/* ===================================================================== */
/* O3 step 2. Face hash, Eq.(hash value) P:581-583, in uint64 (A18, A19). */
/* Pins: S:156-158 values 26, 0, 1 (P:584's printed 5 is 626 mod 23).     */
/* ===================================================================== */
uint64_t orc_face_hash(uint64_t l, uint64_t r, uint64_t nf_interior)
{
    return (23u * (l + r) + l * r) % nf_interior;
}

/* skewness of one face g seen from the virtual merged cell, O3 step 5
 * (reading A21 of Eq.(skewness factor) P:593-598): sin(alpha) = d.n/|d|,
 * d = x_g - C_v, n = outward unit normal.  Exact expression order fixed. */
static double skew_one(int dim, double sigma, const double *A, const double *x, const double *Cv)
{
    double S, d0, d1, d2 = 0.0, n0, n1, n2 = 0.0, dn, dd;
    if (dim == 3) S = sqrt(((A[0] * A[0]) + A[1] * A[1]) + A[2] * A[2]);
    else          S = sqrt((A[0] * A[0]) + A[1] * A[1]);
    n0 = (sigma * A[0]) / S;
    n1 = (sigma * A[1]) / S;
    if (dim == 3) n2 = (sigma * A[2]) / S;
    d0 = x[0] - Cv[0];
    d1 = x[1] - Cv[1];
    if (dim == 3) d2 = x[2] - Cv[2];
    if (dim == 3) { dn = ((d0 * n0) + d1 * n1) + d2 * n2; dd = ((d0 * d0) + d1 * d1) + d2 * d2; }
    else          { dn = (d0 * n0) + d1 * n1;             dd = (d0 * d0) + d1 * d1; }
    if (dd == 0.0) return 1.0;
    return dn / sqrt(dd);
}

/* exported for the pins (aligned -> 1, 45 deg -> 0.70711) */
double orc_skewness(int dim, double sigma, const double *A, const double *x, const double *Cv)
{
    return skew_one(dim, sigma, A, x, Cv);
}

/* ===================================================================== */
/* O3. Agglomeration, Algorithm 3: hash-select interior faces */
/* (boundary and parallel-interface faces never deleted), then for */
/* each selected face in selection order merge its two cells iff neither  */
/* is merged yet and min over the virtual cell's faces of sin(alpha) >=   */
/* theta (A21, A22 pairwise).  Coarse ids: scan fine cells ascending.     */
/* part: cell -> partition (NULL = one partition).                        */
/* Returns the number of merges (0 => stall), parent[] filled, *n_coarse. */
/* Pins: ≤2 children, re-evaluated decisions, 2-cell aligned pair merges   */
/* (S:183), conservation of the built level (tests).                      */
/* ===================================================================== */
int64_t orc_agglomerate(const orc_level *L, double theta, const int32_t *part,
                        int64_t *parent, int64_t *n_coarse)
{
    int dim = L->dim;
    int64_t nfi = 0;
    for (int64_t f = 0; f < L->nf; ++f) if (L->right[f] >= 0) nfi++;
    int64_t *mate = malloc(sizeof(int64_t) * (size_t)(L->n + 1));
    for (int64_t i = 0; i < L->n; ++i) mate[i] = -1;
    int64_t merges = 0;
    if (nfi > 0) {
        /* Alg.3 first loop: the collection V_d of faces to delete */
        unsigned char *seen = calloc((size_t)nfi, 1);
        int64_t *sel = malloc(sizeof(int64_t) * (size_t)nfi);
        int64_t nsel = 0;
        for (int64_t f = 0; f < L->nf; ++f) {
            int64_t l = L->left[f], r = L->right[f];
            if (r < 0) continue;                                  /* boundary face */
            if (part && part[l] != part[r]) continue;            /* parallel interface */
            uint64_t h = orc_face_hash((uint64_t)l, (uint64_t)r, (uint64_t)nfi);
            if (!seen[h]) { seen[h] = 1; sel[nsel++] = f; }
        }
        free(seen);
        int64_t *off, *idx;
        cell_faces(L, &off, &idx);
        /* Alg.3 second loop */
        for (int64_t s = 0; s < nsel; ++s) {
            int64_t f = sel[s], l = L->left[f], r = L->right[f];
            if (mate[l] >= 0 || mate[r] >= 0) continue;
            double Vl = L->vol[l], Vr = L->vol[r], Cv[3] = {0, 0, 0};
            for (int k = 0; k < dim; ++k)                         /* Eq.(virtual center) P:589-591 */
                Cv[k] = (Vl * L->ctr[k * L->n + l] + Vr * L->ctr[k * L->n + r]) / (Vl + Vr);
            double smin = 2.0;
            for (int side = 0; side < 2; ++side) {
                int64_t c = side == 0 ? l : r;
                for (int64_t a = off[c]; a < off[c + 1]; ++a) {
                    int64_t g = idx[a];
                    int64_t gl = L->left[g], gr = L->right[g];
                    if ((gl == l && gr == r) || (gl == r && gr == l)) continue;   /* the deleted face */
                    double sigma = (gl == c) ? 1.0 : -1.0;
                    double A[3] = {0, 0, 0}, x[3] = {0, 0, 0};
                    for (int k = 0; k < dim; ++k) { A[k] = L->avec[k * L->nf + g]; x[k] = L->fctr[k * L->nf + g]; }
                    double sg = skew_one(dim, sigma, A, x, Cv);
                    if (sg < smin) smin = sg;
                }
            }
            if (smin >= theta) { mate[l] = r; mate[r] = l; merges++; }
        }
        free(off); free(idx); free(sel);
    }
    int64_t nc = 0;
    for (int64_t i = 0; i < L->n; ++i) {
        if (mate[i] >= 0 && mate[i] < i) parent[i] = parent[mate[i]];
        else parent[i] = nc++;
    }
    *n_coarse = nc;
    free(mate);
    return merges;
}

/* ===================================================================== */
/* O1. Coarse level geometry (P:620-627 V_c = sum V_i, C_c = sum V_i C_i / */
/* V_c) and coarse faces (reading A23: one aggregated face per coarse     */
/* pair a<b, A = sum sigma A_f oriented a->b, x = sum|A_f| x_f / sum|A_f|, */
/* M = max M_f; boundary faces carried one-to-one after, fine-face order).*/
/* Two calls: count (out == NULL) then fill.                              */
/* Pins: V_c = sum V exactly, V_c C_c = sum V C, per-cell closure,         */
/* boundary area preserved (tests).                                       */
/* ===================================================================== */
typedef struct { int64_t a, b, f; } pairrec;
static int cmp_pair(const void *x, const void *y)
{
    const pairrec *p = x, *q = y;
    if (p->a != q->a) return p->a < q->a ? -1 : 1;
    if (p->b != q->b) return p->b < q->b ? -1 : 1;
    if (p->f != q->f) return p->f < q->f ? -1 : 1;
    return 0;
}

typedef struct {
    double *vol, *ctr;            /* [nc], [dim][nc] */
    int64_t *left, *right;        /* [nfc] */
    double *avec, *fctr;          /* [dim][nfc] */
    int8_t *ngauss;               /* [nfc] */
} orc_level_out;

int64_t orc_coarse_build(const orc_level *L, const int64_t *parent, int64_t nc, orc_level_out *out)
{
    int dim = L->dim;
    int64_t np = 0, nb = 0;
    if (nc <= 0 || nc > L->n) return -1;
    pairrec *pr = malloc(sizeof(pairrec) * (size_t)(L->nf + 1));
    for (int64_t f = 0; f < L->nf; ++f) {
        if (L->right[f] < 0) { nb++; continue; }
        int64_t pa = parent[L->left[f]], pb = parent[L->right[f]];
        if (pa == pb) continue;                                   /* deleted (now internal) */
        pairrec p = { pa < pb ? pa : pb, pa < pb ? pb : pa, f };
        pr[np++] = p;
    }
    qsort(pr, (size_t)np, sizeof(pairrec), cmp_pair);
    int64_t nci = 0;
    for (int64_t k = 0; k < np; ++k)
        if (k == 0 || pr[k].a != pr[k - 1].a || pr[k].b != pr[k - 1].b) nci++;
    int64_t nfc = nci + nb;
    if (!out) { free(pr); return nfc; }

    /* cells: children in ascending natural id */
    for (int64_t c = 0; c < nc; ++c) out->vol[c] = 0.0;
    double *vc = calloc((size_t)(dim * nc), sizeof(double));
    char *started = calloc((size_t)nc, 1);
    for (int64_t i = 0; i < L->n; ++i) {
        int64_t c = parent[i];
        if (!started[c]) {
            started[c] = 1;
            out->vol[c] = L->vol[i];
            for (int k = 0; k < dim; ++k) vc[k * nc + c] = L->vol[i] * L->ctr[k * L->n + i];
        } else {
            out->vol[c] = out->vol[c] + L->vol[i];
            for (int k = 0; k < dim; ++k) vc[k * nc + c] = vc[k * nc + c] + L->vol[i] * L->ctr[k * L->n + i];
        }
    }
    for (int64_t c = 0; c < nc; ++c)
        for (int k = 0; k < dim; ++k) out->ctr[k * nc + c] = vc[k * nc + c] / out->vol[c];
    free(vc); free(started);

    /* interior coarse faces, lexicographic (a, b); fine faces ascending */
    int64_t fo = -1;
    double sw = 0.0, sx[3] = {0, 0, 0};
    for (int64_t k = 0; k < np; ++k) {
        int64_t f = pr[k].f;
        int first = (k == 0 || pr[k].a != pr[k - 1].a || pr[k].b != pr[k - 1].b);
        if (first) {
            if (fo >= 0) for (int q = 0; q < dim; ++q) out->fctr[q * nfc + fo] = sx[q] / sw;
            fo++;
            out->left[fo] = pr[k].a; out->right[fo] = pr[k].b; out->ngauss[fo] = 0;
            for (int q = 0; q < dim; ++q) { out->avec[q * nfc + fo] = 0.0; sx[q] = 0.0; }
            sw = 0.0;
        }
        double sigma = (parent[L->left[f]] == pr[k].a) ? 1.0 : -1.0;
        double A[3] = {0, 0, 0};
        for (int q = 0; q < dim; ++q) A[q] = L->avec[q * L->nf + f];
        double S = dim == 3 ? sqrt(((A[0] * A[0]) + A[1] * A[1]) + A[2] * A[2])
                            : sqrt((A[0] * A[0]) + A[1] * A[1]);
        for (int q = 0; q < dim; ++q) {
            out->avec[q * nfc + fo] = out->avec[q * nfc + fo] + sigma * A[q];
            sx[q] = sx[q] + S * L->fctr[q * L->nf + f];
        }
        sw = sw + S;
        if (L->ngauss[f] > out->ngauss[fo]) out->ngauss[fo] = L->ngauss[f];
    }
    if (fo >= 0) for (int q = 0; q < dim; ++q) out->fctr[q * nfc + fo] = sx[q] / sw;
    /* boundary faces, fine-face order */
    for (int64_t f = 0; f < L->nf; ++f) {
        if (L->right[f] >= 0) continue;
        fo++;
        out->left[fo] = parent[L->left[f]];
        out->right[fo] = L->right[f];
        out->ngauss[fo] = L->ngauss[f];
        for (int q = 0; q < dim; ++q) {
            out->avec[q * nfc + fo] = L->avec[q * L->nf + f];
            out->fctr[q * nfc + fo] = L->fctr[q * L->nf + f];
        }
    }
    free(pr);
    return nfc;
}

/* ===================================================================== */
/* Gas state helpers (definitions; gamma-law gas)        */
/* ===================================================================== */
static double pressure(int dim, double gamma, const double *W)
{
    double m2 = 0.0;
    for (int k = 0; k < dim; ++k) m2 += W[1 + k] * W[1 + k];
    return (gamma - 1.0) * (W[dim + 1] - 0.5 * m2 / W[0]);
}

/* O4 ghost states (reading A25): FARFIELD W_inf, SLIP m - 2(m.n)n,        */
/* NOSLIP -m, EXTRAP W_i.  n: unit normal outward from the interior cell. */
static void ghost_state(int dim, int kind, const double *Wi, const double *Winf, const double *n, double *Wg)
{
    int nv = dim + 2;
    if (kind == ORC_FARFIELD) { for (int q = 0; q < nv; ++q) Wg[q] = Winf[q]; return; }
    for (int q = 0; q < nv; ++q) Wg[q] = Wi[q];
    if (kind == ORC_SLIP) {
        double mn = 0.0;
        for (int k = 0; k < dim; ++k) mn += Wi[1 + k] * n[k];
        for (int k = 0; k < dim; ++k) Wg[1 + k] = Wi[1 + k] - 2.0 * mn * n[k];
    } else if (kind == ORC_NOSLIP) {
        for (int k = 0; k < dim; ++k) Wg[1 + k] = -Wi[1 + k];
    }
}

/* exported for cgks3.c (NEXT-1): the same ghost states */
void orc_ghost(int dim, int kind, const double *Wi, const double *Winf, const double *n, double *Wg)
{
    ghost_state(dim, kind, Wi, Winf, n, Wg);
}

/* ===================================================================== */
/* O4. First-order KFVS flux (coarse operator named at P:637; free-       */
/* transport of two Maxwellians) per unit area along unit n:   */
/* F = F(left, +) + F(right, -), half-range moments with erfc / exp and   */
/* the recurrence <u^{k+2}> = U<u^{k+1}> + (k+1)/(2 lambda) <u^k>.        */
/* K = (5-3g)/(g-1) in 3D, (4-2g)/(g-1) in 2D (A27).       */
/* Pins: equal states give the Euler flux exactly up to rounding          */
/* (erfc(x)+erfc(-x)=2); stationary: mass 0, momentum p; Gauss-   */
/* Hermite quadrature of the half-Maxwellians (tests, scipy); supersonic  */
/* upwind limit.                                                          */
/* ===================================================================== */
static void kfvs_half(int dim, double gamma, const double *W, const double *n, int plus, double *F)
{
    double K = (dim == 3) ? (5.0 - 3.0 * gamma) / (gamma - 1.0) : (4.0 - 2.0 * gamma) / (gamma - 1.0);
    double rho = W[0], u[3] = {0, 0, 0}, U = 0.0, u2 = 0.0;
    for (int k = 0; k < dim; ++k) { u[k] = W[1 + k] / rho; U += u[k] * n[k]; u2 += u[k] * u[k]; }
    double p = pressure(dim, gamma, W);
    double lambda = rho / (2.0 * p);
    double sl = sqrt(lambda);
    double e = exp(-lambda * U * U) / (2.0 * sqrt(M_PI * lambda));
    double m0, m1;
    if (plus) { m0 = 0.5 * erfc(-sl * U); m1 = U * m0 + e; }
    else      { m0 = 0.5 * erfc(sl * U);  m1 = U * m0 - e; }
    double m2 = U * m1 + (1.0 / (2.0 * lambda)) * m0;       /* k = 0 */
    double m3 = U * m2 + (2.0 / (2.0 * lambda)) * m1;       /* k = 1 */
    F[0] = rho * m1;
    for (int k = 0; k < dim; ++k) F[1 + k] = rho * m2 * n[k] + rho * m1 * (u[k] - U * n[k]);
    F[dim + 1] = 0.5 * rho * (m3 + m1 * (u2 - U * U + ((double)(dim - 1) + K) / (2.0 * lambda)));
}

void orc_kfvs_flux(int dim, double gamma, const double *WL, const double *WR, const double *n, double *F)
{
    double Fp[5], Fm[5];
    kfvs_half(dim, gamma, WL, n, 1, Fp);
    kfvs_half(dim, gamma, WR, n, 0, Fm);
    for (int q = 0; q < dim + 2; ++q) F[q] = Fp[q] + Fm[q];
}

/* O5. DF helper per face (P:353-365 evaluated with first-order states,  */
/* readings A16, A17): D = |pl-pr|/pl + |pl-pr|/pr + (Ma_n^l - Ma_n^r)^2   */
/* + |Ma_t^l - Ma_t^r|^2, alpha = 1/(1+D^2).                               */
/* Pins: S:264-266 (p 2|1 -> 0.307692; dMa_n = 1 -> 0.5), equal -> 1.      */
double orc_df_face(int dim, double gamma, const double *WL, const double *WR, const double *n)
{
    double pl = pressure(dim, gamma, WL), pr = pressure(dim, gamma, WR);
    double al = sqrt(gamma * pl / WL[0]), ar = sqrt(gamma * pr / WR[0]);
    double ul[3] = {0, 0, 0}, ur[3] = {0, 0, 0}, Ul = 0.0, Ur = 0.0;
    for (int k = 0; k < dim; ++k) {
        ul[k] = WL[1 + k] / WL[0]; ur[k] = WR[1 + k] / WR[0];
        Ul += ul[k] * n[k]; Ur += ur[k] * n[k];
    }
    double dMn = Ul / al - Ur / ar;
    double dMt2 = 0.0;
    for (int k = 0; k < dim; ++k) {
        double t = (ul[k] - Ul * n[k]) / al - (ur[k] - Ur * n[k]) / ar;
        dMt2 += t * t;
    }
    double D = fabs(pl - pr) / pl + fabs(pl - pr) / pr + dMn * dMn + dMt2;
    return 1.0 / (1.0 + D * D);
}

/* O6. interface spectral radius r = omega (|u.n| + a) of the conservative */
/* average W = (W_L + W_G)/2 (reading A5).  Pin: S:433 -> 2.18322. */
double orc_spectral_radius(int dim, double gamma, double omega, const double *WL, const double *WR, const double *n)
{
    double Wb[5];
    for (int q = 0; q < dim + 2; ++q) Wb[q] = 0.5 * (WL[q] + WR[q]);
    double p = pressure(dim, gamma, Wb), U = 0.0;
    for (int k = 0; k < dim; ++k) U += (Wb[1 + k] / Wb[0]) * n[k];
    return omega * (fabs(U) + sqrt(gamma * p / Wb[0]));
}

/* Euler flux T(W; n) = (rho U, m U + p n, (rho E + p) U), U = u.n */
/* Pin: S:442 (1,2,0,4).                                                   */
void orc_euler_flux(int dim, double gamma, const double *W, const double *n, double *T)
{
    double U = 0.0;
    for (int k = 0; k < dim; ++k) U += (W[1 + k] / W[0]) * n[k];
    double p = pressure(dim, gamma, W);
    T[0] = W[0] * U;
    for (int k = 0; k < dim; ++k) T[1 + k] = W[1 + k] * U + p * n[k];
    T[dim + 1] = (W[dim + 1] + p) * U;
}

/* ===================================================================== */
/* Residual R_i = sum_f sigma_if S_f F_f (P:437-440 Eq.(resform), reading  */
/* A4: flux sum, not volume-normalised), with per-face r_f (O6), per-cell */
/* Sigma_i = sum_f S_f r_f over ALL faces (A6) and the DF helper alpha_i = */
/* prod_f alpha_f^{M_f} over all faces (O5).  Outputs natural order:       */
/* R [nv][n], alpha [n], Sigma [n], rf [nf] (may be NULL).                 */
/* Pins: free-stream residual ~ 0 on any mesh (closure P:454); telescoping */
/* of the restricted residual.                                     */
/* ===================================================================== */
void orc_residual(const orc_level *L, double gamma, double omega, const double *W, const double *Winf,
                  double *R, double *alpha, double *Sigma, double *rf)
{
    int dim = L->dim, nv = dim + 2;
    int64_t n = L->n, nf = L->nf;
    /* per face: S, S F (flux, KFVS), r, alpha_f^{M_f} -- independent evaluations */
    double *fS = malloc(sizeof(double) * (size_t)(nf + 1));
    double *fF = malloc(sizeof(double) * (size_t)(nv * nf + 1));
    double *fr = malloc(sizeof(double) * (size_t)(nf + 1));
    double *fa = malloc(sizeof(double) * (size_t)(nf + 1));
#pragma omp parallel for schedule(static)
    for (int64_t f = 0; f < nf; ++f) {
        int64_t l = L->left[f], r = L->right[f];
        double A[3] = {0, 0, 0}, nn[3] = {0, 0, 0};
        for (int k = 0; k < dim; ++k) A[k] = L->avec[k * nf + f];
        double S = 0.0;
        for (int k = 0; k < dim; ++k) S += A[k] * A[k];
        S = sqrt(S);
        for (int k = 0; k < dim; ++k) nn[k] = A[k] / S;
        double WL[5], WR[5], F[5];
        for (int q = 0; q < nv; ++q) WL[q] = W[q * n + l];
        if (r >= 0) for (int q = 0; q < nv; ++q) WR[q] = W[q * n + r];
        else ghost_state(dim, L->patch_kind[-r - 1], WL, Winf, nn, WR);
        orc_kfvs_flux(dim, gamma, WL, WR, nn, F);
        double af = orc_df_face(dim, gamma, WL, WR, nn);
        double afM = 1.0;
        for (int g = 0; g < L->ngauss[f]; ++g) afM *= af;
        fS[f] = S;
        for (int q = 0; q < nv; ++q) fF[q * nf + f] = F[q];
        fr[f] = orc_spectral_radius(dim, gamma, omega, WL, WR, nn);
        fa[f] = afM;
    }
    /* assembly in face order: R_i = sum_f sigma_if S_f F_f, Sigma_i = sum_f S_f r_f, alpha_i = prod_f alpha_f^M_f */
    for (int q = 0; q < nv; ++q) for (int64_t i = 0; i < n; ++i) R[q * n + i] = 0.0;
    for (int64_t i = 0; i < n; ++i) { if (alpha) alpha[i] = 1.0; if (Sigma) Sigma[i] = 0.0; }
    for (int64_t f = 0; f < nf; ++f) {
        int64_t l = L->left[f], r = L->right[f];
        double S = fS[f], rr = fr[f], afM = fa[f];
        if (rf) rf[f] = rr;
        for (int q = 0; q < nv; ++q) R[q * n + l] += S * fF[q * nf + f];
        if (Sigma) Sigma[l] += S * rr;
        if (alpha) alpha[l] *= afM;
        if (r >= 0) {
            for (int q = 0; q < nv; ++q) R[q * n + r] -= S * fF[q * nf + f];
            if (Sigma) Sigma[r] += S * rr;
            if (alpha) alpha[r] *= afM;
        }
    }
    free(fS); free(fF); free(fr); free(fa);
}

/* O6. DF-hybrid diagonal (Eq.(gpu-forward-relaxation) P:538 with readings */
/* A2, A3: Dt_imp|exp = CFL_imp|exp V / Sigma):                            */
/* D_i = alpha (V/Dt_imp + Sigma/2) + (1 - alpha) V/Dt_exp                 */
/*     = Sigma [alpha (1/CFL_imp + 1/2) + (1 - alpha)/CFL_exp].            */
/* Pins: S:453 -> 11; alpha = 0 -> V/Dt_exp; alpha = 1 -> V/Dt + Sigma/2.  */
void orc_diag(int64_t n, const double *Sigma, const double *alpha, double cfl_imp, double cfl_exp, double *D)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
        D[i] = alpha[i] * (Sigma[i] / cfl_imp + 0.5 * Sigma[i]) + (1.0 - alpha[i]) * (Sigma[i] / cfl_exp);
}

/* ===================================================================== */
/* O7. MC-SGS smoothing step: Algorithm 2 with the DF-relaxed  */
/* sweeps Eq.(gpu-forward-relaxation) / Eq.(gpu-backward-relaxation)       */
/* (P:536-551), readings A1 (blended D both sides) and A7 (every half-     */
/* sweep reads all neighbours' current increments; sweep 1 equals the     */
/* printed equations):                                                     */
/*   dW_i <- -( Rt_i + 1/2 alpha_i sum_{interior f ni i, j = other(f)}     */
/*             S_f [T(W_j+dW_j; sigma n_f) - T(W_j; sigma n_f)             */
/*                  - r_f dW_j] ) / D_i                                    */
/* colors 1..Nc then Nc..1, cells of a color in ascending id, n_sweeps    */
/* times; boundary faces: no off-diagonal (ghost dW = 0, A6).             */
/* dW (out) [nv][n].                                                      */
/* Pins: alpha = 0 explicit identity, isolated cell -R/D, sweep 1  */
/* = literal printed forward/backward, sequential GS brute force, linear- */
/* flux reduction to scipy SGS, fixed point vs dense Newton (tests).      */
/* ===================================================================== */
void orc_smooth(const orc_level *L, double gamma, const double *W, const double *Rt, const double *alpha,
                const double *D, const double *rf, const int32_t *color, int ncolor, int n_sweeps, double *dW)
{
    int dim = L->dim, nv = dim + 2;
    int64_t n = L->n;
    int64_t *off, *idx;
    cell_faces(L, &off, &idx);
    for (int q = 0; q < nv; ++q) for (int64_t i = 0; i < n; ++i) dW[q * n + i] = 0.0;
    for (int s = 0; s < n_sweeps; ++s) {
        for (int half = 0; half < 2; ++half) {
            for (int cc = 0; cc < ncolor; ++cc) {
                int c = half == 0 ? cc + 1 : ncolor - cc;      /* forward 1..Nc, backward Nc..1 */
                /* cells of one color never neighbour each other: independent updates */
#pragma omp parallel for schedule(dynamic, 256)
                for (int64_t i = 0; i < n; ++i) {
                    if (color[i] != c) continue;
                    double sum[5] = {0, 0, 0, 0, 0};
                    for (int64_t a = off[i]; a < off[i + 1]; ++a) {
                        int64_t f = idx[a];
                        if (L->right[f] < 0) continue;
                        int64_t j = (L->left[f] == i) ? L->right[f] : L->left[f];
                        double sigma = (L->left[f] == i) ? 1.0 : -1.0;
                        double A[3] = {0, 0, 0}, nn[3] = {0, 0, 0}, S = 0.0;
                        for (int k = 0; k < dim; ++k) { A[k] = L->avec[k * L->nf + f]; S += A[k] * A[k]; }
                        S = sqrt(S);
                        for (int k = 0; k < dim; ++k) nn[k] = sigma * A[k] / S;
                        double Wj[5], Wjd[5], dWj[5], T1[5], T0[5];
                        for (int q = 0; q < nv; ++q) {
                            Wj[q] = W[q * n + j];
                            dWj[q] = dW[q * n + j];
                            Wjd[q] = Wj[q] + dWj[q];
                        }
                        orc_euler_flux(dim, gamma, Wjd, nn, T1);
                        orc_euler_flux(dim, gamma, Wj, nn, T0);
                        for (int q = 0; q < nv; ++q) sum[q] += S * (T1[q] - T0[q] - rf[f] * dWj[q]);
                    }
                    for (int q = 0; q < nv; ++q)
                        dW[q * n + i] = -(Rt[q * n + i] + 0.5 * alpha[i] * sum[q]) / D[i];
                }
            }
        }
    }
    free(off); free(idx);
}

/* ===================================================================== */
/* O8 pieces.                                                             */
/* ===================================================================== */
/* Eq.(smo) P:638-641 with reading A9: W <- W - (Dt_exp/V) R,              */
/* Dt_exp = CFL_exp V / Sigma.                                             */
void orc_explicit_update(int64_t n, int nv, double cfl_exp, const double *Sigma, const double *R, double *W)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
        for (int q = 0; q < nv; ++q) W[q * n + i] = W[q * n + i] - (cfl_exp / Sigma[i]) * R[q * n + i];
}

/* State restriction W0_2h = sum V W / V_2h, residual          */
/* restriction Res* = sum Res, DF restriction alpha = min      */
/* (reading A15).  Children in ascending natural id.                       */
/* Pins: sum V_c W0_c = sum V W, S:520 -> 4, telescoping.  */
void orc_restrict(int64_t nfine, int64_t nc, int nv, const int64_t *parent, const double *vol_f,
                  const double *vol_c, const double *Wf, const double *Rf, const double *af,
                  double *W0c, double *Rc, double *ac)
{
    char *started = calloc((size_t)nc, 1);
    for (int64_t i = 0; i < nfine; ++i) {
        int64_t c = parent[i];
        if (!started[c]) {
            started[c] = 1;
            for (int q = 0; q < nv; ++q) { W0c[q * nc + c] = vol_f[i] * Wf[q * nfine + i]; Rc[q * nc + c] = Rf[q * nfine + i]; }
            ac[c] = af[i];
        } else {
            for (int q = 0; q < nv; ++q) {
                W0c[q * nc + c] = W0c[q * nc + c] + vol_f[i] * Wf[q * nfine + i];
                Rc[q * nc + c] = Rc[q * nc + c] + Rf[q * nfine + i];
            }
            if (af[i] < ac[c]) ac[c] = af[i];
        }
    }
    for (int64_t c = 0; c < nc; ++c)
        for (int q = 0; q < nv; ++q) W0c[q * nc + c] = W0c[q * nc + c] / vol_c[c];
    free(started);
}

/* DF-limited prolongation Eq.(prolongation) P:672-678 with piecewise-     */
/* constant injection (A13): W_h += alpha_h (W_2h - W0_2h)[parent].        */
/* Pins: alpha = 0 leaves cells bit-identical, uniform shift. */
void orc_prolong(int64_t nfine, int64_t nc, int nv, const int64_t *parent, const double *alpha_f,
                 const double *Wc, const double *W0c, double *Wf)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nfine; ++i) {
        int64_t c = parent[i];
        for (int q = 0; q < nv; ++q)
            Wf[q * nfine + i] = Wf[q * nfine + i] + alpha_f[i] * (Wc[q * nc + c] - W0c[q * nc + c]);
    }
}
