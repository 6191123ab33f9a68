// plan.cu -- GPU plan build (T_pre of the paper): Morton-sorted box octree,
// neighbour / cousin lists, cone grids and the relevant cone segments of
// every level (eq. defallrelevantconesegments).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "ifgf_internal.cuh"

namespace ifgf {

namespace {

constexpr int TPB = 256;

inline int nblocks(int64_t n, int tpb = TPB) {
    int64_t b = (n + tpb - 1) / tpb;
    if (b < 1) b = 1;
    if (b > 2147483647) b = 2147483647;
    return (int)b;
}

// ---------------------------------------------------------------- validation
__global__ void k_minmax(const double* __restrict__ pts, int64_t n, double* part, int* bad) {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    int nonfinite = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        for (int a = 0; a < 3; ++a) {
            double v = pts[3 * i + a];
            if (!isfinite(v)) nonfinite = 1;
            lo[a] = fmin(lo[a], v);
            hi[a] = fmax(hi[a], v);
        }
    }
    __shared__ double s[6][TPB];
    for (int a = 0; a < 3; ++a) {
        s[a][threadIdx.x] = lo[a];
        s[3 + a][threadIdx.x] = hi[a];
    }
    if (nonfinite) atomicOr(bad, 1);
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w)
            for (int a = 0; a < 3; ++a) {
                s[a][threadIdx.x] = fmin(s[a][threadIdx.x], s[a][threadIdx.x + w]);
                s[3 + a][threadIdx.x] = fmax(s[3 + a][threadIdx.x], s[3 + a][threadIdx.x + w]);
            }
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int a = 0; a < 6; ++a) part[6 * blockIdx.x + a] = s[a][0];
}

// --------------------------------------------------------------- Morton keys
__device__ __forceinline__ uint64_t spread3(uint64_t v) {  // bit b -> bit 3b
    uint64_t r = 0;
    for (int b = 0; b < 21; ++b) r |= ((v >> b) & 1ull) << (3 * b);
    return r;
}
__device__ __forceinline__ int compact3(uint64_t v) {
    int r = 0;
    for (int b = 0; b < 21; ++b) r |= (int)((v >> (3 * b)) & 1ull) << b;
    return r;
}
__device__ __forceinline__ uint64_t morton(int qx, int qy, int qz) {
    return (spread3((uint64_t)qx) << 2) | (spread3((uint64_t)qy) << 1) | spread3((uint64_t)qz);
}

// Leaf coordinates q = clamp(floor((x - x0)/H_D)) (contract) and keys.
__global__ void k_keys(const double* __restrict__ pts, int64_t n, double x0x, double x0y, double x0z, double HD,
                       int nmax, uint64_t* keys, int* idx) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double x0[3] = {x0x, x0y, x0z};
    int q[3];
    for (int a = 0; a < 3; ++a) {
        double t = floor(__ddiv_rn(__dsub_rn(pts[3 * i + a], x0[a]), HD));
        q[a] = t < 0.0 ? 0 : (t >= (double)nmax ? nmax - 1 : (int)t);
    }
    keys[i] = morton(q[0], q[1], q[2]);
    idx[i] = (int)i;
}

__global__ void k_gather_points(const double* __restrict__ pts, const int* __restrict__ perm, int64_t n, double* px,
                                double* py, double* pz) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t j = perm[i];
    px[i] = pts[3 * j];
    py[i] = pts[3 * j + 1];
    pz[i] = pts[3 * j + 2];
}

// ------------------------------------------------------------- box building
__global__ void k_flag_runs(const uint64_t* __restrict__ key, int64_t n, int shift, int* flag) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    flag[i] = (i == 0 || (key[i] >> shift) != (key[i - 1] >> shift)) ? 1 : 0;
}

// Leaf level: box index per point from the inclusive scan; box start and key.
__global__ void k_leaf_boxes(const uint64_t* __restrict__ key, const int* __restrict__ flag,
                             const int* __restrict__ incl, int64_t n, int* box_start, uint64_t* box_key) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (flag[i]) {
        int b = incl[i] - 1;
        box_start[b] = (int)i;
        box_key[b] = key[i];
    }
}

// Coarser level d-1 from level d boxes.
__global__ void k_parent_boxes(const uint64_t* __restrict__ key_d, const int* __restrict__ start_d,
                               const int* __restrict__ flag, const int* __restrict__ incl, int64_t nb, int* parent_d,
                               int* start_p, uint64_t* key_p, int* child_start_p) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= nb) return;
    int q = incl[b] - 1;
    parent_d[b] = q;
    if (flag[b]) {
        start_p[q] = start_d[b];
        key_p[q] = key_d[b] >> 3;
        child_start_p[q] = (int)b;
    }
}

__global__ void k_box_ijk(const uint64_t* __restrict__ key, int64_t nb, int* ijk) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= nb) return;
    uint64_t k = key[b];
    ijk[3 * b] = compact3(k >> 2);
    ijk[3 * b + 1] = compact3(k >> 1);
    ijk[3 * b + 2] = compact3(k);
}

// Box centres x0 + (k + 1/2) H_d, IEEE-rounded exactly as box_centre (eq.
// defboxsizesandcenters), 4 doubles per box for aligned loads.
__global__ void k_box_c(const int* __restrict__ ijk, int64_t nb, LevelParams L, double* c) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= nb) return;
    for (int a = 0; a < 3; ++a) c[4 * b + a] = box_centre(L, ijk[3 * b + a], a);
    c[4 * b + 3] = 0.0;
}

// Pairwise-different points: coincident points share a leaf.
__global__ void k_coincident(const double* __restrict__ px, const double* __restrict__ py,
                             const double* __restrict__ pz, const int* __restrict__ start, int64_t nb, int* bad) {
    int64_t b = blockIdx.x;
    if (b >= nb) return;
    int s0 = start[b], s1 = start[b + 1];
    for (int i = s0 + threadIdx.x; i < s1; i += blockDim.x)
        for (int j = i + 1; j < s1; ++j)
            if (px[i] == px[j] && py[i] == py[j] && pz[i] == pz[j]) atomicOr(bad, 1);
}

__device__ __forceinline__ int64_t find_key(const uint64_t* __restrict__ keys, int64_t nb, uint64_t k) {
    int64_t lo = 0, hi = nb;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (keys[mid] < k) lo = mid + 1; else hi = mid;
    }
    return (lo < nb && keys[lo] == k) ? lo : -1;
}

// Neighbours N B: relevant boxes with ||a - k||_inf <= 1, B included.
// pass 0: count into cnt[b]; pass 1: fill idx from off[b].
__global__ void k_neighbours(const uint64_t* __restrict__ keys, const int* __restrict__ ijk, int64_t nb, int nside,
                             int pass, int* cnt, const int* __restrict__ off, int* idx) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= nb) return;
    int i0 = ijk[3 * b], j0 = ijk[3 * b + 1], k0 = ijk[3 * b + 2];
    int c = 0;
    int64_t o = pass ? off[b] : 0;
    for (int di = -1; di <= 1; ++di)
        for (int dj = -1; dj <= 1; ++dj)
            for (int dk = -1; dk <= 1; ++dk) {
                int i = i0 + di, j = j0 + dj, k = k0 + dk;
                if (i < 0 || j < 0 || k < 0 || i >= nside || j >= nside || k >= nside) continue;
                int64_t a = find_key(keys, nb, morton(i, j, k));
                if (a < 0) continue;
                if (pass) idx[o + c] = (int)a;
                ++c;
            }
    if (!pass) cnt[b] = c;
}

// Cousins M B = (R_B^d \ N B) cap Q N P B (eq. defcousinboxes).
__global__ void k_cousins(const int* __restrict__ ijk, const int* __restrict__ parent, int64_t nb,
                          const int* __restrict__ pnbr_off, const int* __restrict__ pnbr_idx,
                          const int* __restrict__ pchild_start, int pass, int* cnt, const int* __restrict__ off,
                          int* idx) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= nb) return;
    int i0 = ijk[3 * b], j0 = ijk[3 * b + 1], k0 = ijk[3 * b + 2];
    int P = parent[b];
    int c = 0;
    int64_t o = pass ? off[b] : 0;
    for (int e = pnbr_off[P]; e < pnbr_off[P + 1]; ++e) {
        int A = pnbr_idx[e];
        for (int ch = pchild_start[A]; ch < pchild_start[A + 1]; ++ch) {
            int dist = max(abs(ijk[3 * ch] - i0), max(abs(ijk[3 * ch + 1] - j0), abs(ijk[3 * ch + 2] - k0)));
            if (dist < 2) continue;
            if (pass) idx[o + c] = ch;
            ++c;
        }
    }
    if (!pass) cnt[b] = c;
}

// Partition work units per box: near-field pairs of a leaf as
// source (its points times the points of its neighbour leaves, minus the self
// pairs) and cousin evaluations of a box as source (the points of its cousins).
__global__ void k_box_units(const int* __restrict__ start, const int* __restrict__ nbr_off,
                            const int* __restrict__ nbr_idx, const int* __restrict__ cou_off,
                            const int* __restrict__ cou_idx, int64_t nb, double* near_units, double* cou_units) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= nb) return;
    const double nbx = (double)(start[b + 1] - start[b]);
    if (near_units) {
        int64_t s = 0;
        for (int e = nbr_off[b]; e < nbr_off[b + 1]; ++e) s += start[nbr_idx[e] + 1] - start[nbr_idx[e]];
        near_units[b] = nbx * (double)s - nbx;
    }
    if (cou_units) {
        int64_t s = 0;
        if (cou_off)
            for (int e = cou_off[b]; e < cou_off[b + 1]; ++e) s += start[cou_idx[e] + 1] - start[cou_idx[e]];
        cou_units[b] = (double)s;
    }
}

// Warp work items: (box, first point) chunks of 32 points.
__global__ void k_witem_count(const int* __restrict__ start, int64_t nb, int* cnt) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= nb) return;
    cnt[b] = (start[b + 1] - start[b] + 31) / 32;
}
__global__ void k_witem_fill(const int* __restrict__ start, int64_t nb, const int* __restrict__ off, int2* items) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= nb) return;
    int o = off[b];
    for (int p = start[b]; p < start[b + 1]; p += 32) items[o++] = make_int2((int)b, p);
}

// --------------------------------------------------------- relevance flags
__device__ __forceinline__ void set_bit(unsigned long long* bm, int64_t w, unsigned long long bit) {
    if (!(bm[w] & bit)) atomicOr(bm + w, bit);
}

// (i) cousin surface points: target-major over warp
// items of level d; every (point x in T, cousin B of T) classifies x - c_B.
__global__ void k_flag_cousin_points(LevelParams L, const double* __restrict__ px, const double* __restrict__ py,
                                     const double* __restrict__ pz, unsigned long long* bm, int* bad) {
    int64_t item = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (item >= L.nwitems) return;
    int2 it = L.witems[item];
    int T = it.x, l = it.y + lane;
    if (l >= L.box_start[T + 1]) return;
    double x = px[l], y = py[l], z = pz[l];
    for (int e = L.cou_off[T]; e < L.cou_off[T + 1]; ++e) {
        int B = L.cou_idx[e];
        if (B < L.b0 || B >= L.b1) continue;
        double cx, cy, cz;
        box_centre3(L, B, cx, cy, cz);
        Cls c = classify(L, __dsub_rn(x, cx), __dsub_rn(y, cy), __dsub_rn(z, cz));
        int64_t cell = cell_of(L, c);
        if (cell < 0 || cell >= L.ncell) { atomicOr(bad, 1); continue; }
        set_bit(bm, (B - L.b0) * L.W + (cell >> 6), 1ull << (cell & 63));
    }
}

// Node offset of node n = (kp*Pa + kt)*Ps + ks of cell `cell` at level LP
// (eq. interp_pts): r = h/s_k, (r sin th cos ph, r sin th sin ph, r cos th).
__device__ __forceinline__ void node_offset(const LevelParams& LP, int Ps, int Pa, int cell, int n, double off[3],
                                            double* r_out) {
    int is = cell % LP.ns;
    int ith = (cell / LP.ns) % LP.nC;
    int iph = cell / (LP.ns * LP.nC);
    int ks = n % Ps, kt = (n / Ps) % Pa, kp = n / (Ps * Pa);
    double r = __ldg(LP.rtab + is * Ps + ks);
    double st = __ldg(LP.st_tab + ith * Pa + kt), ct = __ldg(LP.ct_tab + ith * Pa + kt);
    double sp = __ldg(LP.sp_tab + iph * Pa + kp), cp = __ldg(LP.cp_tab + iph * Pa + kp);
    double rs = __dmul_rn(r, st);
    off[0] = __dmul_rn(rs, cp);
    off[1] = __dmul_rn(rs, sp);
    off[2] = __dmul_rn(r, ct);
    if (r_out) *r_out = r;
}

// (ii) nodes of relevant parent segments: thread per
// (parent segment, node); each owned child B of Q classifies off + delta.
__global__ void k_flag_parent_nodes(LevelParams L, LevelParams LP, int Ps, int Pa, unsigned long long* bm,
                                    int* bad) {
    const int P = Ps * Pa * Pa;
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= LP.nseg * P) return;
    int64_t s = t / P;
    int n = (int)(t - s * P);
    int Q = LP.seg_box[s];
    double off[3];
    node_offset(LP, Ps, Pa, LP.seg_cell[s], n, off, nullptr);
    const double hh = 0.5 * L.H;  // exact
    for (int B = LP.child_start[Q]; B < LP.child_start[Q + 1]; ++B) {
        if (B < L.b0 || B >= L.b1) continue;
        double dx = (L.box_ijk[3 * B] & 1) ? -hh : hh, dy = (L.box_ijk[3 * B + 1] & 1) ? -hh : hh,
               dz = (L.box_ijk[3 * B + 2] & 1) ? -hh : hh;
        Cls c = classify(L, __dadd_rn(off[0], dx), __dadd_rn(off[1], dy), __dadd_rn(off[2], dz));
        int64_t cell = cell_of(L, c);
        if (cell < 0 || cell >= L.ncell) { atomicOr(bad, 1); continue; }
        set_bit(bm, (B - L.b0) * L.W + (cell >> 6), 1ull << (cell & 63));
    }
}

// (ii'), the same flags by runs of parent segments sharing a cone cell: the
// child-relative geometry of a parent node depends only on (cell, node, octant)
// (DESIGN.md §7), so a warp per run classifies each (octant, node) once and sets
// that child cell's bit in every run segment's child box of that octant (one
// lane per distinct cell).  Same decisions as k_flag_parent_nodes, run-length
// times fewer classifications.  sorted_seg: parent segments sorted by cell;
// run_start: first sorted position of each run (runs cut every 32 segments).
__global__ void k_flag_parent_runs(LevelParams L, LevelParams LP, int Ps, int Pa, const int* __restrict__ sorted_seg,
                                   const int* __restrict__ run_start, int64_t nrun, unsigned long long* bm, int* bad) {
    const int P = Ps * Pa * Pa;
    const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= nrun) return;  // warp-uniform
    const int s_begin = run_start[r];
    const int s_end = (r + 1 < nrun) ? run_start[r + 1] : (int)LP.nseg;
    const int cell = LP.seg_cell[sorted_seg[s_begin]];
    // octants with a child in some run segment
    unsigned om = 0u;
    for (int s = s_begin + lane; s < s_end; s += 32) {
        const int Q = LP.seg_box[sorted_seg[s]];
        for (int o = 0; o < 8; ++o) {
            const int B = LP.child_oct[8 * Q + o];
            if (B >= L.b0 && B < L.b1) om |= 1u << o;
        }
    }
    om = __reduce_or_sync(~0u, om);
    const double hh = 0.5 * L.H;  // exact
    for (int n0 = 0; n0 < P; n0 += 32) {
        const int n = n0 + lane;
        double off[3] = {0.0, 0.0, 0.0};
        if (n < P) node_offset(LP, Ps, Pa, cell, n, off, nullptr);
        for (int o = 0; o < 8; ++o) {
            if (!((om >> o) & 1u)) continue;
            int64_t c = -1;
            if (n < P) {
                const double dx = (o & 4) ? -hh : hh, dy = (o & 2) ? -hh : hh, dz = (o & 1) ? -hh : hh;
                const Cls cl = classify(L, __dadd_rn(off[0], dx), __dadd_rn(off[1], dy), __dadd_rn(off[2], dz));
                c = cell_of(L, cl);
                if (c < 0 || c >= L.ncell) {
                    atomicOr(bad, 1);
                    c = -1;
                }
            }
            const unsigned grp = __match_any_sync(~0u, (unsigned long long)c);
            const bool lead = c >= 0 && lane == __ffs(grp) - 1;
            if (!__any_sync(~0u, lead)) continue;
            for (int s = s_begin; s < s_end; ++s) {
                const int Q = LP.seg_box[sorted_seg[s]];
                const int B = LP.child_oct[8 * Q + o];
                if (B < L.b0 || B >= L.b1 || !lead) continue;
                set_bit(bm, (B - L.b0) * L.W + (c >> 6), 1ull << (c & 63));
            }
        }
    }
}

__global__ void k_popc(const unsigned long long* __restrict__ bm, int64_t nw, unsigned* out) {
    int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (w >= nw) return;
    out[w] = (unsigned)__popcll(bm[w]);
}

__global__ void k_emit_segments(const unsigned long long* __restrict__ bm, const unsigned* __restrict__ rank,
                                int64_t nw, int64_t W, int64_t b0, int* seg_box, int* seg_cell) {
    int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (w >= nw) return;
    unsigned long long v = bm[w];
    if (!v) return;
    int64_t idx = rank[w];
    int b = (int)(b0 + w / W);
    int base = (int)((w % W) * 64);
    while (v) {
        int bit = __ffsll((long long)v) - 1;
        seg_box[idx] = b;
        seg_cell[idx] = base + bit;
        ++idx;
        v &= v - 1;
    }
}

// ------------------------------------------- K7 grouping by cone cell
__global__ void k_child_oct(const int* __restrict__ child_start, const int* __restrict__ ijk_child, int64_t nb,
                            int* child_oct) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= nb) return;
    for (int o = 0; o < 8; ++o) child_oct[8 * b + o] = -1;
    for (int ch = child_start[b]; ch < child_start[b + 1]; ++ch) {
        int o = ((ijk_child[3 * ch] & 1) << 2) | ((ijk_child[3 * ch + 1] & 1) << 1) | (ijk_child[3 * ch + 2] & 1);
        child_oct[8 * b + o] = ch;
    }
}
__global__ void k_iota(int64_t n, int* v) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) v[i] = (int)i;
}
// key = (tile, cell) or, with the quarter-turn symmetry (hq = n_C/2 > 0), (tile,
// representative cell: phi sector mod n_C/2)
__global__ void k_tile_keys(const int* __restrict__ seg_box, const int* __restrict__ seg_cell, int64_t n,
                            int64_t tile, int bits, int hq, int nsc, uint64_t* key) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int cell = seg_cell[i];
    if (hq > 0) {
        const int ip = cell / nsc;
        cell = (ip % hq) * nsc + (cell - ip * nsc);
    }
    key[i] = ((uint64_t)(seg_box[i] / tile) << bits) | (uint64_t)cell;
}
__global__ void k_run_start(const uint64_t* __restrict__ key, int64_t n, int* rs) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) rs[i] = (i == 0 || key[i] != key[i - 1]) ? (int)i : 0;
}
// run starts of a sorted key array, runs also cut every `cut` positions (bounded work per run)
__global__ void k_key_change(const int* __restrict__ key, int64_t n, int cut, int* flag) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) flag[i] = (i == 0 || key[i] != key[i - 1] || i % cut == 0) ? 1 : 0;
}
__global__ void k_chunk_flag(const int* __restrict__ rs, int64_t n, int ch, int* flag) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) flag[i] = ((i - rs[i]) % ch == 0) ? 1 : 0;
}
__global__ void k_chunk_emit(const int* __restrict__ flag, const int* __restrict__ incl, int64_t n, int* start) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && flag[i]) start[incl[i] - 1] = (int)i;
}
// Execution order of a level's TC chunks (L2 locality of the child coefficients):
// key = (tile, parent cell coarsened to the child grid, chunk index within its
// run, sub-cell), so the sibling cells that read the same child cells run their
// k-th chunks (the same boxes) at the same time.
__global__ void k_chunk_keys(const int* __restrict__ chunk_start, int64_t nch, const int* __restrict__ cell_seg,
                             const int* __restrict__ seg_box, const int* __restrict__ seg_cell,
                             const int* __restrict__ rsm, int64_t tile, int ch, int ns, int nC, int hq, int fs,
                             int fc, int bsub, int bk, int bcoarse, uint64_t* key, int* val) {
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= nch) return;
    const int s = chunk_start[c];
    const int seg = cell_seg[s];
    const int cell = seg_cell[seg];
    const int is = cell % ns, it = (cell / ns) % nC, ip = (cell / (ns * nC)) % (hq > 0 ? hq : 2 * nC);
    const int nsc = ns / fs, ncc = nC / fc;
    const uint64_t coarse = ((uint64_t)(ip / fc) * ncc + (it / fc)) * nsc + (is / fs);
    const uint64_t sub = ((uint64_t)(ip % fc) * fc + (it % fc)) * fs + (is % fs);
    const uint64_t k = (uint64_t)((s - rsm[s]) / ch);
    const uint64_t tl = (uint64_t)(seg_box[seg] / tile);
    key[c] = (((tl << bcoarse | coarse) << bk | k) << bsub) | sub;
    val[c] = (int)c;
}
struct MaxOp {
    __device__ __forceinline__ int operator()(int a, int b) const { return a > b ? a : b; }
};

// ---------------------------------------------------------------- stats
__global__ void k_stat_near(LevelParams L, unsigned long long* acc) {
    int64_t T = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (T >= L.nbox) return;
    int64_t nT = L.box_start[T + 1] - L.box_start[T], s = 0;
    for (int e = L.nbr_off[T]; e < L.nbr_off[T + 1]; ++e) {
        int B = L.nbr_idx[e];
        if (B < L.b0 || B >= L.b1) continue;
        s += L.box_start[B + 1] - L.box_start[B];
    }
    int64_t own = (T >= L.b0 && T < L.b1) ? nT : 0;  // self pairs excluded
    atomicAdd(acc, (unsigned long long)(nT * s - own));
}
__global__ void k_stat_cousin(LevelParams L, unsigned long long* acc) {
    int64_t T = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (T >= L.nbox) return;
    int64_t nT = L.box_start[T + 1] - L.box_start[T], c = 0;
    for (int e = L.cou_off[T]; e < L.cou_off[T + 1]; ++e) {
        int B = L.cou_idx[e];
        if (B >= L.b0 && B < L.b1) ++c;
    }
    atomicAdd(acc, (unsigned long long)(nT * c));
}
__global__ void k_stat_s2c(LevelParams L, int P, unsigned long long* acc) {
    int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= L.nseg) return;
    int B = L.seg_box[s];
    atomicAdd(acc, (unsigned long long)((int64_t)P * (L.box_start[B + 1] - L.box_start[B])));
}
__global__ void k_stat_up(LevelParams L, LevelParams LP, int P, unsigned long long* acc) {
    int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= LP.nseg) return;
    int Q = LP.seg_box[s];
    int64_t c = 0;
    for (int B = LP.child_start[Q]; B < LP.child_start[Q + 1]; ++B)
        if (B >= L.b0 && B < L.b1) ++c;
    atomicAdd(acc, (unsigned long long)(c * P));
}

// ------------------------------------------------------------ host helpers
// Temporary device buffers of the plan build: stream-ordered allocations from the
// device's default memory pool (kept cached while the build runs, trimmed at the
// end), so the many short-lived scratch arrays cost no cudaMalloc / cudaFree syncs.
struct Scratch {
    cudaStream_t s;
    cudaMemPool_t pool = nullptr;
    std::vector<void*> ptrs;
    explicit Scratch(cudaStream_t st) : s(st) {
        int dev = 0;
        IFGF_CUDA(cudaGetDevice(&dev));
        IFGF_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
        uint64_t thr = UINT64_MAX;
        IFGF_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    }
    template <class T>
    T* get(int64_t n) {
        if (n <= 0) n = 1;
        void* p = nullptr;
        IFGF_CUDA(cudaMallocAsync(&p, sizeof(T) * (size_t)n, s));
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    void release(void* p) {
        for (auto& q : ptrs)
            if (q == p) {
                cudaFreeAsync(q, s);
                q = nullptr;
            }
    }
    ~Scratch() {
        for (void* p : ptrs)
            if (p) cudaFreeAsync(p, s);
        cudaStreamSynchronize(s);
        if (pool) cudaMemPoolTrimTo(pool, 0);
    }
};

template <class T>
void inclusive_scan(Scratch& S, const T* in, T* out, int64_t n, cudaStream_t st) {
    size_t bytes = 0;
    IFGF_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, in, out, (int)n, st));
    void* tmp = S.get<char>((int64_t)bytes);
    IFGF_CUDA(cub::DeviceScan::InclusiveSum(tmp, bytes, in, out, (int)n, st));
    S.release(tmp);
}
template <class T>
void exclusive_scan(Scratch& S, const T* in, T* out, int64_t n, cudaStream_t st) {
    size_t bytes = 0;
    IFGF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, (int)n, st));
    void* tmp = S.get<char>((int64_t)bytes);
    IFGF_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, (int)n, st));
    S.release(tmp);
}

template <class T>
T d2h_one(const T* p, cudaStream_t st) {
    T v;
    IFGF_CUDA(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, st));
    IFGF_CUDA(cudaStreamSynchronize(st));
    return v;
}

// CSR build from a count kernel: off = exclusive scan of counts (+ total).
// Multi-rank: a rank only evaluates its own source boxes, so its target-major
// kernels get neighbour / cousin lists filtered to owned boxes and work items only
// for target boxes with at least one owned entry.
__global__ void k_count_owned(const int* __restrict__ off, const int* __restrict__ idx, int64_t nb, int64_t b0,
                              int64_t b1, int* cnt) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= nb) return;
    int c = 0;
    for (int e = off[b]; e < off[b + 1]; ++e) c += (idx[e] >= b0 && idx[e] < b1);
    cnt[b] = c;
}
__global__ void k_emit_owned(const int* __restrict__ off, const int* __restrict__ idx, int64_t nb, int64_t b0,
                             int64_t b1, const int* __restrict__ off2, int* idx2) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= nb) return;
    int o = off2[b];
    for (int e = off[b]; e < off[b + 1]; ++e)
        if (idx[e] >= b0 && idx[e] < b1) idx2[o++] = idx[e];
}
__global__ void k_witem_count_masked(const int* __restrict__ start, int64_t nb, const int* __restrict__ own,
                                     int* cnt) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= nb) return;
    cnt[b] = own[b] > 0 ? (start[b + 1] - start[b] + 31) / 32 : 0;
}
__global__ void k_witem_fill_masked(const int* __restrict__ start, int64_t nb, const int* __restrict__ own,
                                    const int* __restrict__ off, int2* items) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= nb || own[b] == 0) return;
    int o = off[b];
    for (int q = start[b]; q < start[b + 1]; q += 32) items[o++] = make_int2((int)b, q);
}

int* csr_offsets(ifgf_plan_s* p, Scratch& S, const int* cnt, int64_t n, cudaStream_t st, int64_t* total) {
    int* off = dev_alloc<int>(p, n + 1);
    int* incl = S.get<int>(n);
    inclusive_scan(S, cnt, incl, n, st);
    IFGF_CUDA(cudaMemsetAsync(off, 0, sizeof(int), st));
    IFGF_CUDA(cudaMemcpyAsync(off + 1, incl, sizeof(int) * n, cudaMemcpyDeviceToDevice, st));
    *total = d2h_one(off + n, st);
    S.release(incl);
    return off;
}

template <class T>
T* upload(ifgf_plan_s* p, const std::vector<T>& v, cudaStream_t st) {
    T* d = dev_alloc<T>(p, (int64_t)v.size());
    IFGF_CUDA(cudaMemcpyAsync(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, st));
    IFGF_CUDA(cudaStreamSynchronize(st));
    return d;
}

std::vector<double> cheb_nodes(int n) {
    std::vector<double> t(n);
    for (int k = 0; k < n; ++k) t[k] = std::cos((2.0 * k + 1.0) * kPi / (2.0 * n));
    return t;
}

// Fit matrix M[i][k] = ((2 - delta_i0)/n) T_i(t_k)  (reading R1).
std::vector<double> cheb_fit_matrix(int n) {
    std::vector<double> t = cheb_nodes(n), M(n * n);
    for (int k = 0; k < n; ++k) {
        double T0 = 1.0, T1 = t[k];
        for (int i = 0; i < n; ++i) {
            double Ti;
            if (i == 0) Ti = T0;
            else if (i == 1) Ti = T1;
            else {
                Ti = 2.0 * t[k] * T1 - T0;
                T0 = T1;
                T1 = Ti;
            }
            M[i * n + k] = (i == 0 ? 1.0 : 2.0) / n * Ti;
        }
    }
    return M;
}

}  // namespace

void build_plan(ifgf_plan_s* p, const double* pts, const ifgf_opts& o) {
    auto t_start = std::chrono::steady_clock::now();
    const int64_t n = p->n;
    const int D = p->D, Ps = p->Ps, Pa = p->Pa, P = p->P;
    cudaStream_t st;
    IFGF_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};
    Scratch S(st);
    const bool verbose = std::getenv("IFGF_PLAN_VERBOSE") != nullptr;
    auto t_mark = std::chrono::steady_clock::now();
    auto step_time = [&](const char* what) {  // plan-step wall times (IFGF_PLAN_VERBOSE)
        if (!verbose) return;
        cudaStreamSynchronize(st);
        const auto t = std::chrono::steady_clock::now();
        fprintf(stderr, "[ifgf] plan step %-28s %8.1f ms\n", what,
                std::chrono::duration<double, std::milli>(t - t_mark).count());
        t_mark = t;
    };

    // The plan works on its own non-blocking stream: finish every piece of work
    // already enqueued on the device (e.g. the caller's copy into `points`) first.
    IFGF_CUDA(cudaDeviceSynchronize());

    // 1. validation + bounding box
    {
        int nb = 148 * 4;
        double* part = S.get<double>(6 * nb);
        int* bad = S.get<int>(1);
        IFGF_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
        k_minmax<<<nb, TPB, 0, st>>>(pts, n, part, bad);
        IFGF_CUDA(cudaGetLastError());
        std::vector<double> h(6 * nb);
        IFGF_CUDA(cudaMemcpyAsync(h.data(), part, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st));
        int hbad = d2h_one(bad, st);
        if (hbad) throw Error{IFGF_EINVAL, "non-finite point coordinates"};
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int b = 0; b < nb; ++b)
            for (int a = 0; a < 3; ++a) {
                lo[a] = std::min(lo[a], h[6 * b + a]);
                hi[a] = std::max(hi[a], h[6 * b + 3 + a]);
            }
        // Root box (reading R9)
        if (o.has_root) {
            for (int a = 0; a < 3; ++a) p->root_c[a] = o.root_center[a];
            p->H1 = o.root_side;
        } else {
            double ext = 0.0;
            for (int a = 0; a < 3; ++a) {
                p->root_c[a] = (lo[a] + hi[a]) / 2.0;
                ext = std::max(ext, hi[a] - lo[a]);
            }
            if (ext == 0.0) {
                if (n > 1) throw Error{IFGF_EDOMAIN, "zero-extent point cloud"};
                ext = 1.0;
            }
            p->H1 = (1.0 + std::ldexp(1.0, -20)) * ext;
        }
        for (int a = 0; a < 3; ++a) p->x0[a] = p->root_c[a] - p->H1 / 2.0;
        // A caller-supplied root box must contain Gamma_N (eq. deffirstbox);
        // points outside it would be clamped into boundary leaves and the cousin
        // separation the interpolation relies on would not hold.
        if (o.has_root)
            for (int a = 0; a < 3; ++a)
                if (!(lo[a] >= p->x0[a] && hi[a] <= p->x0[a] + p->H1))
                    throw Error{IFGF_EDOMAIN, "the root box does not contain every point"};
    }

    step_time("1 validation+bbox");
    // 2. levels, cone grids (readings R5, R6, R8) and tables
    p->lev.assign(D + 1, LevelHost());
    for (int d = 1; d <= D; ++d) {
        LevelParams& L = p->lev[d].p;
        L.d = d;
        L.H = std::ldexp(p->H1, -(d - 1));
        for (int a = 0; a < 3; ++a) L.x0[a] = p->x0[a];
    }
    p->lev[D].p.ns = o.leaf_ns > 0 ? o.leaf_ns : 1;
    p->lev[D].p.nC = o.leaf_nc > 0 ? o.leaf_nc : 2;
    for (int d = D; d >= 2; --d) {
        bool refine = p->k * p->lev[d - 1].p.H > 1.0;
        p->lev[d - 1].p.ns = refine ? 2 * p->lev[d].p.ns : p->lev[d].p.ns;
        p->lev[d - 1].p.nC = refine ? 2 * p->lev[d].p.nC : p->lev[d].p.nC;
    }
    const std::vector<double> ts = cheb_nodes(Ps), ta = cheb_nodes(Pa);
    for (int d = 1; d <= D; ++d) {
        LevelHost& LH = p->lev[d];
        LevelParams& L = LH.p;
        const double eta = std::sqrt(3.0) / 3.0;
        L.h = std::sqrt(3.0) / 2.0 * L.H;
        L.ds = eta / L.ns;
        L.dth = kPi / L.nC;
        L.cls_exact = p->cls_exact;
        L.ids = 1.0 / L.ds;  // reciprocals: first guesses and local coordinates only
        L.idth = 1.0 / L.dth;
        L.ncell = 2LL * L.ns * (int64_t)L.nC * L.nC;
        L.W = (L.ncell + 63) / 64;
        if (d < 3) continue;  // no relevant segments at levels 1-2
        if (L.ncell > (int64_t)1 << 31) throw Error{IFGF_ENOMEM, "cone grid too fine for the cell index"};
        std::vector<double> ctb(L.nC + 1), cph(2 * L.nC + 1), sph(2 * L.nC + 1);
        for (int kk = 0; kk <= L.nC; ++kk) ctb[kk] = std::cos((double)kk * kPi / (double)L.nC);
        // phi tables: n_C even -> exact quarter-turn symmetry (reading R18; the K7
        // tensor-core kernels share one geometry between the four rotated cells);
        // else exact half-turn symmetry
        const int hq = L.nC / 2;
        auto turns = [](double c, double sn, int q, double* co, double* so) {
            switch (q & 3) {
                case 0: *co = c; *so = sn; break;
                case 1: *co = -sn; *so = c; break;
                case 2: *co = -c; *so = -sn; break;
                default: *co = sn; *so = -c; break;
            }
        };
        if (L.nC % 2 == 0) {
            for (int j = 0; j <= 2 * L.nC; ++j) {
                const double a = (double)(j % hq) * kPi / (double)L.nC;
                turns(std::cos(a), std::sin(a), j / hq, &cph[j], &sph[j]);
            }
        } else {
            for (int j = 0; j < L.nC; ++j) {
                double a = (double)j * kPi / (double)L.nC;
                cph[j] = std::cos(a);
                sph[j] = std::sin(a);
                cph[j + L.nC] = -cph[j];
                sph[j + L.nC] = -sph[j];
            }
            cph[2 * L.nC] = cph[0];
            sph[2 * L.nC] = sph[0];
        }
        std::vector<double> rt(L.ns * Ps), stt(L.nC * Pa), ctt(L.nC * Pa), spt(2 * L.nC * Pa), cpt(2 * L.nC * Pa);
        for (int is = 0; is < L.ns; ++is)
            for (int ks = 0; ks < Ps; ++ks) {
                double s = ((double)is + (1.0 + ts[ks]) / 2.0) * L.ds;
                rt[is * Ps + ks] = L.h / s;
            }
        for (int it = 0; it < L.nC; ++it)
            for (int kt = 0; kt < Pa; ++kt) {
                double th = ((double)it + (1.0 + ta[kt]) / 2.0) * L.dth;
                stt[it * Pa + kt] = std::sin(th);
                ctt[it * Pa + kt] = std::cos(th);
            }
        for (int ip = 0; ip < 2 * L.nC; ++ip)
            for (int kp = 0; kp < Pa; ++kp) {
                if (L.nC % 2 == 0) {
                    const double ph = ((double)(ip % hq) + (1.0 + ta[kp]) / 2.0) * L.dth;
                    turns(std::cos(ph), std::sin(ph), ip / hq, &cpt[ip * Pa + kp], &spt[ip * Pa + kp]);
                } else {
                    double ph = ((double)ip + (1.0 + ta[kp]) / 2.0) * L.dth;
                    spt[ip * Pa + kp] = std::sin(ph);
                    cpt[ip * Pa + kp] = std::cos(ph);
                }
            }
        L.cos_tb = LH.cos_tb = upload(p, ctb, st);
        L.cphi = LH.cphi = upload(p, cph, st);
        L.sphi = LH.sphi = upload(p, sph, st);
        L.rtab = LH.rtab = upload(p, rt, st);
        L.st_tab = LH.st_tab = upload(p, stt, st);
        L.ct_tab = LH.ct_tab = upload(p, ctt, st);
        L.sp_tab = LH.sp_tab = upload(p, spt, st);
        L.cp_tab = LH.cp_tab = upload(p, cpt, st);
    }
    p->cheb_Ms = upload(p, cheb_fit_matrix(Ps), st);
    p->cheb_Ma = upload(p, cheb_fit_matrix(Pa), st);

    step_time("2 grids+tables");
    // 3. Morton keys + radix sort (relevant boxes via integer quotients)
    uint64_t* keys_sorted = S.get<uint64_t>(n);
    {
        uint64_t* keys = S.get<uint64_t>(n);
        int* idx = S.get<int>(n);
        p->perm = dev_alloc<int>(p, n);
        k_keys<<<nblocks(n), TPB, 0, st>>>(pts, n, p->x0[0], p->x0[1], p->x0[2], p->lev[D].p.H, 1 << (D - 1), keys,
                                           idx);
        IFGF_CUDA(cudaGetLastError());
        size_t bytes = 0;
        int bits = 3 * (D - 1);
        if (bits < 1) bits = 1;
        IFGF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, keys_sorted, idx, p->perm, (int)n, 0, bits, st));
        void* tmp = S.get<char>((int64_t)bytes);
        IFGF_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, keys, keys_sorted, idx, p->perm, (int)n, 0, bits, st));
        IFGF_CUDA(cudaStreamSynchronize(st));
        S.release(tmp);
        S.release(keys);
        S.release(idx);
    }
    p->px = dev_alloc<double>(p, n);
    p->py = dev_alloc<double>(p, n);
    p->pz = dev_alloc<double>(p, n);
    k_gather_points<<<nblocks(n), TPB, 0, st>>>(pts, p->perm, n, p->px, p->py, p->pz);
    IFGF_CUDA(cudaGetLastError());

    step_time("3 morton sort");
    // 4. boxes per level (leaf from points, coarser from finer)
    std::vector<uint64_t*> bkey(D + 1, nullptr);
    {
        int* flag = S.get<int>(n);
        int* incl = S.get<int>(n);
        k_flag_runs<<<nblocks(n), TPB, 0, st>>>(keys_sorted, n, 0, flag);
        inclusive_scan(S, flag, incl, n, st);
        int64_t nbD = d2h_one(incl + n - 1, st);
        LevelHost& LD = p->lev[D];
        LD.p.nbox = nbD;
        LD.box_start = dev_alloc<int>(p, nbD + 1);
        bkey[D] = S.get<uint64_t>(nbD);
        k_leaf_boxes<<<nblocks(n), TPB, 0, st>>>(keys_sorted, flag, incl, n, LD.box_start, bkey[D]);
        int nn = (int)n;
        IFGF_CUDA(cudaMemcpyAsync(LD.box_start + nbD, &nn, sizeof(int), cudaMemcpyHostToDevice, st));
        IFGF_CUDA(cudaStreamSynchronize(st));
        S.release(flag);
        S.release(incl);
        S.release(keys_sorted);
        for (int d = D; d >= 2; --d) {
            LevelHost& L = p->lev[d];
            LevelHost& LP = p->lev[d - 1];
            int64_t nb = L.p.nbox;
            int* f = S.get<int>(nb);
            int* inc = S.get<int>(nb);
            k_flag_runs<<<nblocks(nb), TPB, 0, st>>>(bkey[d], nb, 3, f);
            inclusive_scan(S, f, inc, nb, st);
            int64_t nbp = d2h_one(inc + nb - 1, st);
            LP.p.nbox = nbp;
            L.box_parent = dev_alloc<int>(p, nb);
            LP.box_start = dev_alloc<int>(p, nbp + 1);
            LP.child_start = dev_alloc<int>(p, nbp + 1);
            bkey[d - 1] = S.get<uint64_t>(nbp);
            k_parent_boxes<<<nblocks(nb), TPB, 0, st>>>(bkey[d], L.box_start, f, inc, nb, L.box_parent, LP.box_start,
                                                        bkey[d - 1], LP.child_start);
            int nn2 = (int)n, nb2 = (int)nb;
            IFGF_CUDA(cudaMemcpyAsync(LP.box_start + nbp, &nn2, sizeof(int), cudaMemcpyHostToDevice, st));
            IFGF_CUDA(cudaMemcpyAsync(LP.child_start + nbp, &nb2, sizeof(int), cudaMemcpyHostToDevice, st));
            IFGF_CUDA(cudaStreamSynchronize(st));
            S.release(f);
            S.release(inc);
        }
        for (int d = 1; d <= D; ++d) {
            LevelHost& L = p->lev[d];
            L.box_ijk = dev_alloc<int>(p, 3 * L.p.nbox);
            k_box_ijk<<<nblocks(L.p.nbox), TPB, 0, st>>>(bkey[d], L.p.nbox, L.box_ijk);
            L.box_c = dev_alloc<double>(p, 4 * L.p.nbox);
            k_box_c<<<nblocks(L.p.nbox), TPB, 0, st>>>(L.box_ijk, L.p.nbox, L.p, L.box_c);
            IFGF_CUDA(cudaGetLastError());
        }
    }
    // pairwise-different points
    {
        int* bad = S.get<int>(1);
        IFGF_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
        k_coincident<<<(int)p->lev[D].p.nbox, 64, 0, st>>>(p->px, p->py, p->pz, p->lev[D].box_start,
                                                            p->lev[D].p.nbox, bad);
        if (d2h_one(bad, st)) throw Error{IFGF_EDOMAIN, "coincident points (the paper requires pairwise-different points)"};
    }

    step_time("4 box lists");
    // 5. neighbours and cousins
    for (int d = 1; d <= D; ++d) {
        LevelHost& L = p->lev[d];
        int64_t nb = L.p.nbox;
        int* cnt = S.get<int>(nb);
        k_neighbours<<<nblocks(nb), TPB, 0, st>>>(bkey[d], L.box_ijk, nb, 1 << (d - 1), 0, cnt, nullptr, nullptr);
        L.nbr_off = csr_offsets(p, S, cnt, nb, st, &L.nnbr);
        L.nbr_idx = dev_alloc<int>(p, L.nnbr);
        k_neighbours<<<nblocks(nb), TPB, 0, st>>>(bkey[d], L.box_ijk, nb, 1 << (d - 1), 1, nullptr, L.nbr_off,
                                                  L.nbr_idx);
        IFGF_CUDA(cudaGetLastError());
        if (d >= 3) {
            LevelHost& LP = p->lev[d - 1];
            k_cousins<<<nblocks(nb), TPB, 0, st>>>(L.box_ijk, L.box_parent, nb, LP.nbr_off, LP.nbr_idx, LP.child_start,
                                                   0, cnt, nullptr, nullptr);
            L.cou_off = csr_offsets(p, S, cnt, nb, st, &L.ncou);
            L.cou_idx = dev_alloc<int>(p, L.ncou);
            k_cousins<<<nblocks(nb), TPB, 0, st>>>(L.box_ijk, L.box_parent, nb, LP.nbr_off, LP.nbr_idx, LP.child_start,
                                                   1, nullptr, L.cou_off, L.cou_idx);
            IFGF_CUDA(cudaGetLastError());
        }
        // warp work items over all boxes of the level (targets)
        if (d >= 3 || d == D) {
            k_witem_count<<<nblocks(nb), TPB, 0, st>>>(L.box_start, nb, cnt);
            int64_t ni = 0;
            int* off = csr_offsets(p, S, cnt, nb, st, &ni);
            L.witems = dev_alloc<int2>(p, ni);
            L.p.nwitems = ni;
            k_witem_fill<<<nblocks(nb), TPB, 0, st>>>(L.box_start, nb, off, L.witems);
            IFGF_CUDA(cudaGetLastError());
        }
        S.release(cnt);
    }
    for (int d = 1; d <= D; ++d) S.release(bkey[d]);

    step_time("5 neighbours+cousins");
    // 6. source partition: owned leaf range -> owned box range per level
    {
        LevelHost& LD = p->lev[D];
        int64_t nleaf = LD.p.nbox;
        int64_t L0 = 0, L1 = nleaf;
        p->stats.partition_weight_total = p->stats.partition_weight_owned = 0.0;
        if (p->nranks > 1) {
            // Work weight per leaf L, in ps on one B200:
            //   w(L) = c3 near(L) + c4 s2c(L) + n_L sum_{A ancestor of L, d >= 3} (c6 + rho c7) cou(A) / n_A
            // with the plan's unit counts: near(L) = near-field pairs with L as source,
            // s2c(L) = n_L |cells_D| P (source-to-cone pairs; every leaf cell is relevant
            // at the default grid), cou(A) = cousin evaluations with A as source; the
            // upward evaluations of A (known only after the relevance pass) are proxied
            // by rho cou(A), rho = 2.7 = sum upward / sum cousin evaluations at cfg4; A's
            // work is apportioned to its leaves by their points.  c3 = 6.0, c4 = 4.7,
            // c6 = 41, c7 = 32 ps per unit: the measured cfg4 kernel time per unit
            // (r01m: 48 ms / 8.0e9, 71 ms / 1.5e10, 384 ms / 9.3e9, 805 ms / 2.5e10).
            const double c3 = 6.0, c4 = 4.7, c6 = 41.0, c7 = 32.0, rho = 2.7;
            std::vector<std::vector<int>> start(D + 1), parent(D + 1);
            std::vector<std::vector<double>> cou(D + 1);
            std::vector<double> near(nleaf);
            for (int d = 3; d <= D; ++d) {
                LevelHost& L = p->lev[d];
                const int64_t nb = L.p.nbox;
                double* dnear = d == D ? S.get<double>(nb) : nullptr;
                double* dcou = S.get<double>(nb);
                k_box_units<<<nblocks(nb), TPB, 0, st>>>(L.box_start, L.nbr_off, L.nbr_idx, L.cou_off, L.cou_idx, nb,
                                                         dnear, dcou);
                IFGF_CUDA(cudaGetLastError());
                start[d].resize(nb + 1);
                cou[d].resize(nb);
                parent[d].resize(nb);
                IFGF_CUDA(cudaMemcpyAsync(start[d].data(), L.box_start, sizeof(int) * (nb + 1), cudaMemcpyDeviceToHost, st));
                IFGF_CUDA(cudaMemcpyAsync(cou[d].data(), dcou, sizeof(double) * nb, cudaMemcpyDeviceToHost, st));
                IFGF_CUDA(cudaMemcpyAsync(parent[d].data(), L.box_parent, sizeof(int) * nb, cudaMemcpyDeviceToHost, st));
                if (dnear)
                    IFGF_CUDA(cudaMemcpyAsync(near.data(), dnear, sizeof(double) * nb, cudaMemcpyDeviceToHost, st));
                IFGF_CUDA(cudaStreamSynchronize(st));
                if (dnear) S.release(dnear);
                S.release(dcou);
            }
            std::vector<double> w(nleaf);
            const double cells_D = (double)LD.p.ncell;
            for (int64_t b = 0; b < nleaf; ++b) {
                const double m = start[D][b + 1] - start[D][b];
                double anc = 0.0;
                for (int64_t a = b, d = D; d >= 3; --d) {
                    const double na = start[d][a + 1] - start[d][a];
                    anc += (c6 + rho * c7) * cou[d][a] / std::max(1.0, na);
                    a = parent[d][a];
                }
                w[b] = c3 * near[b] + c4 * cells_D * P * m + m * anc;
            }
            std::vector<int64_t> bounds(p->nranks + 1);
            ifgf_status ps = ifgf_partition(w.data(), nleaf, p->nranks, bounds.data());
            if (ps != IFGF_OK) throw Error{ps, "partition failed"};
            L0 = bounds[p->rank];
            L1 = bounds[p->rank + 1];
            for (int64_t b = 0; b < nleaf; ++b) {
                p->stats.partition_weight_total += w[b];
                if (b >= L0 && b < L1) p->stats.partition_weight_owned += w[b];
            }
        }
        // owned range as leaf Morton keys (half-open; the end is the first leaf of the next rank)
        auto leaf_key = [&](int64_t b) -> uint64_t {
            int ijk[3];
            IFGF_CUDA(cudaMemcpy(ijk, LD.box_ijk + 3 * b, sizeof(ijk), cudaMemcpyDeviceToHost));
            uint64_t r = 0;
            for (int bit = 0; bit < 21; ++bit)
                r |= ((uint64_t)((ijk[0] >> bit) & 1) << (3 * bit + 2)) | ((uint64_t)((ijk[1] >> bit) & 1) << (3 * bit + 1)) |
                     ((uint64_t)((ijk[2] >> bit) & 1) << (3 * bit));
            return r;
        };
        p->stats.owned_morton_begin = L0 == 0 ? 0 : (L0 < nleaf ? leaf_key(L0) : ~(uint64_t)0);
        p->stats.owned_morton_end = L1 >= nleaf ? ~(uint64_t)0 : leaf_key(L1);
        p->stats.owned_leaf_begin = L0;
        p->stats.owned_leaf_end = L1;
        int64_t a = L0, b = L1 - 1;  // inclusive leaf range (may be empty)
        for (int d = D; d >= 1; --d) {
            LevelHost& L = p->lev[d];
            if (L1 <= L0) {
                L.p.b0 = L.p.b1 = 0;
                continue;
            }
            L.p.b0 = a;
            L.p.b1 = b + 1;
            if (d > 1) {
                a = d2h_one(L.box_parent + a, st);
                b = d2h_one(L.box_parent + b, st);
            }
        }
    }

    // publish pointers into LevelParams
    for (int d = 1; d <= D; ++d) {
        LevelHost& L = p->lev[d];
        L.p.box_ijk = L.box_ijk;
        L.p.box_c = L.box_c;
        L.p.box_start = L.box_start;
        L.p.box_parent = L.box_parent;
        L.p.child_start = L.child_start;
        L.p.nbr_off = L.nbr_off;
        L.p.nbr_idx = L.nbr_idx;
        L.p.cou_off = L.cou_off;
        L.p.cou_idx = L.cou_idx;
        L.p.witems = L.witems;
    }

    step_time("6 partition+witems");
    // 7. relevant cone segments, single sweep d = 3..D
    int* bad = S.get<int>(1);
    IFGF_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
    for (int d = 3; d <= D; ++d) {
        LevelHost& L = p->lev[d];
        int64_t nown = L.p.b1 - L.p.b0;
        int64_t nw = nown * L.p.W;
        L.bitmap = dev_alloc<unsigned long long>(p, nw);
        L.rank = dev_alloc<unsigned>(p, nw + 1);
        L.p.bitmap = L.bitmap;
        L.p.rank = L.rank;
        IFGF_CUDA(cudaMemsetAsync(L.bitmap, 0, sizeof(unsigned long long) * (size_t)std::max<int64_t>(nw, 1), st));
        if (nown > 0) {
            k_flag_cousin_points<<<nblocks(L.p.nwitems * 32), TPB, 0, st>>>(L.p, p->px, p->py, p->pz, L.bitmap, bad);
            IFGF_CUDA(cudaGetLastError());
            if (d >= 4 && p->lev[d - 1].p.nseg > 0) {
                LevelHost& LH = p->lev[d - 1];
                LevelParams& LP = LH.p;
                if (std::getenv("IFGF_FLAG_PER_NODE")) {  // A/B: one thread per (segment, node)
                    k_flag_parent_nodes<<<nblocks(LP.nseg * P), TPB, 0, st>>>(L.p, LP, Ps, Pa, L.bitmap, bad);
                } else {
                    // parent segments sorted by cell, runs of equal cells, then a warp per run
                    if (!LH.child_oct) {
                        LH.child_oct = dev_alloc<int>(p, 8 * LP.nbox);
                        k_child_oct<<<nblocks(LP.nbox), TPB, 0, st>>>(LH.child_start, L.box_ijk, LP.nbox, LH.child_oct);
                        LP.child_oct = LH.child_oct;
                    }
                    const int64_t nsp = LP.nseg;
                    int bits = 1;
                    while (bits < 31 && ((int64_t)1 << bits) < LP.ncell) ++bits;
                    int* idx_in = S.get<int>(nsp);
                    int* idx_out = S.get<int>(nsp);
                    int* key_in = S.get<int>(nsp);
                    int* key_out = S.get<int>(nsp);
                    k_iota<<<nblocks(nsp), TPB, 0, st>>>(nsp, idx_in);
                    IFGF_CUDA(cudaMemcpyAsync(key_in, LH.seg_cell, sizeof(int) * nsp, cudaMemcpyDeviceToDevice, st));
                    size_t bytes = 0;
                    IFGF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key_in, key_out, idx_in, idx_out,
                                                              (int)nsp, 0, bits, st));
                    void* tmp = S.get<char>((int64_t)bytes);
                    IFGF_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, key_in, key_out, idx_in, idx_out, (int)nsp,
                                                              0, bits, st));
                    S.release(tmp);
                    int* flag = S.get<int>(nsp);
                    int* incl = S.get<int>(nsp);
                    k_key_change<<<nblocks(nsp), TPB, 0, st>>>(key_out, nsp, 32, flag);
                    inclusive_scan(S, flag, incl, nsp, st);
                    const int64_t nrun = d2h_one(incl + nsp - 1, st);
                    int* rstart = S.get<int>(nrun);
                    k_chunk_emit<<<nblocks(nsp), TPB, 0, st>>>(flag, incl, nsp, rstart);
                    k_flag_parent_runs<<<nblocks(nrun * 32), TPB, 0, st>>>(L.p, LP, Ps, Pa, idx_out, rstart, nrun,
                                                                          L.bitmap, bad);
                    IFGF_CUDA(cudaStreamSynchronize(st));
                    S.release(rstart);
                    S.release(incl);
                    S.release(flag);
                    S.release(key_out);
                    S.release(key_in);
                    S.release(idx_out);
                    S.release(idx_in);
                }
                IFGF_CUDA(cudaGetLastError());
            }
        }
        // compaction: global exclusive prefix of popcounts -> rank; emit (box, cell) list
        int64_t nseg = 0;
        if (nw > 0) {
            unsigned* pc = S.get<unsigned>(nw + 1);
            k_popc<<<nblocks(nw), TPB, 0, st>>>(L.bitmap, nw, pc);
            IFGF_CUDA(cudaMemsetAsync(pc + nw, 0, sizeof(unsigned), st));
            exclusive_scan(S, pc, L.rank, nw + 1, st);
            nseg = d2h_one(L.rank + nw, st);
            S.release(pc);
        }
        if (nseg >= ((int64_t)1 << 31)) throw Error{IFGF_ENOMEM, "too many relevant segments in one level"};
        L.p.nseg = nseg;
        L.seg_box = dev_alloc<int>(p, nseg);
        L.seg_cell = dev_alloc<int>(p, nseg);
        L.p.seg_box = L.seg_box;
        L.p.seg_cell = L.seg_cell;
        if (nseg > 0) {
            k_emit_segments<<<nblocks(nw), TPB, 0, st>>>(L.bitmap, L.rank, nw, L.p.W, L.p.b0, L.seg_box, L.seg_cell);
            IFGF_CUDA(cudaGetLastError());
        }
        IFGF_CUDA(cudaStreamSynchronize(st));
    }
    if (d2h_one(bad, st)) throw Error{IFGF_EINTERNAL, "classification produced a cell outside the grid"};

    step_time("7 relevance");
    // 7b. K7 support: children by octant; parent segments grouped by cone cell
    for (int d = 1; d < D; ++d) {
        LevelHost& L = p->lev[d];
        if (!L.child_oct) {
            L.child_oct = dev_alloc<int>(p, 8 * L.p.nbox);
            k_child_oct<<<nblocks(L.p.nbox), TPB, 0, st>>>(L.child_start, p->lev[d + 1].box_ijk, L.p.nbox,
                                                            L.child_oct);
            IFGF_CUDA(cudaGetLastError());
        }
        L.p.child_oct = L.child_oct;
        const int64_t ns = L.p.nseg;
        if (d < 3 || ns == 0) continue;
        int* vals_in = S.get<int>(ns);
        uint64_t* keys_in = S.get<uint64_t>(ns);
        uint64_t* keys_out = S.get<uint64_t>(ns);
        L.cell_seg = dev_alloc<int>(p, ns);
        k_iota<<<nblocks(ns), TPB, 0, st>>>(ns, vals_in);
        int bits = 1;
        while (bits < 31 && ((int64_t)1 << bits) < L.p.ncell) ++bits;
        // Tiles: consecutive parent boxes whose children's coefficients total
        // tile_bytes; segments are grouped by cell only inside a tile.  Large tiles
        // give long cell runs (geometry reuse); where runs are very long (fine
        // levels) the tile shrinks so that a tile's child data stays L2-resident
        // while its cells' chunks run (target ~256 segments per run).
        const double child_bytes_per_box =
            (double)p->lev[d + 1].p.nseg * P * 16.0 / (double)std::max<int64_t>(1, L.p.b1 - L.p.b0);
        double tile_bytes = 4096.0e6;  // child bytes per tile (env IFGF_TILE_MB: fixed)
        const char* tile_env = std::getenv("IFGF_TILE_MB");
        // adaptive tiles: aim at ~tile_target segments per run where runs are very long
        const double tile_target = std::getenv("IFGF_TILE_TARGET") ? std::atof(std::getenv("IFGF_TILE_TARGET")) : 256.0;
        const double tile_min = std::getenv("IFGF_TILE_MIN_MB") ? std::atof(std::getenv("IFGF_TILE_MIN_MB")) * 1e6 : 32.0e6;
        if (tile_env) tile_bytes = std::atof(tile_env) * 1.0e6;
        int* rs = S.get<int>(ns);
        int* rsm = S.get<int>(ns);
        int* incl = S.get<int>(ns);
        int* flag = rs;  // reused after the run-start max-scan
        // Quarter-turn symmetry (reading R18): with n_C even on both levels, the four
        // parent cells related by quarter turns about z share one child-relative
        // geometry, so the tensor-core kernels group segments by orbit (4x longer runs).
        const LevelParams& LCh = p->lev[d + 1].p;
        const bool sym_ok = !p->no_symmetry && L.p.nC % 2 == 0 && LCh.nC % 2 == 0 && LCh.ncell < ((int64_t)1 << 30);
        int sym = sym_ok ? 1 : 0;
        auto group = [&](double tb) -> int64_t {  // sort by (tile, cell, segment); number of runs
            const int64_t tile = (int64_t)std::max(1.0, tb / std::max(1.0, child_bytes_per_box));
            int tbits = 1;
            while (tbits < 32 && ((int64_t)1 << tbits) <= L.p.nbox / tile + 1) ++tbits;
            k_tile_keys<<<nblocks(ns), TPB, 0, st>>>(L.seg_box, L.seg_cell, ns, tile, bits, sym ? L.p.nC / 2 : 0,
                                                     L.p.ns * L.p.nC, keys_in);
            size_t bytes = 0;
            IFGF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys_in, keys_out, vals_in, L.cell_seg, (int)ns,
                                                      0, bits + tbits, st));
            void* tmp = S.get<char>((int64_t)bytes);
            IFGF_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, keys_in, keys_out, vals_in, L.cell_seg, (int)ns, 0,
                                                      bits + tbits, st));
            S.release(tmp);
            k_run_start<<<nblocks(ns), TPB, 0, st>>>(keys_out, ns, rs);
            bytes = 0;
            IFGF_CUDA(cub::DeviceScan::InclusiveScan(nullptr, bytes, rs, rsm, MaxOp(), (int)ns, st));
            tmp = S.get<char>((int64_t)bytes);
            IFGF_CUDA(cub::DeviceScan::InclusiveScan(tmp, bytes, rs, rsm, MaxOp(), (int)ns, st));
            S.release(tmp);
            k_chunk_flag<<<nblocks(ns), TPB, 0, st>>>(rsm, ns, 0x7fffffff, flag);
            inclusive_scan(S, flag, incl, ns, st);
            return d2h_one(incl + ns - 1, st);
        };
        // K7 kernel by mean segments per cell (or orbit) run (measured on B200, DESIGN.md
        // §7): >= 24 -> FP64 tensor-core GEMM (96-chunks, basis in shared memory);
        // 10-24 -> register-basis tensor-core GEMM (32-chunks, 2 blocks/SM) for (3, 5),
        // else the cell-grouped staged DFMA kernel; < 10 -> per-evaluation geometry
        // (cfg4 parent level 4, 6.5 segments per orbit run: TC2 228 ms, pe 168 ms)
        auto choose = [&](double pr) {
            int kn = pr >= 24.0 ? 1 : (pr >= 10.0 ? ((Ps == 3 && Pa == 5) ? 3 : 0) : 2);
            if (p->legacy_upward == 1 || p->legacy_upward == 7) kn = 2;  // per-evaluation (1: per-lane loads)
            if (p->legacy_upward == 3) kn = 0;                           // staged DFMA everywhere
            if (p->legacy_upward == 5) kn = 1;                           // force the tensor-core kernel
            if (p->legacy_upward == 8) kn = 3;                           // force the tensor-core kernel v2
            if (P > 80 && kn == 1) kn = 0;  // TC kernel shared memory is sized for P <= 80 ((P_s, P_ang) = (3, 5))
            if (kn == 3 && !(Ps == 3 && Pa == 5)) kn = 1;  // TC v2 k-permutation is specific to (3, 5)
            // orders without a compiled specialisation run the generic per-evaluation kernel
            if (!((Ps == 3 && Pa == 5) || (Ps == 5 && Pa == 5))) kn = 2;  // incl. (5, 7): specialised pe
            return kn;
        };
        int64_t nrun = 0;
        double per_run = 0.0;
        auto regroup = [&]() {
            nrun = group(tile_bytes);
            per_run = (double)ns / (double)std::max<int64_t>(1, nrun);
            if (!tile_env && per_run > 4.0 * tile_target) {
                tile_bytes = std::max(tile_min, tile_bytes * tile_target / per_run);
                nrun = group(tile_bytes);
                per_run = (double)ns / (double)std::max<int64_t>(1, nrun);
            }
        };
        regroup();
        int kern = choose(per_run);
        double per_run_orbit = sym ? per_run : 0.0;
        if (sym && !(kern == 1 || kern == 3)) {  // only the tensor-core kernels use orbits
            sym = 0;
            tile_bytes = tile_env ? std::atof(tile_env) * 1.0e6 : 4096.0e6;
            regroup();
            kern = choose(per_run);
        }
        S.release(keys_in);
        const int tc = kern == 1 || kern == 3;
        L.p.up_kernel = kern;
        L.p.sym = sym;
        if (std::getenv("IFGF_PLAN_VERBOSE"))
            fprintf(stderr, "[ifgf] level %d: %lld boxes, nC %d ns %d, %lld segments, %lld %s runs, %.2f per run "
                    "(orbit runs %.2f), tile %.0f MB, K7 kernel %d\n",
                    d, (long long)(L.p.b1 - L.p.b0), L.p.nC, L.p.ns, (long long)ns, (long long)nrun,
                    sym ? "orbit" : "cell", per_run, per_run_orbit, tile_bytes / 1e6, kern);
        int chunk_len = kern == 3 ? kChunkTC2 : (tc ? kChunkTC : kChunk);
        // small levels: shorter chunks, so that the pass still spans every SM (>= 2 chunks per SM)
        if (tc) chunk_len = (int)std::min<int64_t>(chunk_len, std::max<int64_t>(16, (ns + 2 * 148 - 1) / (2 * 148)));
        k_chunk_flag<<<nblocks(ns), TPB, 0, st>>>(rsm, ns, chunk_len, flag);
        inclusive_scan(S, flag, incl, ns, st);
        int64_t nch = d2h_one(incl + ns - 1, st);
        L.chunk_start = dev_alloc<int>(p, nch);
        k_chunk_emit<<<nblocks(ns), TPB, 0, st>>>(flag, incl, ns, L.chunk_start);
        IFGF_CUDA(cudaGetLastError());
        IFGF_CUDA(cudaStreamSynchronize(st));
        L.p.cell_seg = L.cell_seg;
        L.p.chunk_start = L.chunk_start;
        L.p.nchunk = nch;
        L.p.chunk_order = nullptr;
        if ((kern == 1 || kern == 3) && d < D && !std::getenv("IFGF_NO_CHUNK_ORDER")) {
            const LevelParams& LC = p->lev[d + 1].p;  // child grid
            const int fs = std::max(1, L.p.ns / std::max(1, LC.ns)), fc = std::max(1, L.p.nC / std::max(1, LC.nC));
            auto nbits = [](uint64_t v) { int b = 1; while (b < 63 && ((uint64_t)1 << b) <= v) ++b; return b; };
            const int64_t tile = (int64_t)std::max(1.0, tile_bytes / std::max(1.0, child_bytes_per_box));
            const int ch = chunk_len;
            const int bsub = nbits((uint64_t)(fs * fc * fc));
            const int bk = nbits((uint64_t)(ns / ch + 1));
            const int bcoarse = nbits((uint64_t)(L.p.ncell / (fs * fc * fc) + 1));
            const int btile = nbits((uint64_t)(L.p.nbox / tile + 1));
            if (btile + bcoarse + bk + bsub <= 64) {
                uint64_t* kin = S.get<uint64_t>(nch);
                uint64_t* kout = S.get<uint64_t>(nch);
                int* vin = S.get<int>(nch);
                L.chunk_order = dev_alloc<int>(p, nch);
                k_chunk_keys<<<nblocks(nch), TPB, 0, st>>>(L.chunk_start, nch, L.cell_seg, L.seg_box, L.seg_cell, rsm,
                                                           tile, ch, L.p.ns, L.p.nC, sym ? L.p.nC / 2 : 0, fs, fc,
                                                           bsub, bk, bcoarse, kin, vin);
                size_t bytes = 0;
                const int nb = btile + bcoarse + bk + bsub;
                IFGF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, L.chunk_order, (int)nch, 0,
                                                          nb, st));
                void* tmp = S.get<char>((int64_t)bytes);
                IFGF_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, kin, kout, vin, L.chunk_order, (int)nch, 0, nb,
                                                          st));
                IFGF_CUDA(cudaStreamSynchronize(st));
                S.release(tmp);
                S.release(kin);
                S.release(kout);
                S.release(vin);
                L.p.chunk_order = L.chunk_order;
            }
        }
        S.release(vals_in);
        S.release(keys_out);
        S.release(rs);
        S.release(rsm);
        S.release(incl);
    }

    step_time("7b K7 grouping");
    // 7c. multi-rank: owned-only neighbour / cousin lists and work items
    if (p->nranks > 1) {
        for (int d = 3; d <= D; ++d) {
            LevelHost& L = p->lev[d];
            const int64_t nb = L.p.nbox;
            int* cnt = S.get<int>(nb);
            int* wc = S.get<int>(nb);
            auto filter = [&](const int* off, const int* idx, const int** off_out, const int** idx_out,
                              const int2** items_out, int64_t* nitems_out) {
                k_count_owned<<<nblocks(nb), TPB, 0, st>>>(off, idx, nb, L.p.b0, L.p.b1, cnt);
                int64_t tot = 0;
                int* off2 = csr_offsets(p, S, cnt, nb, st, &tot);
                int* idx2 = dev_alloc<int>(p, tot);
                k_emit_owned<<<nblocks(nb), TPB, 0, st>>>(off, idx, nb, L.p.b0, L.p.b1, off2, idx2);
                k_witem_count_masked<<<nblocks(nb), TPB, 0, st>>>(L.box_start, nb, cnt, wc);
                int64_t ni = 0;
                int* woff = csr_offsets(p, S, wc, nb, st, &ni);
                int2* items = dev_alloc<int2>(p, ni);
                k_witem_fill_masked<<<nblocks(nb), TPB, 0, st>>>(L.box_start, nb, cnt, woff, items);
                IFGF_CUDA(cudaGetLastError());
                *off_out = off2;
                *idx_out = idx2;
                *items_out = items;
                *nitems_out = ni;
            };
            filter(L.cou_off, L.cou_idx, &L.p.cou_off, &L.p.cou_idx, &L.p.witems, &L.p.nwitems);
            if (d == D)
                filter(L.nbr_off, L.nbr_idx, &L.p.nbr_off, &L.p.nbr_idx, &L.p.witems_near, &L.p.nwitems_near);
            IFGF_CUDA(cudaStreamSynchronize(st));
            S.release(cnt);
            S.release(wc);
        }
    }
    if (p->nranks == 1 || D < 3) {
        LevelHost& LD = p->lev[D];
        LD.p.witems_near = LD.p.witems;
        LD.p.nwitems_near = LD.p.nwitems;
    }

    // 7d. source-list split of K3 / K6 on small problems: aim at >= 148 x 32 warps
    {
        auto split = [](int64_t nitems) {
            const int64_t target = 148 * 32;
            int64_t sp = nitems > 0 ? (target + nitems - 1) / nitems : 1;
            return (int)std::max<int64_t>(1, std::min<int64_t>(8, sp));
        };
        p->nparts_cou = 1;
        for (int d = 1; d <= D; ++d) {
            LevelParams& L = p->lev[d].p;
            L.nsplit_cou = d >= 3 ? split(L.nwitems) : 1;
            L.nsplit_near = 1;
            p->nparts_cou = std::max(p->nparts_cou, L.nsplit_cou);
        }
        p->lev[D].p.nsplit_near = split(p->lev[D].p.nwitems_near);
        p->nparts_near = p->lev[D].p.nsplit_near;
        for (int d = 1; d <= D; ++d) p->lev[d].p.nsplit_s2c = 1;
        const int64_t nleaf_owned = p->lev[D].p.b1 - p->lev[D].p.b0;  // K4: >= 4 blocks per SM
        if (nleaf_owned > 0)
            p->lev[D].p.nsplit_s2c = (int)std::max<int64_t>(1, std::min<int64_t>(8, (4 * 148 + nleaf_owned - 1) / nleaf_owned));
    }

    step_time("7c multi-rank lists");
    // 8. stats (algorithmic work units)
    {
        ifgf_stats& s = p->stats;
        s.n = n;
        s.levels = D;
        s.P_s = Ps;
        s.P_ang = Pa;
        s.P = P;
        s.k = p->k;
        for (int a = 0; a < 3; ++a) s.root_center[a] = p->root_c[a];
        s.root_side = p->H1;
        unsigned long long* acc = S.get<unsigned long long>(4 * (D + 2));
        IFGF_CUDA(cudaMemsetAsync(acc, 0, sizeof(unsigned long long) * 4 * (D + 2), st));
        k_stat_near<<<nblocks(p->lev[D].p.nbox), TPB, 0, st>>>(p->lev[D].p, acc);
        if (D >= 3 && p->lev[D].p.nseg > 0)
            k_stat_s2c<<<nblocks(p->lev[D].p.nseg), TPB, 0, st>>>(p->lev[D].p, P, acc + 1);
        for (int d = 3; d <= D; ++d) {
            k_stat_cousin<<<nblocks(p->lev[d].p.nbox), TPB, 0, st>>>(p->lev[d].p, acc + 4 * d);
            if (d > 3 && p->lev[d - 1].p.nseg > 0)
                k_stat_up<<<nblocks(p->lev[d - 1].p.nseg), TPB, 0, st>>>(p->lev[d].p, p->lev[d - 1].p, P,
                                                                          acc + 4 * d + 1);
        }
        IFGF_CUDA(cudaGetLastError());
        std::vector<unsigned long long> h(4 * (D + 2));
        IFGF_CUDA(cudaMemcpyAsync(h.data(), acc, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost, st));
        IFGF_CUDA(cudaStreamSynchronize(st));
        s.near_pairs = (int64_t)h[0];
        s.s2c_pairs = (int64_t)h[1];
        for (int d = 1; d <= D; ++d) {
            s.nbox[d] = p->lev[d].p.nbox;
            s.nseg[d] = p->lev[d].p.nseg;
            s.ns[d] = p->lev[d].p.ns;
            s.nC[d] = p->lev[d].p.nC;
            s.cousin_evals[d] = d >= 3 ? (int64_t)h[4 * d] : 0;
            s.upward_evals[d] = d >= 4 ? (int64_t)h[4 * d + 1] : 0;
            s.segment_bytes[d] = 16LL * P * p->lev[d].p.nseg;
            s.upward_kernel[d] = (d >= 4 && p->lev[d - 1].p.nseg > 0) ? p->lev[d - 1].p.up_kernel : -1;
        }
    }

    step_time("8 stats");
    // 9. apply scratch: permuted densities, sorted field, two segment-value levels
    p->a_sorted = dev_alloc<double2>(p, n);
    p->out_sorted = dev_alloc<double2>(p, n * p->nparts_cou);
    p->near_sorted = dev_alloc<double2>(p, n * p->nparts_near);
    for (int par = 0; par < 2; ++par) {
        int64_t mx = 0;
        for (int d = 3; d <= D; ++d)
            if ((d & 1) == par) mx = std::max(mx, p->lev[d].p.nseg);
        p->vals_cap[par] = mx * P;
        // one extra zeroed segment: the TC K7 reads k = 4*ceil(P/4)-1 >= P past a
        // segment's end (times a zero weight), so that memory must be finite
        p->vals[par] = dev_alloc<double2>(p, (mx + 1) * P);
        IFGF_CUDA(cudaMemsetAsync(p->vals[par], 0, sizeof(double2) * (size_t)(mx + 1) * P, st));
    }
    p->zseg = dev_alloc<double2>(p, P + 4);
    IFGF_CUDA(cudaMemsetAsync(p->zseg, 0, sizeof(double2) * (size_t)(P + 4), st));
    IFGF_CUDA(cudaStreamSynchronize(st));
    step_time("9 apply buffers");
    p->stats.plan_device_bytes = p->device_bytes;
    p->stats.plan_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
}

}  // namespace ifgf
