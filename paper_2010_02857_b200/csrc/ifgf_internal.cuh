// ifgf_internal.cuh -- plan layout, device math and shared helpers of libifgf.
// Citations P:n are lines of /root/reference/PAPER.md.  Nothing here is shared
// with oracle/ (the oracle implements the same written contract independently,
// DESIGN.md "Classification contract").
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/ifgf.h"
#include "fastmath.cuh"

namespace ifgf {

constexpr double kPi = 3.14159265358979323846;
constexpr int kMaxP1 = 16;  // max P_s, P_ang

// ---------------------------------------------------------------------------
// Error plumbing (host)
// ---------------------------------------------------------------------------
struct Error {
    ifgf_status st;
    std::string msg;
};
void set_error(const std::string& msg);
// Device-side bounds checks of the debug build (IFGF_CHECKS=1 at build time; the
// stand-in for compute-sanitizer, which this GPU pool does not allow): a failed
// check prints its location and traps (the apply then returns IFGF_ECUDA).
#ifdef IFGF_CHECKS
#define IFGF_DCHECK(cond)                                                                     \
    do {                                                                                      \
        if (!(cond)) {                                                                        \
            printf("IFGF_DCHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__,  \
                   __LINE__, (int)blockIdx.x, (int)threadIdx.x);                              \
            __trap();                                                                         \
        }                                                                                     \
    } while (0)
#else
#define IFGF_DCHECK(cond) \
    do {                  \
    } while (0)
#endif

#define IFGF_CUDA(call)                                                                              \
    do {                                                                                             \
        cudaError_t e_ = (call);                                                                     \
        if (e_ != cudaSuccess) {                                                                     \
            throw ::ifgf::Error{e_ == cudaErrorMemoryAllocation ? IFGF_ENOMEM : IFGF_ECUDA,         \
                                std::string(#call) + ": " + cudaGetErrorString(e_)};                 \
        }                                                                                            \
    } while (0)

// ---------------------------------------------------------------------------
// Level data: box tree + cone grid + relevant segments of one level d.
// Boxes are in Morton order; each box owns a contiguous range of the sorted
// points.  Segment s of the level is (seg_box[s], seg_cell[s]) in (box, cell)
// order; its P coefficients live at vals[s * P].
// ---------------------------------------------------------------------------
struct LevelParams {  // passed by value to kernels
    int d;
    int ns, nC;
    int64_t ncell;       // 2 * ns * nC^2
    int64_t W;           // 64-bit bitmap words per box
    double H, h, ds, dth, x0[3];
    double ids, idth;    // 1/ds, 1/dth (values only, never decisions)
    int64_t nbox;
    int64_t b0, b1;      // owned box range [b0, b1) (source partition)
    // boxes
    const int* box_ijk;       // 3 per box
    const double* box_c;      // 4 per box: centre x0 + (ijk + 1/2) H (IEEE, as box_centre) and 0
    const int* box_start;     // nbox + 1 (sorted point ranges)
    const int* box_parent;    // nbox
    const int* child_start;   // nbox + 1 (boxes of level d + 1)
    const int* nbr_off;       // nbox + 1
    const int* nbr_idx;
    const int* cou_off;       // nbox + 1
    const int* cou_idx;
    // relevant segments (owned boxes only; bitmap rows indexed by b - b0)
    const unsigned long long* bitmap;
    const unsigned* rank;     // exclusive prefix popcount over all words (global)
    int64_t nseg;
    const int* seg_box;
    const int* seg_cell;
    // classification boundary tables (host libm)
    const double* cos_tb;     // nC + 1
    const double* cphi;       // 2 nC + 1
    const double* sphi;       // 2 nC + 1
    // node geometry tables (host libm): h/s_k, sin/cos theta_i, sin/cos phi_j
    const double* rtab;       // ns * Ps
    const double* st_tab;     // nC * Pa
    const double* ct_tab;
    const double* sp_tab;     // 2 nC * Pa
    const double* cp_tab;
    // K6 warp work items (box, first point); multi-rank: only target boxes with an
    // owned cousin (and cou_off / cou_idx filtered to owned boxes)
    const int2* witems;
    int64_t nwitems;
    // K3 (leaf level) work items; multi-rank: target boxes with an owned neighbour
    const int2* witems_near;
    int64_t nwitems_near;
    // children of each box by octant ((i&1)<<2 | (j&1)<<1 | (k&1)) at level d + 1, -1 if absent
    const int* child_oct;
    // segments grouped by cone cell (box-independent K7 geometry): cell_seg = segment
    // indices sorted by (cell, segment); chunk_start = first position of each chunk
    // of <= kChunk segments sharing one cell
    const int* cell_seg;
    const int* chunk_start;
    int64_t nchunk;
    const int* chunk_order;  // execution order of the chunks (TC levels, L2 locality) or null
    // K7 kernel of the pass into this level (as PARENT level), chosen at plan time
    // from the segments per cell: 0 = cell-grouped staged DFMA (chunks of
    // <= kChunk), 1 = FP64 tensor-core GEMM (chunks of <= kChunkTC), 2 =
    // per-evaluation geometry (no chunks, separate K5 fit)
    int up_kernel;
    int sym;  // K7 chunks grouped by quarter-turn orbits of the parent cell (reading R18)
    int cls_exact;  // 1: classify always takes the exact IEEE chain (env IFGF_EXACT_CLASSIFY; tests)
    // source-list split of the target-major kernels on small problems: K6 (this level)
    // and K3 (leaf level) run nsplit warps per work item, warp p taking every nsplit-th
    // cousin / neighbour box and accumulating into field part p (summed in a fixed
    // order by the un-permute); 1 on large problems
    int nsplit_cou, nsplit_near;
    int nsplit_s2c;  // K4 blocks per leaf (leaf level; small problems only)
};

constexpr int kChunk = 16;
constexpr int kChunkTC = 96;
constexpr int kChunkTC2 = 32;

struct LevelHost {
    LevelParams p{};
    // owned device allocations
    int *box_ijk = nullptr, *box_start = nullptr, *box_parent = nullptr, *child_start = nullptr;
    double* box_c = nullptr;
    int *nbr_off = nullptr, *nbr_idx = nullptr, *cou_off = nullptr, *cou_idx = nullptr;
    unsigned long long* bitmap = nullptr;
    unsigned* rank = nullptr;
    int *seg_box = nullptr, *seg_cell = nullptr;
    double *cos_tb = nullptr, *cphi = nullptr, *sphi = nullptr;
    double *rtab = nullptr, *st_tab = nullptr, *ct_tab = nullptr, *sp_tab = nullptr, *cp_tab = nullptr;
    int2* witems = nullptr;
    int *child_oct = nullptr, *cell_seg = nullptr, *chunk_start = nullptr, *chunk_order = nullptr;
    int64_t ncou = 0, nnbr = 0;
    std::vector<int> box_ijk_host;  // kept for plan export (small levels only)
};

}  // namespace ifgf

struct ifgf_plan_s {
    int device = 0;
    int64_t n = 0;
    double k = 0;
    int D = 1, Ps = 3, Pa = 5, P = 75;
    unsigned stage_mask = IFGF_STAGE_ALL;
    int rank = 0, nranks = 1;
    double root_c[3] = {0, 0, 0}, H1 = 1, x0[3] = {0, 0, 0};
    std::vector<ifgf::LevelHost> lev;  // 1..D
    // sorted points (SoA), permutation sorted -> caller
    double *px = nullptr, *py = nullptr, *pz = nullptr;
    int* perm = nullptr;
    // Chebyshev tables
    double* cheb_Ms = nullptr;  // Ps x Ps fit matrix (2 - delta_i0)/n T_i(t_k)
    double* cheb_Ma = nullptr;  // Pa x Pa
    // apply scratch
    double2* a_sorted = nullptr;
    double2* out_sorted = nullptr;   // cousin (K6) sums, Morton order, nparts_cou parts of n
    double2* near_sorted = nullptr;  // near field (K3), Morton order, nparts_near parts of n
    int nparts_cou = 1, nparts_near = 1;
    double2* vals[2] = {nullptr, nullptr};  // ping-pong by level parity (+1 zeroed tail segment)
    double2* zseg = nullptr;                // P + 4 zeros: the TC K7's absent-column operand
    int64_t vals_cap[2] = {0, 0};
    double2* host_stage_dev_in = nullptr;   // ifgf_apply_host buffers
    double2* host_stage_dev_out = nullptr;
    // stats / profiling
    ifgf_stats stats{};
    bool sticky_cuda_error = false;
    int profile = 0;
    double prof_ms[IFGF_NUM_KCLASS] = {0};
    int64_t prof_launches[IFGF_NUM_KCLASS] = {0};
    std::vector<cudaEvent_t> ev_pool;
    struct PendingEv {
        int cls;
        cudaEvent_t a, b;
    };
    std::vector<PendingEv> pending;
    int* dev_bad = nullptr;  // device flag: apply-time invariant violation (EINTERNAL)
    int legacy_upward = 0;   // env IFGF_LEGACY_UPWARD: K7 variant override (A/B testing, tests)
    int no_symmetry = 0;     // env IFGF_NO_SYMMETRY: K7 chunks by cell only (A/B testing, tests)
    int cls_exact = 0;       // env IFGF_EXACT_CLASSIFY: no classification fast path (tests)
    int tc_umax = 1 << 30;      // env IFGF_TC_UMAX: cap on staged child cells in the TC K7 (tests the fallback)
    int stage_slots = 1 << 30;  // env IFGF_STAGE_SLOTS: cap on staged child segments per warp in K6 / K7-pe (tests)
    int legacy_cousin = 0;      // env IFGF_LEGACY_COUSIN=1: per-lane global-load K6 (A/B testing)
    unsigned long long* phase_clk = nullptr;  // env IFGF_PHASE_PROF: TC K7 per-phase clock sums
    int64_t device_bytes = 0;
    std::vector<void*> allocs;  // every cudaMalloc of the plan
    // multi-GPU: borrowed ncclComm_t (opts.nccl_comm); ifgf_apply all-reduces out
    void* nccl_comm = nullptr;
    // CUDA graph of one apply (captured on cap_stream for one (densities, out) pair,
    // replayed on the caller's stream)
    bool use_graph = true;
    bool no_concurrency = false;  // env IFGF_NO_CONCURRENCY: captured apply on one stream (A/B)
    bool graph_failed = false;
    cudaStream_t cap_stream = nullptr;
    cudaGraphExec_t gexec = nullptr;
    const void* g_dens = nullptr;
    void* g_out = nullptr;
    cudaStream_t side[2] = {nullptr, nullptr};  // captured apply: K3 stream, K4/K5/K7 stream
    std::vector<cudaEvent_t> ev;                // their fork / join / per-level events
};

namespace ifgf {

// Allocation helper that records ownership in the plan.
template <class T>
T* dev_alloc(ifgf_plan_s* p, int64_t count) {
    if (count <= 0) count = 1;
    void* ptr = nullptr;
    IFGF_CUDA(cudaMalloc(&ptr, sizeof(T) * (size_t)count));
    p->allocs.push_back(ptr);
    p->device_bytes += (int64_t)(sizeof(T) * (size_t)count);
    return static_cast<T*>(ptr);
}
void dev_free(ifgf_plan_s* p, void* ptr);

void build_plan(ifgf_plan_s* p, const double* points_dev, const ifgf_opts& o);
void run_apply(ifgf_plan_s* p, const double2* dens, double2* out, cudaStream_t st, bool conc);
void debug_level_pass(ifgf_plan_s* p, int d, const double2* values_h, unsigned what, double2* field_h,
                      double2* parent_h);

// ---------------------------------------------------------------------------
// Device helpers
// ---------------------------------------------------------------------------
struct Cls {
    int is, it, ip;
    double r, ir, us, ut, up;  // ir = 1/r (value, ~1 ulp)
};

// Classification of the relative vector v at a level (DESIGN.md
// "Classification contract", reading R7).  The
// discrete decisions are those of IEEE-rounded + - * / sqrt without contraction
// against host-libm boundary tables: r, s = h/r, i_s = floor(s/ds),
// cos(theta) = v_z/r and the phi cross products.  The angles
// theta = atan2(rho, v_z), phi = atan2(v_y, v_x) (reading R13) come from the lean
// fm::atan2 and only supply first guesses and the local coordinates
// u = 2 (v - v_a)/dv - 1 (values).
//
// Fast path: s/ds and v_z/r from one rsqrt (relative error < 1e-15 against the
// IEEE chain); i_s and i_theta are accepted when s/ds is >= 1e-13 (s/ds + 1)
// from an integer and v_z/r is >= 8e-15 from the boundary cosines on both sides
// (> 100x the error bound), so they equal the contract's decisions; otherwise
// (probability ~1e-12 per call) the exact IEEE chain decides.  The phi cross
// products are exact IEEE products in every case.
__device__ __forceinline__ Cls classify(const LevelParams& L, double vx, double vy, double vz) {
    Cls c;
    const double rho2 = __dadd_rn(__dmul_rn(vx, vx), __dmul_rn(vy, vy));
    const double r2 = __dadd_rn(rho2, __dmul_rn(vz, vz));
    const double y = fm::rsqrt_fast(r2);
    double s = L.h * y;
    const double q = s * L.ids;
    const double fq = floor(q), tq = 1e-13 * (q + 1.0);
    int is = (int)fq;
    bool ok;
    if (is >= L.ns - 1) {
        is = L.ns - 1;
        ok = q - (double)(L.ns - 1) >= tq;
    } else {
        ok = (q - fq >= tq) && (fq + 1.0 - q >= tq);
    }
    // theta: i_theta = #{k in 1..nC-1 : vz/r <= cos(k dtheta)}
    const double ct = vz * y;
    const double rho = rho2 > 0.0 ? rho2 * fm::rsqrt_fast(rho2) : 0.0;
    const double th = fm::atan2(rho, vz);
    int it = (int)(th * L.idth);
    it = it < 0 ? 0 : (it > L.nC - 1 ? L.nC - 1 : it);
    constexpr double tc = 8e-15;
    if (it > 0 && !(ct <= __ldg(L.cos_tb + it) - tc)) ok = false;
    if (it < L.nC - 1 && !(ct > __ldg(L.cos_tb + it + 1) + tc)) ok = false;
    c.r = r2 * y;
    c.ir = y;
    if (!ok || L.cls_exact) {  // near a boundary: the contract's exact IEEE chain
        c.r = __dsqrt_rn(r2);
        s = __ddiv_rn(L.h, c.r);
        const int ie = (int)floor(__ddiv_rn(s, L.ds));
        is = ie > L.ns - 1 ? L.ns - 1 : ie;
        const double cte = __ddiv_rn(vz, c.r);
        while (it > 0 && !(cte <= __ldg(L.cos_tb + it))) --it;
        while (it < L.nC - 1 && cte <= __ldg(L.cos_tb + it + 1)) ++it;
    }
    c.is = is;
    c.it = it;
    // phi: unique j with cross_j >= 0 > cross_{j+1}; poles -> 0
    const int n2 = 2 * L.nC;
    double ph = 0.0;
    int ip = 0;
    if (!(vx == 0.0 && vy == 0.0)) {
        ph = fm::atan2_2pi(vy, vx);
        ip = (int)(ph * L.idth);
        ip = ip < 0 ? 0 : (ip > n2 - 1 ? n2 - 1 : ip);
        for (int iter = 0; iter < 2 * n2; ++iter) {
            double cj = __dsub_rn(__dmul_rn(vy, __ldg(L.cphi + ip)), __dmul_rn(vx, __ldg(L.sphi + ip)));
            if (!(cj >= 0.0)) {
                ip = ip == 0 ? n2 - 1 : ip - 1;
                continue;
            }
            double cj1 = __dsub_rn(__dmul_rn(vy, __ldg(L.cphi + ip + 1)), __dmul_rn(vx, __ldg(L.sphi + ip + 1)));
            if (cj1 >= 0.0) {
                ip = ip == n2 - 1 ? 0 : ip + 1;
                continue;
            }
            break;
        }
    }
    c.ip = ip;
    const double i2s = 2.0 * L.ids, i2t = 2.0 * L.idth;
    c.us = fma(s - c.is * L.ds, i2s, -1.0);
    c.ut = fma(th - c.it * L.dth, i2t, -1.0);
    c.up = fma(ph - c.ip * L.dth, i2t, -1.0);
    return c;
}

__device__ __forceinline__ int64_t cell_of(const LevelParams& L, const Cls& c) {
    return ((int64_t)c.ip * L.nC + c.it) * L.ns + c.is;
}

// Slot of (box b, cell) among the level's relevant segments (O(1) rank lookup),
// or -1 if the segment is not relevant.
__device__ __forceinline__ int64_t seg_slot(const LevelParams& L, int64_t b, int64_t cell) {
    IFGF_DCHECK(b >= L.b0 && b < L.b1 && cell >= 0 && cell < L.ncell);
    int64_t w = (b - L.b0) * L.W + (cell >> 6);
    unsigned long long word = __ldg(L.bitmap + w);
    unsigned long long bit = 1ull << (cell & 63);
    if (!(word & bit)) return -1;
    const int64_t slot = (int64_t)__ldg(L.rank + w) + __popcll(word & (bit - 1));
    IFGF_DCHECK(slot >= 0 && slot < L.nseg);
    return slot;
}

__device__ __forceinline__ double box_centre(const LevelParams& L, int k, int axis) {
    return __dadd_rn(L.x0[axis], __dmul_rn((double)k + 0.5, L.H));
}

// ---- quarter-turn symmetry about z (reading R18) ----------------
// With n_C even on both levels the phi tables are exactly quarter-turn symmetric,
// so rotating a parent cell by q quarter turns (phi sector + q n_C/2) rotates its
// nodes exactly; the node's child-relative geometry is that of the
// representative cell for child octant rot_oct(o, q) and child cell
// rot_cell(u, q) (poles v_x = v_y = 0 excepted: sector 0 stays 0).
constexpr int kPoleFlag = 1 << 30;
__device__ __forceinline__ int rot_oct(int o, int q) {  // (x, y) -> (-y, x), q times
    for (int i = 0; i < (q & 3); ++i) o = ((~o & 2) << 1) | ((o & 4) >> 1) | (o & 1);
    return o;
}
__device__ __forceinline__ int rot_cell(const LevelParams& L, int cell, int q) {
    const int nsc = L.ns * L.nC;
    const int ip = cell / nsc;
    return ((ip + q * (L.nC >> 1)) % (2 * L.nC)) * nsc + (cell - ip * nsc);
}
// child cell of a staged geometry entry u for a segment q quarter turns away
__device__ __forceinline__ int sym_cell(const LevelParams& L, int u, int q) {
    return (u & kPoleFlag) ? (u & ~kPoleFlag) : (q ? rot_cell(L, u, q) : u);
}
// quarter turns of parent cell `cell` and its representative (sector mod n_C/2)
__device__ __forceinline__ int sym_quarter(const LevelParams& LP, int cell) {
    return LP.sym ? (cell / (LP.ns * LP.nC)) / (LP.nC >> 1) : 0;
}
__device__ __forceinline__ int sym_rep(const LevelParams& LP, int cell) {
    if (!LP.sym) return cell;
    const int nsc = LP.ns * LP.nC;
    const int ip = cell / nsc;
    return (ip % (LP.nC >> 1)) * nsc + (cell - ip * nsc);
}

// Centre of box B from the plan's table (bit-identical to box_centre).
__device__ __forceinline__ void box_centre3(const LevelParams& L, int B, double& cx, double& cy, double& cz) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(L.box_c) + 2 * (int64_t)B);
    cx = a.x;
    cy = a.y;
    cz = __ldg(L.box_c + 4 * (int64_t)B + 2);
}

// Chebyshev polynomials T_0..T_{n-1} at u (three-term recurrence).
template <int N>
__device__ __forceinline__ void cheb_T(double u, double* T) {
    T[0] = 1.0;
    if (N > 1) T[1] = u;
    const double u2 = 2.0 * u;
#pragma unroll
    for (int i = 2; i < N; ++i) T[i] = fma(u2, T[i - 1], -T[i - 2]);
}
__device__ __forceinline__ void cheb_T_rt(int n, double u, double* T) {
    T[0] = 1.0;
    if (n > 1) T[1] = u;
    const double u2 = 2.0 * u;
    for (int i = 2; i < n; ++i) T[i] = fma(u2, T[i - 1], -T[i - 2]);
}

// Evaluate the tensor Chebyshev interpolant with coefficients C (layout
// ((c * PA + b) * PS + a) for s-index a, theta-index b, phi-index c) at local
// coordinates (us, ut, up): contraction over phi, then theta, then s.
// The phi loop is kept rolled (T_c by recurrence) so that only one phi-slab of
// P_ang * P_s coefficients is in flight per thread (register pressure).
template <int PS, int PA>
__device__ __forceinline__ double2 contract(const double2* __restrict__ C, const double* Ts, const double* Tt,
                                            double up) {
    double wr[PA * PS], wi[PA * PS];
#pragma unroll
    for (int i = 0; i < PA * PS; ++i) {
        double2 v = __ldg(C + i);
        wr[i] = v.x;
        wi[i] = v.y;
    }
    double tm1 = 1.0, t = up;
    const double u2 = 2.0 * up;
#pragma unroll 1
    for (int c = 1; c < PA; ++c) {
        const double2* __restrict__ Cc = C + c * PA * PS;
#pragma unroll
        for (int i = 0; i < PA * PS; ++i) {
            double2 v = __ldg(Cc + i);
            wr[i] = fma(t, v.x, wr[i]);
            wi[i] = fma(t, v.y, wi[i]);
        }
        const double tn = fma(u2, t, -tm1);
        tm1 = t;
        t = tn;
    }
    double xr[PS], xi[PS];
#pragma unroll
    for (int a = 0; a < PS; ++a) {
        xr[a] = wr[a];
        xi[a] = wi[a];
    }
#pragma unroll
    for (int b = 1; b < PA; ++b)
#pragma unroll
        for (int a = 0; a < PS; ++a) {
            xr[a] = fma(Tt[b], wr[b * PS + a], xr[a]);
            xi[a] = fma(Tt[b], wi[b * PS + a], xi[a]);
        }
    double fr = xr[0], fi = xi[0];
#pragma unroll
    for (int a = 1; a < PS; ++a) {
        fr = fma(Ts[a], xr[a], fr);
        fi = fma(Ts[a], xi[a], fi);
    }
    return make_double2(fr, fi);
}

// Tensor contraction from shared memory (same order as contract()).
template <int PS, int PA>
__device__ __forceinline__ double2 contract_sm(const double2* C, const double* Ts, const double* Tt, double up) {
    double wr[PA * PS], wi[PA * PS];
#pragma unroll
    for (int i = 0; i < PA * PS; ++i) {
        double2 v = C[i];
        wr[i] = v.x;
        wi[i] = v.y;
    }
    double tm1 = 1.0, t = up;
    const double u2 = 2.0 * up;
#pragma unroll
    for (int c = 1; c < PA; ++c) {
#pragma unroll
        for (int i = 0; i < PA * PS; ++i) {
            double2 v = C[c * PA * PS + i];
            wr[i] = fma(t, v.x, wr[i]);
            wi[i] = fma(t, v.y, wi[i]);
        }
        const double tn = fma(u2, t, -tm1);
        tm1 = t;
        t = tn;
    }
    double xr[PS], xi[PS];
#pragma unroll
    for (int a = 0; a < PS; ++a) {
        xr[a] = wr[a];
        xi[a] = wi[a];
    }
#pragma unroll
    for (int b = 1; b < PA; ++b)
#pragma unroll
        for (int a = 0; a < PS; ++a) {
            xr[a] = fma(Tt[b], wr[b * PS + a], xr[a]);
            xi[a] = fma(Tt[b], wi[b * PS + a], xi[a]);
        }
    double fr = xr[0], fi = xi[0];
#pragma unroll
    for (int a = 1; a < PS; ++a) {
        fr = fma(Ts[a], xr[a], fr);
        fi = fma(Ts[a], xi[a], fi);
    }
    return make_double2(fr, fi);
}

// Same contraction with a small live register set: phi innermost per (a, b)
// (one complex accumulator), then theta, then s; 3 x 5 x 5 + 15 + 3 complex x
// real MACs as contract_sm.  Tp is formed from u_phi by the recurrence.
template <int PS, int PA, bool GLOBAL = false, int UNR = 1>
__device__ __forceinline__ double2 contract_sm_lr(const double2* C, const double* Ts, const double* Tt, double up) {
    // theta outermost and rolled (T_b by recurrence from Tt[0..1]); per b the
    // 3 x 5 (s, phi) slab: phi contraction, then accumulate T_b * (.) per s.
    double Tp[PA];
    cheb_T<PA>(up, Tp);
    double xr[PS], xi[PS];
#pragma unroll
    for (int a = 0; a < PS; ++a) xr[a] = xi[a] = 0.0;
    const double ut = PA > 1 ? Tt[1] : 0.0, u2 = 2.0 * ut;
    double tbm1 = 0.0, tb = 1.0;
#pragma unroll UNR
    for (int b = 0; b < PA; ++b) {
        const double2* Cb = C + b * PS;
#pragma unroll
        for (int a = 0; a < PS; ++a) {
            double gr = 0.0, gi = 0.0;
#pragma unroll
            for (int c = 0; c < PA; ++c) {
                const double2 v = GLOBAL ? __ldg(Cb + c * PA * PS + a) : Cb[c * PA * PS + a];
                gr = fma(Tp[c], v.x, gr);
                gi = fma(Tp[c], v.y, gi);
            }
            xr[a] = fma(tb, gr, xr[a]);
            xi[a] = fma(tb, gi, xi[a]);
        }
        const double tn = b == 0 ? ut : fma(u2, tb, -tbm1);
        tbm1 = tb;
        tb = tn;
    }
    double fr = 0.0, fi = 0.0;
#pragma unroll
    for (int a = 0; a < PS; ++a) {
        fr = fma(Ts[a], xr[a], fr);
        fi = fma(Ts[a], xi[a], fi);
    }
    return make_double2(fr, fi);
}

template <int PS, int PA>
__device__ __forceinline__ double2 eval_interp(const double2* __restrict__ C, double us, double ut, double up) {
    double Ts[PS], Tt[PA];
    cheb_T<PS>(us, Ts);
    cheb_T<PA>(ut, Tt);
    return contract<PS, PA>(C, Ts, Tt, up);
}

// Runtime-order fallback (any P_s, P_ang <= kMaxP1).
__device__ __forceinline__ double2 eval_interp_rt(const double2* __restrict__ C, int PS, int PA, double us, double ut,
                                                  double up) {
    double Ts[kMaxP1], Tt[kMaxP1], Tp[kMaxP1];
    cheb_T_rt(PS, us, Ts);
    cheb_T_rt(PA, ut, Tt);
    cheb_T_rt(PA, up, Tp);
    double fr = 0.0, fi = 0.0;
    for (int c = 0; c < PA; ++c) {
        double gr = 0.0, gi = 0.0;
        for (int b = 0; b < PA; ++b) {
            double hr = 0.0, hi = 0.0;
            for (int a = 0; a < PS; ++a) {
                double2 v = __ldg(C + (c * PA + b) * PS + a);
                hr = fma(Ts[a], v.x, hr);
                hi = fma(Ts[a], v.y, hi);
            }
            gr = fma(Tt[b], hr, gr);
            gi = fma(Tt[b], hi, gi);
        }
        fr = fma(Tp[c], gr, fr);
        fi = fma(Tp[c], gi, fi);
    }
    return make_double2(fr, fi);
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

}  // namespace ifgf
