// apply.cu -- one IFGF operator application (Algorithm 1):
//   K3 near field, K4 leaf source-to-cone,
//   K5 Chebyshev coefficient fit,
//   K6 cousin-point interpolation,
//   K7 upward interpolation + recentering.
// Every output has exactly one writer (target-major K3/K6, parent-node-major
// K7): no atomics on values, deterministic results.
#include <climits>


#include <cstdio>
#include <cmath>

#include "ifgf_internal.cuh"

namespace ifgf {

namespace {

constexpr int TPB = 128;
constexpr double kInv4Pi = 0.079577471545947667884;  // 1/(4 pi)

inline int nblk(int64_t n, int tpb = TPB) {
    int64_t b = (n + tpb - 1) / tpb;
    return (int)(b < 1 ? 1 : b);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Bulk (TMA) copies global -> shared completing on an mbarrier (sm_90+ async proxy):
// one instruction per contiguous segment instead of one 16-byte cp.async per lane.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    unsigned ok = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!ok);
}

// 1/x for x > 0 (values only): hardware approximation + two Newton steps (~1 ulp).
__device__ __forceinline__ double rcp_nr(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}

// Warp-cooperative staging of the distinct child segments the lanes need: lanes
// with equal slots form one group (match.any), the lowest lane of each group with
// slot >= 0 copies its segment (one bulk copy) into buffer slot `idx` (groups in
// lane order, at most cap); returns the lane's buffer slot, or -1 (no segment, or
// beyond cap: the caller reads global memory).  Completion: the buffer's mbarrier
// (expect_tx of the total bytes by lane 0).
template <int P>
__device__ __forceinline__ int stage_distinct(int slot, int lane, int cap, const double2* __restrict__ vals,
                                              double2* buf0, int sp, unsigned long long* bar) {
    const unsigned grp = __match_any_sync(~0u, slot);
    const int leader = __ffs(grp) - 1;
    const bool lead = slot >= 0 && lane == leader;
    const unsigned leaders = __ballot_sync(~0u, lead);
    const int idx = __popc(leaders & ((1u << lane) - 1u));
    const int nd = min(__popc(leaders), cap);
    if (lead && idx < cap) {
        fence_proxy_async();  // the buffer's previous contents were read (generic proxy)
        bulk_g2s(buf0 + idx * sp, vals + (int64_t)slot * P, P * sizeof(double2), bar);
    }
    if (lane == 0) mbar_arrive_expect_tx(bar, (unsigned)(nd * P * sizeof(double2)));
    const int bi = __shfl_sync(~0u, idx, leader);
    return (slot >= 0 && bi < cap) ? bi : -1;
}

__global__ void k_permute(const double2* __restrict__ in, const int* __restrict__ perm, int64_t n, double2* out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[perm[i]];
}
// out[perm[i]] = sum of the nfar cousin parts (levels D..3) + sum of the nnear
// near-field parts, in that fixed order
__global__ void k_unpermute_sum(const double2* __restrict__ far, int nfar, const double2* __restrict__ near,
                                int nnear, const int* __restrict__ perm, int64_t n, double2* out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        double2 acc = far[i];
        for (int q = 1; q < nfar; ++q) {
            const double2 v = far[q * n + i];
            acc.x += v.x;
            acc.y += v.y;
        }
        for (int q = 0; q < nnear; ++q) {
            const double2 v = near[q * n + i];
            acc.x += v.x;
            acc.y += v.y;
        }
        out[perm[i]] = acc;
    }
}

// K3: out[l] = sum over owned neighbour boxes B of the leaf T containing l,
// sum_{m in B, m != l} a_m e^{ik r}/(4 pi r)  (raw kernel, reading R11).
// One warp per (leaf, 32 targets).  The neighbours' sources are staged per warp
// in shared memory in chunks of 32 (one coalesced load per lane), then every
// lane sweeps the chunk (broadcast reads); 1/r from one rsqrt, phase by fm::sincos.
template <bool SPLIT>  // SPLIT (small problems only, nsplit_near > 1): nsplit warps per work item
__global__ void __launch_bounds__(TPB, 8) k_near(LevelParams L, const double* __restrict__ px,
                                              const double* __restrict__ py, const double* __restrict__ pz,
                                              const double2* __restrict__ a, double k, double2* out) {
    __shared__ double sx[TPB / 32][32], sy[TPB / 32][32], sz[TPB / 32][32];
    __shared__ double2 sa[TPB / 32][32];
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int nsplit = SPLIT ? L.nsplit_near : 1;
    const int64_t item = SPLIT ? wid / nsplit : wid;
    const int part = SPLIT ? (int)(wid - item * nsplit) : 0;  // this warp's share of the neighbour boxes
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (item >= L.nwitems_near) return;  // warp-uniform
    if (SPLIT) out += (int64_t)part * (L.box_start[L.nbox]);  // field part (parts are n apart)
    const int2 it = L.witems_near[item];
    // items with <= 16 targets run split: lanes l and l + 16 take the same target
    // and alternate sources; the halves are summed at the end (fixed order)
    const int T = it.x, nT = min(32, L.box_start[T + 1] - it.y);
    const bool split = nT <= 16;
    const int half = split ? lane >> 4 : 0, step = split ? 2 : 1;
    const int l = it.y + (split ? (lane & 15) : lane);
    const bool active = l < it.y + nT;
    double x = 0.0, y = 0.0, z = 0.0;
    if (active) {
        x = px[l];
        y = py[l];
        z = pz[l];
    }
    double ar = 0.0, ai = 0.0;
    const int e1 = L.nbr_off[T + 1];
    for (int e = L.nbr_off[T] + part; e < e1; e += nsplit) {
        const int B = L.nbr_idx[e];
        if (B < L.b0 || B >= L.b1) continue;
        const int m0 = L.box_start[B], m1 = L.box_start[B + 1];
        for (int c0 = m0; c0 < m1; c0 += 32) {
            const int cn = min(32, m1 - c0);
            __syncwarp();
            if (lane < cn) {
                sx[w][lane] = px[c0 + lane];
                sy[w][lane] = py[c0 + lane];
                sz[w][lane] = pz[c0 + lane];
                sa[w][lane] = a[c0 + lane];
            }
            __syncwarp();
            if (active) {
#pragma unroll 2
                for (int t = half; t < cn; t += step) {
                    if (c0 + t == l) continue;
                    const double dx = x - sx[w][t], dy = y - sy[w][t], dz = z - sz[w][t];
                    const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
                    const double ri = fm::rsqrt_fast(r2);
                    const double r = r2 * ri;
                    double sn, cs;
                    fm::sincos(k * r, &sn, &cs);
                    const double wr = kInv4Pi * ri;
                    const double2 am = sa[w][t];
                    const double gr = cs * wr, gi = sn * wr;
                    ar = fma(am.x, gr, fma(-am.y, gi, ar));
                    ai = fma(am.x, gi, fma(am.y, gr, ai));
                }
            }
        }
    }
    if (split) {
        ar += __shfl_down_sync(~0u, ar, 16);
        ai += __shfl_down_sync(~0u, ai, 16);
    }
    if (active && half == 0) out[l] = make_double2(ar, ai);
}

__device__ __forceinline__ void node_off(const LevelParams& LP, int Ps, int Pa, int cell, int n, double off[3]) {
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
}

// K4: V[B, gamma, y] = sum_{m in B} a_m (|y-c|/|y-x_m|) e^{ik(|y-x_m| - |y-c|)}
// (eq. factored_f P:432-434 at the nodes of eq. interp_pts), block per owned leaf.
template <int PS, int PA>
__device__ __forceinline__ void fit_lines_inplace(double2* V, int cnt, const int* seg, const double* Ms,
                                                  const double* Ma, double2* out, int tid, int nt);

// PS_ > 0: orders known at compile time and <= 8 segments per leaf (leaf grid
// (1, 2)): the node values stay in shared memory and the K5 fit is fused.
constexpr int S2C_CHUNK = 256;
template <int PS_, int PA_>
__global__ void __launch_bounds__(TPB, 8) k_s2c(LevelParams L, const double* __restrict__ px,
                                             const double* __restrict__ py, const double* __restrict__ pz,
                                             const double2* __restrict__ a, double k, int Ps, int Pa,
                                             double2* vals, const double* __restrict__ Ms,
                                             const double* __restrict__ Ma) {
    constexpr bool FUSE = PS_ > 0;
    constexpr int PF = FUSE ? PS_ * PA_ * PA_ : 1;
    __shared__ double2 sV[FUSE ? 8 * PF : 1];
    __shared__ int sSeg[8];
    const int P = FUSE ? PF : Ps * Pa * Pa;
    // small problems (nsplit_s2c > 1): several blocks per leaf, each a contiguous share of its segments
    const int64_t B = L.b0 + blockIdx.x / L.nsplit_s2c;
    const int part = (int)(blockIdx.x % L.nsplit_s2c);
    __shared__ double sw[S2C_CHUNK][4];  // source - centre (x, y, z), |source - centre|^2
    __shared__ double2 sa[S2C_CHUNK];
    const int64_t row = (B - L.b0) * L.W;
    int64_t s0 = L.rank[row], s1 = L.rank[row + L.W];
    if (L.nsplit_s2c > 1) {
        const int64_t q = (s1 - s0 + L.nsplit_s2c - 1) / L.nsplit_s2c;
        s0 = min(s1, s0 + part * q);
        s1 = min(s1, s0 + q);
    }
    const int64_t nitem = (s1 - s0) * P;
    if (nitem == 0) return;
    double cx, cy, cz;
    box_centre3(L, B, cx, cy, cz);
    const int m0 = L.box_start[B], m1 = L.box_start[B + 1];
    for (int64_t base = 0; base < nitem; base += blockDim.x) {
        int64_t j = base + threadIdx.x;
        bool active = j < nitem;
        double off[3] = {0, 0, 0};
        int64_t s = 0;
        int n = 0;
        if (active) {
            s = s0 + j / P;
            n = (int)(j % P);
            node_off(L, Ps, Pa, L.seg_cell[s], n, off);
        }
        const double oo = off[0] * off[0] + off[1] * off[1] + off[2] * off[2];
        const double ro = sqrt(oo);
        double vr = 0.0, vi = 0.0;
        for (int c0 = m0; c0 < m1; c0 += S2C_CHUNK) {
            int cn = min(S2C_CHUNK, m1 - c0);
            __syncthreads();
            for (int t = threadIdx.x; t < cn; t += blockDim.x) {
                const double wx = px[c0 + t] - cx, wy = py[c0 + t] - cy, wz = pz[c0 + t] - cz;
                sw[t][0] = wx;
                sw[t][1] = wy;
                sw[t][2] = wz;
                sw[t][3] = fma(wx, wx, fma(wy, wy, wz * wz));
                sa[t] = a[c0 + t];
            }
            __syncthreads();
            if (active) {
#pragma unroll 2
                for (int t = 0; t < cn; ++t) {
                    const double wx = sw[t][0], wy = sw[t][1], wz = sw[t][2], ww = sw[t][3];
                    const double dx = off[0] - wx, dy = off[1] - wy, dz = off[2] - wz;
                    const double d2 = fma(dx, dx, fma(dy, dy, dz * dz));
                    const double rdi = fm::rsqrt_fast(d2);
                    const double rd = d2 * rdi;
                    // |y - x_m| - |y - c| = (w.w - 2 off.w) / (|off - w| + |off|)   (reading R17)
                    const double num = fma(-2.0, fma(off[0], wx, fma(off[1], wy, off[2] * wz)), ww);
                    const double diff = num * rcp_nr(rd + ro);
                    double ratio = ro * rdi;
                    double sn, cs;
                    fm::sincos(k * diff, &sn, &cs);
                    double gr = ratio * cs, gi = ratio * sn;
                    double2 am = sa[t];
                    vr = fma(am.x, gr, fma(-am.y, gi, vr));
                    vi = fma(am.x, gi, fma(am.y, gr, vi));
                }
            }
        }
        if (active) {
            if constexpr (FUSE) sV[j] = make_double2(vr, vi);
            else vals[s * P + n] = make_double2(vr, vi);
        }
    }
    if constexpr (FUSE) {
        const int cnt = (int)(s1 - s0);
        if (threadIdx.x < cnt) sSeg[threadIdx.x] = (int)(s0 + threadIdx.x);
        fit_lines_inplace<PS_, PA_>(sV, cnt, sSeg, Ms, Ma, vals, threadIdx.x, blockDim.x);
    }
}

// K5: node values -> tensor Chebyshev coefficients in place (reading R1),
// separable passes along s, theta, phi; one warp per segment.
__global__ void k_fit(int64_t nseg, int Ps, int Pa, const double* __restrict__ Ms, const double* __restrict__ Ma,
                      double2* vals) {
    extern __shared__ double2 sm[];
    const int P = Ps * Pa * Pa;
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (s >= nseg) return;
    double2* b0 = sm + (size_t)warp * 2 * P;
    double2* b1 = b0 + P;
    double2* g = vals + s * P;
    for (int i = lane; i < P; i += 32) b0[i] = g[i];
    __syncwarp();
    for (int i = lane; i < P; i += 32) {  // along s
        int a = i % Ps, rest = i / Ps;
        double xr = 0, xi = 0;
        for (int q = 0; q < Ps; ++q) {
            double m = __ldg(Ms + a * Ps + q);
            double2 v = b0[rest * Ps + q];
            xr = fma(m, v.x, xr);
            xi = fma(m, v.y, xi);
        }
        b1[i] = make_double2(xr, xi);
    }
    __syncwarp();
    for (int i = lane; i < P; i += 32) {  // along theta
        int a = i % Ps, b = (i / Ps) % Pa, c = i / (Ps * Pa);
        double xr = 0, xi = 0;
        for (int q = 0; q < Pa; ++q) {
            double m = __ldg(Ma + b * Pa + q);
            double2 v = b1[(c * Pa + q) * Ps + a];
            xr = fma(m, v.x, xr);
            xi = fma(m, v.y, xi);
        }
        b0[i] = make_double2(xr, xi);
    }
    __syncwarp();
    for (int i = lane; i < P; i += 32) {  // along phi
        int ab = i % (Ps * Pa), c = i / (Ps * Pa);
        double xr = 0, xi = 0;
        for (int q = 0; q < Pa; ++q) {
            double m = __ldg(Ma + c * Pa + q);
            double2 v = b0[q * Ps * Pa + ab];
            xr = fma(m, v.x, xr);
            xi = fma(m, v.y, xi);
        }
        g[i] = make_double2(xr, xi);
    }
}

template <int PS, int PA>
__device__ __forceinline__ double2 interp(const double2* C, int Ps, int Pa, double us, double ut, double up) {
    if constexpr (PS > 0) {
        return eval_interp<PS, PA>(C, us, ut, up);
    } else {
        return eval_interp_rt(C, Ps, Pa, us, ut, up);
    }
}

// K6: I(x) += G(x, c_B) Interp_{B, gamma(x)} F_B(x) for every owned source box B
// of which x is a cousin point.  Target-major: one warp per
// (target box T, 32 targets); the cousin relation is symmetric.
template <int PS, int PA>
__global__ void __launch_bounds__(TPB) k_cousin(LevelParams L, const double* __restrict__ px,
                                                const double* __restrict__ py, const double* __restrict__ pz,
                                                const double2* __restrict__ vals, double k, int Ps, int Pa,
                                                double2* out, int* bad) {
    const int P = Ps * Pa * Pa;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t item = wid / L.nsplit_cou;
    const int part = (int)(wid - item * L.nsplit_cou);  // this warp's share of the cousin boxes
    int lane = threadIdx.x & 31;
    if (item >= L.nwitems) return;
    out += (int64_t)part * (L.box_start[L.nbox]);
    int2 it = L.witems[item];
    int T = it.x, l = it.y + lane;
    if (l >= L.box_start[T + 1]) return;
    const double x = px[l], y = py[l], z = pz[l];
    double ar = 0.0, ai = 0.0;
    for (int e = L.cou_off[T] + part; e < L.cou_off[T + 1]; e += L.nsplit_cou) {
        int B = L.cou_idx[e];
        if (B < L.b0 || B >= L.b1) continue;
        double cx, cy, cz;
        box_centre3(L, B, cx, cy, cz);
        Cls c = classify(L, __dsub_rn(x, cx), __dsub_rn(y, cy), __dsub_rn(z, cz));
        int64_t slot = seg_slot(L, B, cell_of(L, c));
        if (slot < 0) {
            atomicOr(bad, 1);
            continue;
        }
        double2 F = interp<PS, PA>(vals + slot * P, Ps, Pa, c.us, c.ut, c.up);
        double sn, cs;
        fm::sincos(k * c.r, &sn, &cs);
        double w = kInv4Pi / c.r;
        double gr = cs * w, gi = sn * w;
        ar = fma(gr, F.x, fma(-gi, F.y, ar));
        ai = fma(gr, F.y, fma(gi, F.x, ai));
    }
    double2 o = out[l];
    out[l] = make_double2(o.x + ar, o.y + ai);
}

// K6, warp-staged and pipelined: target-major as k_cousin (one warp per
// (target box T, 32 targets); the cousin source box B is warp-uniform).  For
// each B the warp finds the distinct (B, cell) segments its targets fall in
// (<= SMAX, leader election with ballots) and copies their coefficient vectors
// into the warp's shared-memory slots with cp.async; every lane then contracts
// from its own slot at the same time (distinct slots sit in disjoint banks), so
// neither the DFMA work nor the loads serialise over distinct segments.  The
// classification of box e+1 and its copies are issued before box e is
// contracted (double-buffered slots), hiding the global-memory latency.
template <int PS, int PA>
struct CousinEv {
    int slot;  // segment slot (-1: none; a level has < 2^31 segments)
    int bi;        // shared-memory slot index, -1 if beyond SMAX (global fallback)
    double gr, gi, us, ut, up;
};

// SPLIT (small problems only, LevelParams::nsplit_cou > 1): nsplit warps per work item.
template <int PS, int PA, bool SPLIT>
// 5 blocks/SM (96 registers) measured best for K6
__global__ void __launch_bounds__(128, 5) k_cousin_ws(LevelParams L, const double* __restrict__ px,
                                                   const double* __restrict__ py, const double* __restrict__ pz,
                                                   const double2* __restrict__ vals, double k, double2* out,
                                                   int* bad, int smax) {
    constexpr int P = PS * PA * PA;
    constexpr int SMAX = P <= 80 ? 4 : (P <= 128 ? 2 : 1);  // static shared memory <= 48 KB per block
    constexpr int SP = P + 2;  // slot stride (double2): 4 slots -> disjoint banks for 16-byte reads
    __shared__ __align__(16) double2 sbuf[TPB / 32][2][SMAX][SP];
    __shared__ __align__(8) unsigned long long sbar[TPB / 32][2];
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int nsplit = SPLIT ? L.nsplit_cou : 1;
    const int64_t item = SPLIT ? wid / nsplit : wid;
    const int part = SPLIT ? (int)(wid - item * nsplit) : 0;  // this warp's share of the cousin boxes
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (item >= L.nwitems) return;  // warp-uniform
    if (SPLIT) out += (int64_t)part * (L.box_start[L.nbox]);  // field part (parts are n apart)
    if (lane == 0) {
        mbar_init(&sbar[w][0], 1);
        mbar_init(&sbar[w][1], 1);
    }
    __syncwarp();
    unsigned phase = 0u;  // bit b: parity of buffer b's next completion
    const int2 it = L.witems[item];
    // items with <= 16 targets run split: lanes l and l + 16 take the same target
    // and alternate cousin boxes (per-lane B; the election spans both halves); the
    // halves are summed at the end (fixed order)
    const int T = it.x, nT = min(32, L.box_start[T + 1] - it.y);
    const bool split = nT <= 16;
    const int half = split ? lane >> 4 : 0, step = split ? 2 : 1;
    const int l = it.y + (split ? (lane & 15) : lane);
    const bool active = l < it.y + nT;
    double x = 0.0, y = 0.0, z = 0.0;
    if (active) {
        x = px[l];
        y = py[l];
        z = pz[l];
    }
    const int e0 = L.cou_off[T], e1 = L.cou_off[T + 1];
    const int stride = step * nsplit, cls = half + step * part;
    auto prep = [&](int i, CousinEv<PS, PA>& v, int buf) {  // iteration i: cousin e0 + stride i + cls
        v.slot = -1;
        v.bi = -1;
        const int e = e0 + stride * i + cls;
        const int B = e < e1 ? L.cou_idx[e] : -1;
        if (active && B >= L.b0 && B < L.b1) {
            double cx, cy, cz;
            box_centre3(L, B, cx, cy, cz);
            const Cls c = classify(L, __dsub_rn(x, cx), __dsub_rn(y, cy), __dsub_rn(z, cz));
            v.slot = (int)seg_slot(L, B, cell_of(L, c));
            if (v.slot < 0) atomicOr(bad, 1);
            double sn, cs;
            fm::sincos(k * c.r, &sn, &cs);
            const double wr = kInv4Pi * c.ir;
            v.gr = cs * wr;
            v.gi = sn * wr;
            v.us = c.us;
            v.ut = c.ut;
            v.up = c.up;
        }
        v.bi = stage_distinct<P>(v.slot, lane, min(SMAX, smax), vals, &sbuf[w][buf][0][0], SP, &sbar[w][buf]);
        IFGF_DCHECK(v.bi < SMAX && v.slot < L.nseg);
    };
    double ar = 0.0, ai = 0.0;
    const int niter = (e1 - e0 + stride - 1) / stride;
    CousinEv<PS, PA> cur, nxt;
    if (niter > 0) prep(0, cur, 0);
    for (int i = 0; i < niter; ++i) {
        if (i + 1 < niter) prep(i + 1, nxt, (i + 1) & 1);
        const int cb = i & 1;
        mbar_wait(&sbar[w][cb], (phase >> cb) & 1u);
        phase ^= 1u << cb;
        if (cur.slot >= 0) {
            double Ts[PS], Tt[2] = {1.0, cur.ut};  // contract_sm_lr needs T_0, T_1 of u_theta only
            cheb_T<PS>(cur.us, Ts);
            const double2 F = cur.bi >= 0 ? contract_sm_lr<PS, PA, false, PA>(&sbuf[w][cb][cur.bi][0], Ts, Tt, cur.up)
                                          : contract_sm_lr<PS, PA>(vals + (int64_t)cur.slot * P, Ts, Tt, cur.up);
            ar = fma(cur.gr, F.x, fma(-cur.gi, F.y, ar));
            ai = fma(cur.gr, F.y, fma(cur.gi, F.x, ai));
        }
        __syncwarp();  // slot buffer (i & 1) is refilled by prep(i + 2)
        cur = nxt;
    }
    if (split) {
        ar += __shfl_down_sync(~0u, ar, 16);
        ai += __shfl_down_sync(~0u, ai, 16);
    }
    if (active && half == 0) {
        const double2 o = out[l];
        out[l] = make_double2(o.x + ar, o.y + ai);
    }
}

// K7, per-evaluation geometry, warp-staged and pipelined (coarse levels, where
// ~1-2 parent segments share a cone cell).  Lane = (parent segment, node) of the
// level, 32 consecutive ones per warp; the warp walks the child octants o = 0..7:
// each lane classifies its node relative to child B_o of its segment, the warp
// elects the distinct child segments (<= SMAX), copies them into its
// shared-memory slots with cp.async and every lane contracts from its slot.
// Octant o+1 is classified and its copies issued before octant o is
// contracted.  Output: node values (the K5 fit runs after).
// pe block: warps and staged child segments per warp step (a warp spans 1-2 parent
// segments, whose nodes hit up to ~6 child cells; static smem <= 48 KB per block)
constexpr int PE_WARPS = 3, PE_SMAX = 6;
template <int PS, int PA>
__global__ void __launch_bounds__(PE_WARPS * 32, 5) k_upward_pe(LevelParams L, LevelParams LP,
                                                      const double2* __restrict__ vals_d, double k, double2* vals_p,
                                                      int* bad, int smax) {
    constexpr int P = PS * PA * PA;
    constexpr int SMAX = P <= 80 ? PE_SMAX : (P <= 128 ? 2 : 1);
    constexpr int SP = P + 2;
    __shared__ __align__(16) double2 sbuf[PE_WARPS][2][SMAX][SP];
    __shared__ __align__(8) unsigned long long sbar[PE_WARPS][2];
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if ((t & ~(int64_t)31) >= LP.nseg * P) return;  // warp-uniform
    if (lane == 0) {
        mbar_init(&sbar[w][0], 1);
        mbar_init(&sbar[w][1], 1);
    }
    __syncwarp();
    unsigned phase = 0u;  // bit b: parity of buffer b's next completion
    const bool active = t < LP.nseg * P;
    const int64_t sp = active ? t / P : 0;
    const int n = active ? (int)(t - sp * P) : 0;
    double off[3] = {0.0, 0.0, 0.0};
    int Q = -1;
    if (active) {
        Q = LP.seg_box[sp];
        node_off(LP, PS, PA, LP.seg_cell[sp], n, off);
    }
    const double rQ = sqrt(fma(off[0], off[0], fma(off[1], off[1], off[2] * off[2])));
    const double hh = 0.5 * L.H;
    struct Ev {
        int slot;  // a level has < 2^31 segments
        int bi;
        double rr, ri, us, ut, up;
    };
    auto prep = [&](int o, Ev& v, int buf) {
        v.slot = -1;
        v.bi = -1;
        int B = active ? LP.child_oct[8 * Q + o] : -1;
        if (B < L.b0 || B >= L.b1) B = -1;
        if (B >= 0) {
            const double dx = (o & 4) ? -hh : hh, dy = (o & 2) ? -hh : hh, dz = (o & 1) ? -hh : hh;
            const Cls c = classify(L, __dadd_rn(off[0], dx), __dadd_rn(off[1], dy), __dadd_rn(off[2], dz));
            v.slot = (int)seg_slot(L, B, cell_of(L, c));
            if (v.slot < 0) atomicOr(bad, 1);
            // r_B - r_Q = (delta.delta + 2 off.delta) / (r_B + r_Q)   (reading R17)
            const double num =
                fma(dx, dx, fma(dy, dy, dz * dz)) + 2.0 * fma(off[0], dx, fma(off[1], dy, off[2] * dz));
            const double ic = rcp_nr(c.r * (c.r + rQ));
            const double diff = num * c.r * ic;
            const double ratio = rQ * (c.r + rQ) * ic;
            double sn, cs;
            fm::sincos(k * diff, &sn, &cs);
            v.rr = ratio * cs;
            v.ri = ratio * sn;
            v.us = c.us;
            v.ut = c.ut;
            v.up = c.up;
        }
        v.bi = stage_distinct<P>(v.slot, lane, min(SMAX, smax), vals_d, &sbuf[w][buf][0][0], SP, &sbar[w][buf]);
        IFGF_DCHECK(v.bi < SMAX && v.slot < L.nseg);
    };
    // octants with a child for some lane of the warp (the others are skipped)
    unsigned mymask = 0u;
    if (active)
        for (int o = 0; o < 8; ++o) {
            const int B = LP.child_oct[8 * Q + o];
            if (B >= L.b0 && B < L.b1) mymask |= 1u << o;
        }
    unsigned omask = __reduce_or_sync(~0u, mymask);
    double ar = 0.0, ai = 0.0;
    Ev cur, nxt;
    int oc = omask ? __ffs(omask) - 1 : 8;
    if (oc < 8) {
        omask &= omask - 1;
        prep(oc, cur, 0);
    }
    for (int it = 0; oc < 8; ++it) {
        const int on = omask ? __ffs(omask) - 1 : 8;
        if (on < 8) {
            omask &= omask - 1;
            prep(on, nxt, (it + 1) & 1);
        }
        const int cb = it & 1;
        mbar_wait(&sbar[w][cb], (phase >> cb) & 1u);
        phase ^= 1u << cb;
        if (cur.slot >= 0) {
            double Ts[PS], Tt[PA];
            cheb_T<PS>(cur.us, Ts);
            cheb_T<PA>(cur.ut, Tt);
            const double2 F = cur.bi >= 0 ? contract_sm_lr<PS, PA, false, PA>(&sbuf[w][cb][cur.bi][0], Ts, Tt, cur.up)
                                          : contract_sm_lr<PS, PA, true>(vals_d + (int64_t)cur.slot * P, Ts, Tt, cur.up);
            ar = fma(cur.rr, F.x, fma(-cur.ri, F.y, ar));
            ai = fma(cur.rr, F.y, fma(cur.ri, F.x, ai));
        }
        __syncwarp();  // slot buffer cb is refilled two steps ahead
        cur = nxt;
        oc = on;
    }
    if (active) vals_p[t] = make_double2(ar, ai);
}

// K7: V_Q[gamma', y] = sum over owned children B of Q of
//   Interp_{B, gamma(y)} F_B(y) * G(y, c_B)/G(y, c_Q)
// one thread per (parent segment, node); y - c_B = off + delta, delta = +-H_d/2.
template <int PS, int PA>
__global__ void __launch_bounds__(TPB, 4) k_upward(LevelParams L, LevelParams LP, const double2* __restrict__ vals_d,
                                                double k, int Ps, int Pa, double2* vals_p, int* bad) {
    const int P = Ps * Pa * Pa;
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= LP.nseg * P) return;
    int64_t sp = t / P;
    int n = (int)(t - sp * P);
    int Q = LP.seg_box[sp];
    double off[3];
    node_off(LP, Ps, Pa, LP.seg_cell[sp], n, off);
    const double rQ = sqrt(fma(off[0], off[0], fma(off[1], off[1], off[2] * off[2])));
    const double hh = 0.5 * L.H;
    double ar = 0.0, ai = 0.0;
    for (int B = LP.child_start[Q]; B < LP.child_start[Q + 1]; ++B) {
        if (B < L.b0 || B >= L.b1) continue;
        double dx = (L.box_ijk[3 * B] & 1) ? -hh : hh, dy = (L.box_ijk[3 * B + 1] & 1) ? -hh : hh,
               dz = (L.box_ijk[3 * B + 2] & 1) ? -hh : hh;
        Cls c = classify(L, __dadd_rn(off[0], dx), __dadd_rn(off[1], dy), __dadd_rn(off[2], dz));
        int64_t slot = seg_slot(L, B, cell_of(L, c));
        if (slot < 0) {
            atomicOr(bad, 1);
            continue;
        }
        double2 F;
        if constexpr (PS > 0) {
            double Ts[PS], Tt[PA];
            cheb_T<PS>(c.us, Ts);
            cheb_T<PA>(c.ut, Tt);
            F = contract_sm_lr<PS, PA, true>(vals_d + slot * P, Ts, Tt, c.up);
        } else {
            F = interp<PS, PA>(vals_d + slot * P, Ps, Pa, c.us, c.ut, c.up);
        }
        // r_B - r_Q = (delta.delta + 2 off.delta) / (r_B + r_Q)   (reading R17)
        double num = fma(dx, dx, fma(dy, dy, dz * dz)) + 2.0 * fma(off[0], dx, fma(off[1], dy, off[2] * dz));
        double diff = num / (c.r + rQ);
        double ratio = rQ / c.r;
        double sn, cs;
        fm::sincos(k * diff, &sn, &cs);
        double gr = ratio * cs, gi = ratio * sn;
        ar = fma(gr, F.x, fma(-gi, F.y, ar));
        ai = fma(gr, F.y, fma(gi, F.x, ai));
    }
    vals_p[sp * P + n] = make_double2(ar, ai);
}

// ---------------------------------------------------------------------------
// K7, cell-grouped + shared-memory staged.  Per (chunk, octant) the nodes of
// the block map to a handful (U) of child cells; those U child segments are
// copied into shared memory with cp.async (double-buffered over the chunk's
// segments) and every thread contracts from shared memory.  This turns the
// per-evaluation chain of dependent global loads into one bulk, fully
// overlapped copy per (segment, octant).

template <int PS, int PA>
struct StagedCfg {
    static constexpr int P = PS * PA * PA;
    static constexpr int NT = ((P + 31) / 32) * 32;
    static constexpr int MAXU = P <= 80 ? 12 : 8;
    static constexpr size_t smem = (size_t)(2 * MAXU * P + kChunk * NT) * sizeof(double2);
};

template <int PS, int PA>
__global__ void __launch_bounds__(128, 3) k_upward_s(LevelParams L, LevelParams LP, const double2* __restrict__ vals_d,
                                                     double k, const double* __restrict__ Ms,
                                                     const double* __restrict__ Ma, double2* vals_p, int* bad) {
    using Cfg = StagedCfg<PS, PA>;
    constexpr int P = Cfg::P, NT = Cfg::NT, MAXU = Cfg::MAXU, CH = kChunk;
    extern __shared__ double2 dsm[];
    double2* sh_coef = dsm;                 // [2][MAXU][P]
    double2* sh_acc = dsm + 2 * MAXU * P;   // [CH][NT]
    __shared__ int sh_seg[CH];
    __shared__ int sh_child[CH][8];
    __shared__ unsigned sh_omask;
    __shared__ int sh_cell[NT];
    __shared__ unsigned char sh_lead[NT];
    __shared__ int sh_ucell[MAXU];
    __shared__ int sh_slot[CH][MAXU];
    __shared__ int sh_jl[CH];
    __shared__ int sh_nj;
    const int tid = threadIdx.x;
    const int64_t c = blockIdx.x;
    const int s0 = LP.chunk_start[c];
    const int s1 = (c + 1 < LP.nchunk) ? LP.chunk_start[c + 1] : (int)LP.nseg;
    const int cnt = min(CH, s1 - s0);
    if (tid == 0) sh_omask = 0u;
    __syncthreads();
    for (int t = tid; t < CH * 8; t += NT) {
        int j = t >> 3, o = t & 7;
        int B = -1;
        if (j < cnt) {
            int seg = LP.cell_seg[s0 + j];
            if (o == 0) sh_seg[j] = seg;
            B = LP.child_oct[8 * LP.seg_box[seg] + o];
            if (B < L.b0 || B >= L.b1) B = -1;
            if (B >= 0) atomicOr(&sh_omask, 1u << o);
        }
        sh_child[j][o] = B;
    }
    __syncthreads();
    const int n = tid;
    const bool active = n < P;
    const unsigned omask = sh_omask;
    double off[3] = {0.0, 0.0, 0.0};
    if (active) node_off(LP, PS, PA, LP.seg_cell[sh_seg[0]], n, off);
    const double rQ = sqrt(fma(off[0], off[0], fma(off[1], off[1], off[2] * off[2])));
    const double hh = 0.5 * L.H;
    for (int j = 0; j < cnt; ++j) sh_acc[j * NT + n] = make_double2(0.0, 0.0);
    for (int o = 0; o < 8; ++o) {
        if (!((omask >> o) & 1u)) continue;
        const double dx = (o & 4) ? -hh : hh, dy = (o & 2) ? -hh : hh, dz = (o & 1) ? -hh : hh;
        double rr = 0.0, ri = 0.0, up = 0.0;
        double Ts[PS], Tt[PA];
        int cellc = -1;
        if (active) {
            Cls cl = classify(L, __dadd_rn(off[0], dx), __dadd_rn(off[1], dy), __dadd_rn(off[2], dz));
            cellc = (int)cell_of(L, cl);
            double num = fma(dx, dx, fma(dy, dy, dz * dz)) + 2.0 * fma(off[0], dx, fma(off[1], dy, off[2] * dz));
            double diff = num / (cl.r + rQ);
            double ratio = rQ / cl.r;
            double sn, cs;
            fm::sincos(k * diff, &sn, &cs);
            rr = ratio * cs;
            ri = ratio * sn;
            cheb_T<PS>(cl.us, Ts);
            cheb_T<PA>(cl.ut, Tt);
            up = cl.up;
        }
        sh_cell[n] = cellc;
        __syncthreads();
        // distinct child cells of this octant: leader = first node with the cell
        int first = n;
        if (active)
            for (int m = 0; m < n; ++m)
                if (sh_cell[m] == cellc) {
                    first = m;
                    break;
                }
        const bool lead = active && first == n;
        sh_lead[n] = lead ? 1 : 0;
        __syncthreads();
        int myu = 0;
        if (active)
            for (int m = 0; m < first; ++m) myu += sh_lead[m];
        if (lead && myu < MAXU) sh_ucell[myu] = cellc;
        const int U = __syncthreads_count(lead);
        if (U > MAXU) {
            // rare: too many distinct cells to stage; evaluate from global memory
            if (active)
                for (int j = 0; j < cnt; ++j) {
                    const int B = sh_child[j][o];
                    if (B < 0) continue;
                    const int64_t slot = seg_slot(L, B, cellc);
                    if (slot < 0) {
                        atomicOr(bad, 1);
                        continue;
                    }
                    double2 F = contract<PS, PA>(vals_d + slot * P, Ts, Tt, up);
                    double2 acc = sh_acc[j * NT + n];
                    acc.x = fma(rr, F.x, fma(-ri, F.y, acc.x));
                    acc.y = fma(rr, F.y, fma(ri, F.x, acc.y));
                    sh_acc[j * NT + n] = acc;
                }
            __syncthreads();
            continue;
        }
        for (int t = tid; t < cnt * U; t += NT) {
            const int j = t / U, u = t - (t / U) * U;
            const int B = sh_child[j][o];
            int sl = -1;
            if (B >= 0) {
                int64_t s = seg_slot(L, B, sh_ucell[u]);
                if (s < 0) atomicOr(bad, 1);
                sl = (int)s;
            }
            sh_slot[j][u] = sl;
        }
        if (tid == 0) {
            int nj = 0;
            for (int j = 0; j < cnt; ++j)
                if (sh_child[j][o] >= 0) sh_jl[nj++] = j;
            sh_nj = nj;
        }
        __syncthreads();
        const int nj = sh_nj;
        auto issue = [&](int q, int buf) {
            const int j = sh_jl[q];
            double2* dst = sh_coef + buf * MAXU * P;
            for (int t = tid; t < U * P; t += NT) {
                const int u = t / P, i = t - (t / P) * P;
                const int sl = sh_slot[j][u];
                if (sl >= 0) cp_async16(dst + t, vals_d + (int64_t)sl * P + i);
                else dst[t] = make_double2(0.0, 0.0);
            }
            cp_async_commit();
        };
        if (nj > 0) issue(0, 0);
        for (int q = 0; q < nj; ++q) {
            if (q + 1 < nj) {
                issue(q + 1, (q + 1) & 1);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();
            if (active) {
                const int j = sh_jl[q];
                double2 F = contract_sm<PS, PA>(sh_coef + (q & 1) * MAXU * P + myu * P, Ts, Tt, up);
                double2 acc = sh_acc[j * NT + n];
                acc.x = fma(rr, F.x, fma(-ri, F.y, acc.x));
                acc.y = fma(rr, F.y, fma(ri, F.x, acc.y));
                sh_acc[j * NT + n] = acc;
            }
            __syncthreads();
        }
    }
    // Fused K5: node values -> tensor Chebyshev coefficients (reading R1), three
    // separable passes through shared memory; thread n produces coefficient n.
    double ms[PS], mt[PA], mp[PA];
    const int ia = n % PS, ib = (n / PS) % PA, ic = n / (PS * PA);
    if (active) {
#pragma unroll
        for (int q = 0; q < PS; ++q) ms[q] = __ldg(Ms + ia * PS + q);
#pragma unroll
        for (int q = 0; q < PA; ++q) {
            mt[q] = __ldg(Ma + ib * PA + q);
            mp[q] = __ldg(Ma + ic * PA + q);
        }
    }
    double2* tA = sh_coef;
    double2* tB = sh_coef + P;
    __syncthreads();
    for (int j = 0; j < cnt; ++j) {
        const double2* V = sh_acc + j * NT;
        if (active) {  // along s
            double xr = 0.0, xi = 0.0;
#pragma unroll
            for (int q = 0; q < PS; ++q) {
                double2 v = V[(ic * PA + ib) * PS + q];
                xr = fma(ms[q], v.x, xr);
                xi = fma(ms[q], v.y, xi);
            }
            tA[n] = make_double2(xr, xi);
        }
        __syncthreads();
        if (active) {  // along theta
            double xr = 0.0, xi = 0.0;
#pragma unroll
            for (int q = 0; q < PA; ++q) {
                double2 v = tA[(ic * PA + q) * PS + ia];
                xr = fma(mt[q], v.x, xr);
                xi = fma(mt[q], v.y, xi);
            }
            tB[n] = make_double2(xr, xi);
        }
        __syncthreads();
        if (active) {  // along phi
            double xr = 0.0, xi = 0.0;
#pragma unroll
            for (int q = 0; q < PA; ++q) {
                double2 v = tB[(q * PA + ib) * PS + ia];
                xr = fma(mp[q], v.x, xr);
                xi = fma(mp[q], v.y, xi);
            }
            vals_p[(int64_t)sh_seg[j] * P + n] = make_double2(xr, xi);
        }
    }
}

// FP64 tensor-core MMA: D(8x8) += A(8x4) B(4x8), lane holds A[gid][tig], B[tig][gid],
// D[gid][2 tig + {0,1}] (gid = lane / 4, tig = lane % 4).
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// K5 fit of cnt segments' node values held in shared memory, IN PLACE (reading R1):
// three separable passes, each thread transforming whole 1-D lines (P_s values
// along s, P_ang along theta / phi) in registers, so no temporary buffer and only
// three barriers; the phi pass writes the coefficients to out[seg[j] * P + i].
template <int PS, int PA>
__device__ __forceinline__ void fit_lines_inplace(double2* V, int cnt, const int* seg, const double* Ms,
                                                  const double* Ma, double2* out, int tid, int nt) {
    constexpr int P = PS * PA * PA;
    double ms[PS * PS], ma[PA * PA];
#pragma unroll
    for (int i = 0; i < PS * PS; ++i) ms[i] = __ldg(Ms + i);
#pragma unroll
    for (int i = 0; i < PA * PA; ++i) ma[i] = __ldg(Ma + i);
    __syncthreads();
    for (int t = tid; t < cnt * PA * PA; t += nt) {  // along s: line (j, b, c)
        const int j = t / (PA * PA), bc = t - j * (PA * PA);
        double2* v = V + j * P + bc * PS;
        double2 x[PS];
#pragma unroll
        for (int q = 0; q < PS; ++q) x[q] = v[q];
#pragma unroll
        for (int a = 0; a < PS; ++a) {
            double xr = 0.0, xi = 0.0;
#pragma unroll
            for (int q = 0; q < PS; ++q) {
                xr = fma(ms[a * PS + q], x[q].x, xr);
                xi = fma(ms[a * PS + q], x[q].y, xi);
            }
            v[a] = make_double2(xr, xi);
        }
    }
    __syncthreads();
    for (int t = tid; t < cnt * PS * PA; t += nt) {  // along theta: line (j, a, c)
        const int j = t / (PS * PA), r = t - j * (PS * PA), c = r / PS, a = r - c * PS;
        double2* v = V + j * P + c * PA * PS + a;
        double2 x[PA];
#pragma unroll
        for (int q = 0; q < PA; ++q) x[q] = v[q * PS];
#pragma unroll
        for (int b = 0; b < PA; ++b) {
            double xr = 0.0, xi = 0.0;
#pragma unroll
            for (int q = 0; q < PA; ++q) {
                xr = fma(ma[b * PA + q], x[q].x, xr);
                xi = fma(ma[b * PA + q], x[q].y, xi);
            }
            v[b * PS] = make_double2(xr, xi);
        }
    }
    __syncthreads();
    for (int t = tid; t < cnt * PS * PA; t += nt) {  // along phi: line (j, a, b) -> global
        const int j = t / (PS * PA), ab = t - j * (PS * PA);
        const double2* v = V + j * P + ab;
        double2 x[PA];
#pragma unroll
        for (int q = 0; q < PA; ++q) x[q] = v[q * PS * PA];
        double2* o = out + (int64_t)seg[j] * P + ab;
#pragma unroll
        for (int c = 0; c < PA; ++c) {
            double xr = 0.0, xi = 0.0;
#pragma unroll
            for (int q = 0; q < PA; ++q) {
                xr = fma(ma[c * PA + q], x[q].x, xr);
                xi = fma(ma[c * PA + q], x[q].y, xi);
            }
            o[c * PS * PA] = make_double2(xr, xi);
        }
    }
}

// K5 for the levels whose K7 writes node values (per-evaluation kernel, leaf):
// block = 8 consecutive segments staged in shared memory, in-place line passes.
template <int PS, int PA>
__global__ void __launch_bounds__(64) k_fit_lines(int64_t nseg, const double* __restrict__ Ms,
                                                  const double* __restrict__ Ma, double2* vals) {
    constexpr int P = PS * PA * PA, NSB = 4;
    __shared__ double2 sv[NSB * P];
    __shared__ int sseg[NSB];
    const int64_t s0 = (int64_t)blockIdx.x * NSB;
    const int cnt = (int)min((int64_t)NSB, nseg - s0);
    for (int t = threadIdx.x; t < cnt * P; t += blockDim.x) sv[t] = vals[s0 * P + t];
    if (threadIdx.x < NSB) sseg[threadIdx.x] = (int)(s0 + threadIdx.x);
    fit_lines_inplace<PS, PA>(sv, cnt, sseg, Ms, Ma, vals, threadIdx.x, blockDim.x);
}

// ---------------------------------------------------------------------------
// K7 on the FP64 tensor core, large cell chunks (fine levels).
//
// Within a chunk of <= J parent segments sharing cone cell gamma' and a child
// octant o, the child-relative geometry of parent node n (child cell u_n, local
// coordinates, recentering factor rec_n = G(y,c_B)/G(y,c_Q)) is box-independent,
// so for every child cell u
//     V[j][n] += rec_n * sum_i W[n][i] C[B_{j,o}, u][i]       (u_n == u)
// with the tensor Chebyshev basis W[n][i] = T_a(u_s) T_b(u_theta) T_c(u_phi)
// (i = (c P_ang + b) P_s + a).  That is a dense (nodes x coefficients) x
// (coefficients x segments) product: DMMA m8n8k4 tiles with rows = nodes
// sorted by child cell, columns = the segments whose box has child o
// (compacted per octant), k = coefficient index; real and imaginary parts share
// the W fragment.  Per block:
//   phase 0  segments, children by octant, per-octant compaction (warp ballots)
//   phase 1  geometry of all (octant, node) pairs (classification contract)
//   phase 2  per octant (one warp each): distinct child cells, node sort by cell
//   phase 3  (octant, cell, segment) -> child segment slot (bitmap rank)
//   phase 4  per octant: W_o into shared memory, then tasks (segment tile, cell):
//            the warp loads the 8 child coefficient vectors once (B fragments in
//            registers) and sweeps the node tiles of that cell (A fragments from
//            shared memory); rows of other cells in a boundary tile are computed
//            and discarded.  Each V entry has one writer per octant and octants
//            are summed in a fixed order (deterministic, no atomics).
//   phase 5  fused K5 fit of the chunk's node values -> Chebyshev coefficients.
template <int PS, int PA>
struct TcCfg {
    static constexpr int P = PS * PA * PA;
    static constexpr int KS = (P + 3) / 4;   // k-steps of 4
    static constexpr int NR = (P + 7) / 8;   // row (node) tiles of 8
    static constexpr int NW = NR * 8;
    // W row stride (doubles): == 4 or 12 mod 16 makes the 8x4 A-fragment loads of
    // each half-warp hit 16 distinct 8-byte bank pairs
    static constexpr int KP = ((4 * KS) % 16 == 4 || (4 * KS) % 16 == 12) ? 4 * KS : 4 * KS + 4;
    static constexpr int J = kChunkTC;
    static constexpr int UM = 8;              // distinct child cells per octant with staged slots
    static constexpr int NT = 384;                 // 12 warps (measured best: 8 with prefetch, 16 spill)
    static constexpr bool PREFETCH = NT <= 256;  // register double buffer of B fragments
    static constexpr int NWARP = NT / 32;
    static constexpr int R = (NW + 31) / 32;
    static constexpr int FG = 16;             // fit group (segments)
    static constexpr size_t a16(size_t x) { return (x + 15) / 16 * 16; }
    static constexpr size_t oV = 0;                                       // double2 [J][P]
    static constexpr size_t oW = a16(oV + (size_t)J * P * 16);            // double [NW][KP]
    static constexpr size_t oG = a16(oW + (size_t)NW * KP * 8);           // double [8][NW][5]
    static constexpr size_t oU = a16(oG + (size_t)8 * NW * 5 * 8);        // int [8][NW]
    static constexpr size_t oSlot = a16(oU + (size_t)8 * NW * 4);         // int [8][UM][J]
    static constexpr size_t oChild = a16(oSlot + (size_t)8 * UM * J * 4); // int [8][J]
    static constexpr size_t oSeg = a16(oChild + (size_t)8 * J * 4);       // int [J]
    static constexpr size_t oUcell = a16(oSeg + (size_t)J * 4);           // int [8][UM]
    static constexpr size_t oMisc = a16(oUcell + (size_t)8 * UM * 4);     // int U[8], nO[8]
    static constexpr size_t oPst = a16(oMisc + 16 * 4);                   // u8 [8][UM + 1] run starts
    static constexpr size_t oOrd = a16(oPst + (size_t)8 * (UM + 1));      // u8 [8][NW]
    static constexpr size_t oJl = a16(oOrd + (size_t)8 * NW);             // u8 [8][J]
    static constexpr size_t oFit = a16(oJl + (size_t)8 * J);              // double Ms, Ma
    static constexpr size_t smem = a16(oFit + (size_t)(PS * PS + PA * PA) * 8);
    static_assert(NWARP >= 8, "phase 0/2 map one warp per octant");
    static_assert(2 * FG * P * 16 <= NW * KP * 8, "fit temporaries live in the W buffer");
    static_assert(J <= 255 && NW <= 255, "u8 indices");
};

template <int PS, int PA>
__global__ void __launch_bounds__(TcCfg<PS, PA>::NT, 1) k_upward_tc(LevelParams L, LevelParams LP, const double2* __restrict__ vals_d,
                                                      double k, const double* __restrict__ Ms,
                                                      const double* __restrict__ Ma, double2* vals_p, int* bad,
                                                      int umax, const double2* __restrict__ zseg,
                                                      unsigned long long* __restrict__ phase_clk) {
    using C = TcCfg<PS, PA>;
    // optional per-phase clock accounting (env IFGF_PHASE_PROF): thread 0 adds the
    // cycles since the previous mark to phase_clk[i]
    long long t_mark = clock64();
    auto mark = [&](int i) {
        if (phase_clk && threadIdx.x == 0) {
            const long long t = clock64();
            atomicAdd(phase_clk + i, (unsigned long long)(t - t_mark));
            t_mark = t;
        }
    };
    constexpr int P = C::P, KS = C::KS, NW = C::NW, KP = C::KP, J = C::J, UM = C::UM, NT = C::NT,
                  NWARP = C::NWARP, R = C::R, FG = C::FG;
    extern __shared__ __align__(16) unsigned char smraw[];
    double2* sV = reinterpret_cast<double2*>(smraw + C::oV);
    double* sW = reinterpret_cast<double*>(smraw + C::oW);
    double* sG = reinterpret_cast<double*>(smraw + C::oG);
    int* sU = reinterpret_cast<int*>(smraw + C::oU);
    int* sSlot = reinterpret_cast<int*>(smraw + C::oSlot);
    int* sChild = reinterpret_cast<int*>(smraw + C::oChild);
    int* sSeg = reinterpret_cast<int*>(smraw + C::oSeg);
    int* sUcell = reinterpret_cast<int*>(smraw + C::oUcell);
    int* sUn = reinterpret_cast<int*>(smraw + C::oMisc);
    int* sNo = sUn + 8;
    unsigned char* sPst = smraw + C::oPst;
    unsigned char* sOrd = smraw + C::oOrd;
    unsigned char* sJl = smraw + C::oJl;
    double* sMs = reinterpret_cast<double*>(smraw + C::oFit);
    double* sMa = sMs + PS * PS;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t c = LP.chunk_order ? LP.chunk_order[blockIdx.x] : blockIdx.x;
    const int s0 = LP.chunk_start[c];
    const int s1 = (c + 1 < LP.nchunk) ? LP.chunk_start[c + 1] : (int)LP.nseg;
    const int cnt = min(J, s1 - s0);

    // per-octant task tables (phase 2): r -> (cell << 8 | node tile), r -> end of the cell's run
    __shared__ unsigned short sTk[8][C::NR + C::UM + 1];
    __shared__ unsigned char sGe[8][C::NR + C::UM + 1];
    __shared__ int sS[8];

    // ---- phase 0
    __shared__ int sBox[J];
    __shared__ unsigned char sQd[J];  // quarter turns of segment j's cell from the representative
    for (int j = tid; j < J; j += NT) {
        int seg = -1, box = -1, qd = 0;
        if (j < cnt) {
            seg = LP.cell_seg[s0 + j];
            box = LP.seg_box[seg];
            qd = sym_quarter(LP, LP.seg_cell[seg]);
        }
        sSeg[j] = seg;
        sBox[j] = box;
        sQd[j] = (unsigned char)qd;
    }
    for (int t = tid; t < J * P; t += NT) sV[t] = make_double2(0.0, 0.0);
    __syncthreads();
    // children by octant: the two rounds' loads are issued together
    for (int t0 = tid; t0 < 8 * J; t0 += 2 * NT) {
        int Bv[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int t = t0 + h * NT;
            Bv[h] = -1;
            if (t < 8 * J) {
                const int o = t / J, j = t - o * J;
                if (sBox[j] >= 0) Bv[h] = LP.child_oct[8 * sBox[j] + rot_oct(o, sQd[j])];
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int t = t0 + h * NT;
            if (t < 8 * J) sChild[t] = (Bv[h] < L.b0 || Bv[h] >= L.b1) ? -1 : Bv[h];
        }
    }
    __syncthreads();
    if (warp < 8) {
        const int o = warp;
        int base = 0;
        for (int j0 = 0; j0 < J; j0 += 32) {
            const int j = j0 + lane;
            const bool pr = j < J && sChild[o * J + j] >= 0;
            const unsigned b = __ballot_sync(~0u, pr);
            if (pr) sJl[o * J + base + __popc(b & lt)] = (unsigned char)j;
            base += __popc(b);
        }
        if (lane == 0) sNo[o] = base;
    }
    __syncthreads();
    if (phase_clk && tid == 0) atomicAdd(phase_clk + 13, 1ull);
    mark(0);

    // ---- phase 1: geometry of (octant, node)
    const int cellp = sym_rep(LP, LP.seg_cell[sSeg[0]]);  // the chunk's (representative) parent cell
    const double hh = 0.5 * L.H;
    for (int t = tid; t < 8 * NW; t += NT) {
        const int o = t / NW, n = t - o * NW;
        int u = INT_MAX;
        if (n < P && sNo[o] > 0) {
            double off[3];
            node_off(LP, PS, PA, cellp, n, off);
            const double rQ = sqrt(fma(off[0], off[0], fma(off[1], off[1], off[2] * off[2])));
            const double dx = (o & 4) ? -hh : hh, dy = (o & 2) ? -hh : hh, dz = (o & 1) ? -hh : hh;
            const double vx = __dadd_rn(off[0], dx), vy = __dadd_rn(off[1], dy);
            const Cls cl = classify(L, vx, vy, __dadd_rn(off[2], dz));
            u = (int)cell_of(L, cl);
            if (LP.sym && vx == 0.0 && vy == 0.0) u |= kPoleFlag;  // pole: sector 0 in every rotation
            // r_B - r_Q = (delta.delta + 2 off.delta) / (r_B + r_Q)   (reading R17)
            const double num = fma(dx, dx, fma(dy, dy, dz * dz)) + 2.0 * fma(off[0], dx, fma(off[1], dy, off[2] * dz));
            const double ic = rcp_nr(cl.r * (cl.r + rQ));
            const double diff = num * cl.r * ic;
            const double ratio = rQ * (cl.r + rQ) * ic;
            double sn, cs;
            fm::sincos(k * diff, &sn, &cs);
            double* g = sG + (size_t)t * 5;
            g[0] = cl.us;
            g[1] = cl.ut;
            g[2] = cl.up;
            g[3] = ratio * cs;
            g[4] = ratio * sn;
        }
        sU[t] = u;
    }
    __syncthreads();
    mark(1);

    // ---- phase 2: per octant (warp): distinct child cells ascending, stable node
    // sort by cell; the nodes of cell index ui occupy sorted positions
    // [pst[ui], pst[ui + 1])
    if (warp < 8) {
        const int o = warp;
        int uv[R];
        bool done[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int n = lane + 32 * r;
            uv[r] = n < NW ? sU[o * NW + n] : INT_MAX;
            done[r] = !(n < P) || uv[r] == INT_MAX;
        }
        int base = 0, U = 0;
        while (true) {
            int m = INT_MAX;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (!done[r]) m = min(m, uv[r]);
            m = __reduce_min_sync(~0u, m);
            if (m == INT_MAX) break;
            if (lane == 0 && U <= UM) sPst[o * (UM + 1) + U] = (unsigned char)base;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const bool hit = !done[r] && uv[r] == m;
                const unsigned b = __ballot_sync(~0u, hit);
                if (hit) {
                    const int pos = base + __popc(b & lt);
                    sOrd[o * NW + pos] = (unsigned char)(lane + 32 * r);
                    done[r] = true;
                }
                base += __popc(b);
            }
            if (lane == 0 && U < UM) sUcell[o * UM + U] = m;
            ++U;
        }
        if (lane == 0 && U <= UM) sPst[o * (UM + 1) + U] = (unsigned char)base;
        for (int pos = base + lane; pos < NW; pos += 32) {
            sOrd[o * NW + pos] = (unsigned char)pos;
        }
        if (lane == 0) sUn[o] = U;
        // task table of the octant: the node tiles of each child cell in cell order,
        // r -> (cell, tile) and r -> end of that cell's run (lane u = cell u)
        __syncwarp();
        if (U <= UM) {
            const unsigned char* ps = sPst + o * (UM + 1);
            const int nt_u = lane < U ? ((ps[lane + 1] - 1) >> 3) - (ps[lane] >> 3) + 1 : 0;
            int r0 = nt_u;
#pragma unroll
            for (int sh = 1; sh < 32; sh <<= 1) {
                const int v = __shfl_up_sync(~0u, r0, sh);
                if (lane >= sh) r0 += v;
            }
            const int rend = r0;  // inclusive prefix: end of this cell's run
            r0 -= nt_u;
            if (lane < U)
                for (int q = 0; q < nt_u; ++q) {
                    sTk[o][r0 + q] = (unsigned short)((lane << 8) | ((ps[lane] >> 3) + q));
                    sGe[o][r0 + q] = (unsigned char)rend;
                }
            if (lane == 31) sS[o] = rend;
        }
    }
    __syncthreads();
    mark(2);

    // ---- phase 3: child segment slots of the staged (octant, cell, compacted
    // segment) triples only (tasks treat columns q >= n_o as absent); two items
    // per thread in flight
    {
        __shared__ int sPre[9];
        if (tid == 0) {
            int acc = 0;
            for (int o = 0; o < 8; ++o) {
                sPre[o] = acc;
                if (sUn[o] <= umax) acc += sUn[o] * sNo[o];
            }
            sPre[8] = acc;
        }
        __syncthreads();
        const int tot = sPre[8];
        for (int t0 = tid; t0 < tot; t0 += 2 * NT) {
            int idx[2], Bv[2], cellv[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int t = t0 + h * NT;
                idx[h] = -1;
                if (t < tot) {
                    int o = 0;
                    while (o < 7 && t >= sPre[o + 1]) ++o;
                    const int rem = t - sPre[o], no = sNo[o];
                    const int ui = rem / no, q = rem - ui * no;
                    idx[h] = (o * UM + ui) * J + q;
                    const int j = sJl[o * J + q];
                    Bv[h] = sChild[o * J + j];
                    cellv[h] = sym_cell(L, sUcell[o * UM + ui], sQd[j]);
                }
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (idx[h] < 0) continue;
                const int64_t s64 = seg_slot(L, Bv[h], cellv[h]);
                if (s64 < 0) atomicOr(bad, 1);
                sSlot[idx[h]] = (int)s64;
            }
        }
    }
    // (no barrier: the first octant's basis build below does not read the slots,
    // and its closing barrier orders them before the first DMMA task)
    mark(3);

    // ---- phase 4: per octant, W_o then DMMA tasks
    const int gid = lane >> 2, tig = lane & 3;
    long long t_task0 = 0;
    // zero the basis padding (rows P..NW-1, columns P..KP-1) once; the octants
    // only rewrite the P x P block (the first barrier below orders it)
    for (int t = tid; t < NW * KP; t += NT) {
        const int pos = t / KP, kk = t - pos * KP;
        if (pos >= P || kk >= P) sW[t] = 0.0;
    }
    for (int o = 0; o < 8; ++o) {
        const int no = sNo[o];
        if (no == 0) continue;
        const int U = sUn[o];
        const double* g0 = sG + (size_t)o * NW * 5;
        if (U <= umax) {
            // basis rows of the P real nodes (P * PA items: one round for NT >= 375);
            // the padding rows and columns were zeroed once per chunk
            for (int t = tid; t < P * PA; t += NT) {
                const int pos = t / PA, cc = t - pos * PA;
                double* wrow = sW + pos * KP;
                const double* g = g0 + (int)sOrd[o * NW + pos] * 5;
                double Ts[PS], Tt[PA];
                cheb_T<PS>(g[0], Ts);
                cheb_T<PA>(g[1], Tt);
                const double up = g[2];
                double tm1 = 1.0, tp = up;
                if (cc == 0) tp = 1.0;
                for (int i = 2; i <= cc; ++i) {
                    const double tn = fma(2.0 * up, tp, -tm1);
                    tm1 = tp;
                    tp = tn;
                }
#pragma unroll
                for (int b = 0; b < PA; ++b) {
                    const double tb = Tt[b] * tp;
#pragma unroll
                    for (int a = 0; a < PS; ++a) wrow[(cc * PA + b) * PS + a] = Ts[a] * tb;
                }
            }
            __syncthreads();
            mark(4);
            t_task0 = clock64();
            // Tasks (segment tile st, child cell ui, node tile) enumerated st-major;
            // warp w takes the contiguous range [w T / NWARP, (w+1) T / NWARP), so
            // consecutive tasks mostly share (st, ui) and its B fragments stay in
            // registers; the next group's B fragments are prefetched while the
            // current group's node tiles run (register double buffer).
            const int nst = (no + 7) >> 3;
            const unsigned char* pst = sPst + o * (UM + 1);
            const int S = sS[o];
            const int T = nst * S;
            if (phase_clk && tid == 0) {  // shape counters: cells, node tiles, segments, octants
                atomicAdd(phase_clk + 9, (unsigned long long)U);
                atomicAdd(phase_clk + 10, (unsigned long long)S);
                atomicAdd(phase_clk + 11, (unsigned long long)no);
                atomicAdd(phase_clk + 12, 1ull);
            }
            const int tau0 = (int)((int64_t)warp * T / NWARP), tau1 = (int)((int64_t)(warp + 1) * T / NWARP);
            // decode task tau -> (segment tile, child cell, its node tile, end of the
            // (segment tile, cell) group) from the octant's task table
            auto decode = [&](int tau, int& st, int& ui, int& tile, int& gend) {
                st = tau / S;
                const int r = tau - st * S;
                const int e = sTk[o][r];
                ui = e >> 8;
                tile = e & 0xFF;
                gend = min(tau1, st * S + (int)sGe[o][r]);
            };
            auto load_b = [&](int st, int ui, double2* bb) {
                const int q = st * 8 + gid;
                IFGF_DCHECK(ui >= 0 && ui < UM && st >= 0 && st * 8 < J);
                const int sl = q < no ? sSlot[(o * UM + ui) * J + q] : -1;
                IFGF_DCHECK(sl < L.nseg);
                const double2* cp = sl >= 0 ? vals_d + (int64_t)sl * P : zseg;
#pragma unroll
                for (int ks = 0; ks < KS; ++ks)  // k = 4 ks + tig >= P (last step): zero, not the next segment
                    bb[ks] = 4 * ks + tig < P ? __ldg(cp + 4 * ks + tig) : make_double2(0.0, 0.0);
            };
            double2 bc[KS], bn[C::PREFETCH ? KS : 1];
            int tau = tau0;
            int st = 0, ui = 0, tl = 0, gend = 0;
            if (tau < tau1) {
                decode(tau, st, ui, tl, gend);
                load_b(st, ui, bc);
            }
            while (tau < tau1) {
                int st2 = 0, ui2 = 0, tl2 = 0, gend2 = 0;
                if (gend < tau1) {
                    decode(gend, st2, ui2, tl2, gend2);
                    if constexpr (C::PREFETCH) load_b(st2, ui2, bn);
                }
                const int p0 = pst[ui], p1 = pst[ui + 1];
                for (int tile = tl; tile < tl + (gend - tau); ++tile) {
                    const int pos = tile * 8 + gid;
                    IFGF_DCHECK(tile >= 0 && tile < C::NR);
                    const double* wr = sW + pos * KP + tig;
                    double dr0 = 0.0, dr1 = 0.0, di0 = 0.0, di1 = 0.0;
                    double er0 = 0.0, er1 = 0.0, ei0 = 0.0, ei1 = 0.0;
#pragma unroll
                    for (int ks = 0; ks < KS; ++ks) {
                        const double a = wr[4 * ks];
                        if (ks & 1) {
                            dmma(er0, er1, a, bc[ks].x);
                            dmma(ei0, ei1, a, bc[ks].y);
                        } else {
                            dmma(dr0, dr1, a, bc[ks].x);
                            dmma(di0, di1, a, bc[ks].y);
                        }
                    }
                    if (pos >= p0 && pos < p1) {
                        dr0 += er0;
                        dr1 += er1;
                        di0 += ei0;
                        di1 += ei1;
                        const int n = sOrd[o * NW + pos];
                        const double rr = g0[n * 5 + 3], ri = g0[n * 5 + 4];
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int qq = st * 8 + 2 * tig + h;
                            if (qq < no) {
                                const int j = sJl[o * J + qq];
                                IFGF_DCHECK(j < J && n < P);
                                const double fr = h ? dr1 : dr0, fi = h ? di1 : di0;
                                double2 acc = sV[j * P + n];
                                acc.x = fma(rr, fr, fma(-ri, fi, acc.x));
                                acc.y = fma(rr, fi, fma(ri, fr, acc.y));
                                sV[j * P + n] = acc;
                            }
                        }
                    }
                }
                tau = gend;
                if (tau < tau1) {
                    st = st2;
                    ui = ui2;
                    tl = tl2;
                    gend = gend2;
                    if constexpr (C::PREFETCH) {
#pragma unroll
                        for (int ks = 0; ks < KS; ++ks) bc[ks] = bn[ks];
                    } else {
                        load_b(st, ui, bc);
                    }
                }
            }
        } else {
            // more distinct child cells than staged (near the poles): evaluate each
            // (segment, node) from global memory; still one writer per V entry
            for (int t = tid; t < no * P; t += NT) {
                const int q = t / P, n = t - q * P;
                const int j = sJl[o * J + q];
                const int B = sChild[o * J + j];
                const double* g = g0 + n * 5;
                const int64_t sl = seg_slot(L, B, sym_cell(L, sU[o * NW + n], sQd[j]));
                if (sl < 0) {
                    atomicOr(bad, 1);
                    continue;
                }
                const double2 F = eval_interp<PS, PA>(vals_d + sl * P, g[0], g[1], g[2]);
                double2 acc = sV[j * P + n];
                acc.x = fma(g[3], F.x, fma(-g[4], F.y, acc.x));
                acc.y = fma(g[3], F.y, fma(g[4], F.x, acc.y));
                sV[j * P + n] = acc;
            }
        }
        if (phase_clk && lane == 0 && U <= umax)  // per-warp busy cycles of the task loop
            atomicAdd(phase_clk + 8, (unsigned long long)(clock64() - t_task0));
        __syncthreads();
        mark(5);
    }

    // ---- phase 5: fused K5 fit, in place, three barriers
    fit_lines_inplace<PS, PA>(sV, cnt, sSeg, Ms, Ma, vals_p, tid, NT);
}

// ---------------------------------------------------------------------------
// K7 on the FP64 tensor core, v2 (P = 75, (P_s, P_ang) = (3, 5)): as k_upward_tc,
// but without the per-octant tensor-basis matrix in shared memory.  The K index
// of the DMMA is permuted so that every lane can form its own A fragments in
// registers from the three 1-D Chebyshev vectors of its node:
//   k' = 4 ks + tig,  ks < 15:  (a, b, c) = (ks % 3, ks / 3, tig)
//                     ks >= 15: j = 4 (ks - 15) + tig, (a, b, c) = (j % 3, j / 3, 4)
// (j = 15 is padding), i.e. coefficient index i = 15 tig + ks, resp. 60 + j: the
// B fragments are plain strided loads of the child coefficient vectors.  Freed
// shared memory (48.6 KB) lets two blocks share an SM, so one block's barriers
// and geometry overlap the other's DMMAs.  Tasks per octant = (node-tile run of
// one child cell, segment tile), contiguous per warp so consecutive tasks reuse
// the A fragments.
template <int PS, int PA>
struct Tc2Cfg {
    static_assert(PS == 3 && PA == 5, "k-permutation is specific to (P_s, P_ang) = (3, 5)");
    static constexpr int P = 75, KS = 19, NR = 10, NW = 80;
    static constexpr int J = kChunkTC2;
    static constexpr int UM = 8;
    static constexpr int NT = 256;  // 2 blocks/SM (measured: 192 threads 214 ms, 384 threads 280 ms, 256 200 ms at cfg4 6->5)
    static constexpr int NWARP = NT / 32;
    static constexpr int R = (NW + 31) / 32;
    static constexpr int FG = 8;  // fit group (aliases the geometry)
    static constexpr size_t a16(size_t x) { return (x + 15) / 16 * 16; }
    static constexpr size_t oV = 0;                                       // double2 [J][P]
    static constexpr size_t oG = a16(oV + (size_t)J * P * 16);            // double [8][NW][5]
    static constexpr size_t oU = a16(oG + (size_t)8 * NW * 5 * 8);        // int [8][NW]
    static constexpr size_t oSlot = a16(oU + (size_t)8 * NW * 4);         // int [8][UM][J]
    static constexpr size_t oChild = a16(oSlot + (size_t)8 * UM * J * 4); // int [8][J]
    static constexpr size_t oSeg = a16(oChild + (size_t)8 * J * 4);       // int [J]
    static constexpr size_t oUcell = a16(oSeg + (size_t)J * 4);           // int [8][UM]
    static constexpr size_t oMisc = a16(oUcell + (size_t)8 * UM * 4);     // int U[8], nO[8]
    static constexpr size_t oPst = a16(oMisc + 16 * 4);                   // u8 [8][UM + 1]
    static constexpr size_t oOrd = a16(oPst + (size_t)8 * (UM + 1));      // u8 [8][NW]
    static constexpr size_t oJl = a16(oOrd + (size_t)8 * NW);             // u8 [8][J]
    static constexpr size_t oFit = a16(oJl + (size_t)8 * J);              // double Ms, Ma
    static constexpr size_t smem = a16(oFit + (size_t)(PS * PS + PA * PA) * 8);
    static_assert(2 * FG * P * 16 <= 8 * NW * 5 * 8, "fit temporaries alias the geometry");
};

template <int PS, int PA>
__global__ void __launch_bounds__(Tc2Cfg<PS, PA>::NT, 2) k_upward_tc2(LevelParams L, LevelParams LP,
                                                       const double2* __restrict__ vals_d, double k,
                                                       const double* __restrict__ Ms, const double* __restrict__ Ma,
                                                       double2* vals_p, int* bad, int umax,
                                                       const double2* __restrict__ zseg) {
    using C = Tc2Cfg<PS, PA>;
    constexpr int P = C::P, KS = C::KS, NW = C::NW, J = C::J, UM = C::UM, NT = C::NT, NWARP = C::NWARP,
                  R = C::R, FG = C::FG;
    extern __shared__ __align__(16) unsigned char smraw[];
    double2* sV = reinterpret_cast<double2*>(smraw + C::oV);
    double* sG = reinterpret_cast<double*>(smraw + C::oG);
    int* sU = reinterpret_cast<int*>(smraw + C::oU);
    int* sSlot = reinterpret_cast<int*>(smraw + C::oSlot);
    int* sChild = reinterpret_cast<int*>(smraw + C::oChild);
    int* sSeg = reinterpret_cast<int*>(smraw + C::oSeg);
    int* sUcell = reinterpret_cast<int*>(smraw + C::oUcell);
    int* sUn = reinterpret_cast<int*>(smraw + C::oMisc);
    int* sNo = sUn + 8;
    unsigned char* sPst = smraw + C::oPst;
    unsigned char* sOrd = smraw + C::oOrd;
    unsigned char* sJl = smraw + C::oJl;
    double* sMs = reinterpret_cast<double*>(smraw + C::oFit);
    double* sMa = sMs + PS * PS;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t c = LP.chunk_order ? LP.chunk_order[blockIdx.x] : blockIdx.x;
    const int s0 = LP.chunk_start[c];
    const int s1 = (c + 1 < LP.nchunk) ? LP.chunk_start[c + 1] : (int)LP.nseg;
    const int cnt = min(J, s1 - s0);

    // ---- phase 0: segments, children by octant, per-octant compaction
    __shared__ int sBox[J];
    __shared__ unsigned char sQd[J];  // quarter turns of segment j's cell from the representative
    for (int j = tid; j < J; j += NT) {
        int seg = -1, box = -1, qd = 0;
        if (j < cnt) {
            seg = LP.cell_seg[s0 + j];
            box = LP.seg_box[seg];
            qd = sym_quarter(LP, LP.seg_cell[seg]);
        }
        sSeg[j] = seg;
        sBox[j] = box;
        sQd[j] = (unsigned char)qd;
    }
    for (int t = tid; t < J * P; t += NT) sV[t] = make_double2(0.0, 0.0);
    __syncthreads();
    for (int t = tid; t < 8 * J; t += NT) {  // 8 J = NT: one round
        const int o = t / J, j = t - o * J;
        int B = sBox[j] >= 0 ? LP.child_oct[8 * sBox[j] + rot_oct(o, sQd[j])] : -1;
        if (B < L.b0 || B >= L.b1) B = -1;
        sChild[t] = B;
    }
    __syncthreads();
    for (int o = warp; o < 8; o += NWARP) {
        int base = 0;
        for (int j0 = 0; j0 < J; j0 += 32) {
            const int j = j0 + lane;
            const bool pr = j < J && sChild[o * J + j] >= 0;
            const unsigned b = __ballot_sync(~0u, pr);
            if (pr) sJl[o * J + base + __popc(b & lt)] = (unsigned char)j;
            base += __popc(b);
        }
        if (lane == 0) sNo[o] = base;
    }
    __syncthreads();

    // ---- phase 1: geometry of (octant, node)
    const int cellp = sym_rep(LP, LP.seg_cell[sSeg[0]]);  // the chunk's (representative) parent cell
    const double hh = 0.5 * L.H;
    for (int t = tid; t < 8 * NW; t += NT) {
        const int o = t / NW, n = t - o * NW;
        int u = INT_MAX;
        if (n < P && sNo[o] > 0) {
            double off[3];
            node_off(LP, PS, PA, cellp, n, off);
            const double rQ = sqrt(fma(off[0], off[0], fma(off[1], off[1], off[2] * off[2])));
            const double dx = (o & 4) ? -hh : hh, dy = (o & 2) ? -hh : hh, dz = (o & 1) ? -hh : hh;
            const double vx = __dadd_rn(off[0], dx), vy = __dadd_rn(off[1], dy);
            const Cls cl = classify(L, vx, vy, __dadd_rn(off[2], dz));
            u = (int)cell_of(L, cl);
            if (LP.sym && vx == 0.0 && vy == 0.0) u |= kPoleFlag;  // pole: sector 0 in every rotation
            // r_B - r_Q = (delta.delta + 2 off.delta) / (r_B + r_Q)   (reading R17)
            const double num = fma(dx, dx, fma(dy, dy, dz * dz)) + 2.0 * fma(off[0], dx, fma(off[1], dy, off[2] * dz));
            const double ic = rcp_nr(cl.r * (cl.r + rQ));
            const double diff = num * cl.r * ic;
            const double ratio = rQ * (cl.r + rQ) * ic;
            double sn, cs;
            fm::sincos(k * diff, &sn, &cs);
            double* g = sG + (size_t)t * 5;
            g[0] = cl.us;
            g[1] = cl.ut;
            g[2] = cl.up;
            g[3] = ratio * cs;
            g[4] = ratio * sn;
        }
        sU[t] = u;
    }
    __syncthreads();

    // ---- phase 2: per octant (warp): distinct child cells ascending, stable node
    // sort by cell; cell index ui owns sorted positions [pst[ui], pst[ui + 1])
    for (int o = warp; o < 8; o += NWARP) {
        int uv[R];
        bool done[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int n = lane + 32 * r;
            uv[r] = n < NW ? sU[o * NW + n] : INT_MAX;
            done[r] = !(n < P) || uv[r] == INT_MAX;
        }
        int base = 0, U = 0;
        while (true) {
            int m = INT_MAX;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (!done[r]) m = min(m, uv[r]);
            m = __reduce_min_sync(~0u, m);
            if (m == INT_MAX) break;
            if (lane == 0 && U <= UM) sPst[o * (UM + 1) + U] = (unsigned char)base;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const bool hit = !done[r] && uv[r] == m;
                const unsigned b = __ballot_sync(~0u, hit);
                if (hit) {
                    const int pos = base + __popc(b & lt);
                    sOrd[o * NW + pos] = (unsigned char)(lane + 32 * r);
                    done[r] = true;
                }
                base += __popc(b);
            }
            if (lane == 0 && U < UM) sUcell[o * UM + U] = m;
            ++U;
        }
        if (lane == 0 && U <= UM) sPst[o * (UM + 1) + U] = (unsigned char)base;
        for (int pos = base + lane; pos < NW; pos += 32) {
            sOrd[o * NW + pos] = (unsigned char)pos;
        }
        if (lane == 0) sUn[o] = U;
    }
    __syncthreads();

    // ---- phase 3: child segment slots of the staged (octant, cell, compacted
    // segment) triples only (tasks treat columns q >= n_o as absent)
    {
        __shared__ int sPre[9];
        if (tid == 0) {
            int acc = 0;
            for (int o = 0; o < 8; ++o) {
                sPre[o] = acc;
                if (sUn[o] <= umax) acc += sUn[o] * sNo[o];
            }
            sPre[8] = acc;
        }
        __syncthreads();
        const int tot = sPre[8];
        for (int t0 = tid; t0 < tot; t0 += 2 * NT) {
            int idx[2], Bv[2], cellv[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int t = t0 + h * NT;
                idx[h] = -1;
                if (t < tot) {
                    int o = 0;
                    while (o < 7 && t >= sPre[o + 1]) ++o;
                    const int rem = t - sPre[o], no = sNo[o];
                    const int ui = rem / no, q = rem - ui * no;
                    idx[h] = (o * UM + ui) * J + q;
                    const int j = sJl[o * J + q];
                    Bv[h] = sChild[o * J + j];
                    cellv[h] = sym_cell(L, sUcell[o * UM + ui], sQd[j]);
                }
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (idx[h] < 0) continue;
                const int64_t s64 = seg_slot(L, Bv[h], cellv[h]);
                if (s64 < 0) atomicOr(bad, 1);
                sSlot[idx[h]] = (int)s64;
            }
        }
    }
    __syncthreads();

    // ---- phase 4: per octant, DMMA tasks (run of one cell's node tiles x segment tile)
    const int gid = lane >> 2, tig = lane & 3;
    // B fragment offsets of this lane (permuted k): i = 15 tig + ks (ks < 15), 60 + 4 (ks - 15) + tig
    for (int o = 0; o < 8; ++o) {
        const int no = sNo[o];
        if (no == 0) continue;
        const int U = sUn[o];
        const double* g0 = sG + (size_t)o * NW * 5;
        if (U <= umax) {
            const unsigned char* pst = sPst + o * (UM + 1);
            const int nst = (no + 7) >> 3;
            // runs: (cell ui, node tile) in sorted order; tasks = runs x segment tiles
            int nrun = 0;
            for (int u = 0; u < U; ++u) nrun += ((pst[u + 1] - 1) >> 3) - (pst[u] >> 3) + 1;
            const int T = nrun * nst;
            const int tau0 = (int)((int64_t)warp * T / NWARP), tau1 = (int)((int64_t)(warp + 1) * T / NWARP);
            int cur_run = -1, ui = 0, tile = 0;
            double a[KS];
            int run = tau0 / nst, st = tau0 - (tau0 / nst) * nst;
            for (int tau = tau0; tau < tau1; ++tau) {
                if (run != cur_run) {
                    cur_run = run;
                    int rr = run;
                    ui = 0;
                    while (true) {
                        const int a0 = pst[ui] >> 3, n_t = ((pst[ui + 1] - 1) >> 3) - a0 + 1;
                        if (rr < n_t) {
                            tile = a0 + rr;
                            break;
                        }
                        rr -= n_t;
                        ++ui;
                    }
                    // A fragments of row (node) pos = 8 tile + gid in registers
                    const int pos = tile * 8 + gid;
                    const int nn = pos < P ? sOrd[o * NW + pos] : 0;
                    const double* g = g0 + nn * 5;
                    double Ts[3], Tt[5], Tp[5];
                    cheb_T<3>(g[0], Ts);
                    cheb_T<5>(g[1], Tt);
                    cheb_T<5>(g[2], Tp);
                    const double tpo = tig == 0 ? Tp[0] : (tig == 1 ? Tp[1] : (tig == 2 ? Tp[2] : Tp[3]));
                    double tt[15];
#pragma unroll
                    for (int b = 0; b < 5; ++b)
#pragma unroll
                        for (int aa = 0; aa < 3; ++aa) tt[b * 3 + aa] = Ts[aa] * Tt[b];
#pragma unroll
                    for (int ks = 0; ks < 15; ++ks) a[ks] = tt[ks] * tpo;
                    // ks = 15..18: j = 4 (ks - 15) + tig, product index j (j = 15: padding)
                    const double t4 = Tp[4];
                    a[15] = (tig == 0 ? tt[0] : (tig == 1 ? tt[1] : (tig == 2 ? tt[2] : tt[3]))) * t4;
                    a[16] = (tig == 0 ? tt[4] : (tig == 1 ? tt[5] : (tig == 2 ? tt[6] : tt[7]))) * t4;
                    a[17] = (tig == 0 ? tt[8] : (tig == 1 ? tt[9] : (tig == 2 ? tt[10] : tt[11]))) * t4;
                    a[18] = (tig == 0 ? tt[12] : (tig == 1 ? tt[13] : (tig == 2 ? tt[14] : 0.0))) * t4;
                }
                // B fragments: column q = st*8 + gid
                const int q = st * 8 + gid;
                const int sl = q < no ? sSlot[(o * UM + ui) * J + q] : -1;
                const double2* cp = sl >= 0 ? vals_d + (int64_t)sl * P : zseg;
                double dr0 = 0.0, dr1 = 0.0, di0 = 0.0, di1 = 0.0;
                double er0 = 0.0, er1 = 0.0, ei0 = 0.0, ei1 = 0.0;
                {
                    double2 b[KS];
#pragma unroll
                    for (int ks = 0; ks < KS; ++ks) {  // k = 60 + 4 (ks - 15) + tig >= P: zero
                        const int kk = ks < 15 ? 15 * tig + ks : 60 + 4 * (ks - 15) + tig;
                        b[ks] = kk < P ? __ldg(cp + kk) : make_double2(0.0, 0.0);
                    }
#pragma unroll
                    for (int ks = 0; ks < KS; ++ks) {
                        if (ks & 1) {
                            dmma(er0, er1, a[ks], b[ks].x);
                            dmma(ei0, ei1, a[ks], b[ks].y);
                        } else {
                            dmma(dr0, dr1, a[ks], b[ks].x);
                            dmma(di0, di1, a[ks], b[ks].y);
                        }
                    }
                }
                const int pos = tile * 8 + gid;
                if (pos >= pst[ui] && pos < pst[ui + 1]) {
                    dr0 += er0;
                    dr1 += er1;
                    di0 += ei0;
                    di1 += ei1;
                    const int n = sOrd[o * NW + pos];
                    const double rr = g0[n * 5 + 3], ri = g0[n * 5 + 4];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int qq = st * 8 + 2 * tig + h;
                        if (qq < no) {
                            const int j = sJl[o * J + qq];
                            const double fr = h ? dr1 : dr0, fi = h ? di1 : di0;
                            double2 acc = sV[j * P + n];
                            acc.x = fma(rr, fr, fma(-ri, fi, acc.x));
                            acc.y = fma(rr, fi, fma(ri, fr, acc.y));
                            sV[j * P + n] = acc;
                        }
                    }
                }
                if (++st == nst) {
                    st = 0;
                    ++run;
                }
            }
        } else {
            // more distinct child cells than staged (near the poles): per (segment, node)
            for (int t = tid; t < no * P; t += NT) {
                const int q = t / P, n = t - q * P;
                const int j = sJl[o * J + q];
                const int B = sChild[o * J + j];
                const double* g = g0 + n * 5;
                const int64_t sl = seg_slot(L, B, sym_cell(L, sU[o * NW + n], sQd[j]));
                if (sl < 0) {
                    atomicOr(bad, 1);
                    continue;
                }
                double Ts[PS], Tt[PA];
                cheb_T<PS>(g[0], Ts);
                cheb_T<PA>(g[1], Tt);
                const double2 F = contract_sm_lr<PS, PA, true>(vals_d + sl * P, Ts, Tt, g[2]);
                double2 acc = sV[j * P + n];
                acc.x = fma(g[3], F.x, fma(-g[4], F.y, acc.x));
                acc.y = fma(g[3], F.y, fma(g[4], F.x, acc.y));
                sV[j * P + n] = acc;
            }
        }
        __syncthreads();
    }

    // ---- phase 5: fused K5 fit, in place, three barriers
    fit_lines_inplace<PS, PA>(sV, cnt, sSeg, Ms, Ma, vals_p, tid, NT);
}

// ------------------------------------------------------------- dispatch
template <int PS, int PA>
struct Kern {
    static void cousin(dim3 g, cudaStream_t st, const LevelParams& L, const ifgf_plan_s* p, const double2* v,
                       double2* out, int* bad) {
        if constexpr (PS > 0) {
            if (!p->legacy_cousin) {
                if (L.nsplit_cou > 1)
                    k_cousin_ws<PS, PA, true><<<g, TPB, 0, st>>>(L, p->px, p->py, p->pz, v, p->k, out, bad,
                                                                 p->stage_slots);
                else
                    k_cousin_ws<PS, PA, false><<<g, TPB, 0, st>>>(L, p->px, p->py, p->pz, v, p->k, out, bad,
                                                                  p->stage_slots);
                return;
            }
        }
        k_cousin<PS, PA><<<g, TPB, 0, st>>>(L, p->px, p->py, p->pz, v, p->k, p->Ps, p->Pa, out, bad);
    }
    // returns true if the kernel also produced the Chebyshev coefficients (fused K5)
    static bool upward(dim3 g, cudaStream_t st, const LevelParams& L, const LevelParams& LP, const ifgf_plan_s* p,
                       const double2* vd, double2* vp, int* bad) {
        if constexpr (PS == 3 && PA == 5) {
            if (LP.up_kernel == 3 && LP.nchunk > 0) {
                using Cfg = Tc2Cfg<PS, PA>;
                // per launch (cheap): the attribute is per device, and a process may drive several
                IFGF_CUDA(cudaFuncSetAttribute(k_upward_tc2<PS, PA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)Cfg::smem));
                k_upward_tc2<PS, PA><<<(unsigned)LP.nchunk, Cfg::NT, Cfg::smem, st>>>(
                    L, LP, vd, p->k, p->cheb_Ms, p->cheb_Ma, vp, bad, std::min(Cfg::UM, p->tc_umax), p->zseg);
                return true;
            }
        }
        if constexpr (PS > 0 && PS * PA * PA <= 80) {
            if (LP.up_kernel == 1 && LP.nchunk > 0) {
                using Cfg = TcCfg<PS, PA>;
                // per launch (cheap): the attribute is per device, and a process may drive several
                IFGF_CUDA(cudaFuncSetAttribute(k_upward_tc<PS, PA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)Cfg::smem));
                k_upward_tc<PS, PA><<<(unsigned)LP.nchunk, Cfg::NT, Cfg::smem, st>>>(
                    L, LP, vd, p->k, p->cheb_Ms, p->cheb_Ma, vp, bad, std::min(Cfg::UM, p->tc_umax), p->zseg,
                    p->phase_clk);
                return true;
            }
        }
        if constexpr (PS > 0 && PS * PA * PA <= 128) {
            if (LP.up_kernel == 0 && LP.nchunk > 0) {
                using Cfg = StagedCfg<PS, PA>;
                // per launch (cheap): the attribute is per device, and a process may drive several
                IFGF_CUDA(cudaFuncSetAttribute(k_upward_s<PS, PA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)Cfg::smem));
                k_upward_s<PS, PA><<<(unsigned)LP.nchunk, Cfg::NT, Cfg::smem, st>>>(L, LP, vd, p->k, p->cheb_Ms,
                                                                                      p->cheb_Ma, vp, bad);
                return true;
            }
        }
        if constexpr (PS > 0) {
            if (p->legacy_upward != 1) {
                const dim3 gpe((unsigned)((LP.nseg * (PS * PA * PA) + PE_WARPS * 32 - 1) / (PE_WARPS * 32)));
                k_upward_pe<PS, PA><<<gpe, PE_WARPS * 32, 0, st>>>(L, LP, vd, p->k, vp, bad, p->stage_slots);
                return false;
            }
        }
        k_upward<PS, PA><<<g, TPB, 0, st>>>(L, LP, vd, p->k, p->Ps, p->Pa, vp, bad);
        return false;
    }
};

// Orders with compiled specialisations: (3, 5) (the BASELINE configs), (5, 5) (cfg3)
// and (5, 7) (the accuracy knob: ~20x lower error than (3, 5)); any
// other order runs the runtime-order kernels.
template <class F3, class F5, class F7, class FG>
void dispatch(int Ps, int Pa, F3 f35, F5 f55, F7 f57, FG fg) {
    if (Ps == 3 && Pa == 5) f35();
    else if (Ps == 5 && Pa == 5) f55();
    else if (Ps == 5 && Pa == 7) f57();
    else fg();
}

struct Prof {  // CUDA events around each launch (ifgf_profile_enable)
    ifgf_plan_s* p;
    cudaStream_t st;
    int cls = 0;
    cudaEvent_t e0 = nullptr;
    Prof(ifgf_plan_s* p_, cudaStream_t s, int c) : p(p_), st(s), cls(c) {
        if (!p->profile) return;
        e0 = take();
        IFGF_CUDA(cudaEventRecord(e0, st));
    }
    cudaEvent_t take() {
        cudaEvent_t e;
        if (!p->ev_pool.empty()) {
            e = p->ev_pool.back();
            p->ev_pool.pop_back();
        } else {
            IFGF_CUDA(cudaEventCreate(&e));
        }
        return e;
    }
    void done() {
        IFGF_CUDA(cudaGetLastError());
        if (!p->profile) return;
        cudaEvent_t e1 = take();
        IFGF_CUDA(cudaEventRecord(e1, st));
        p->pending.push_back({cls, e0, e1});
    }
};

}  // namespace

// K5 fit of level d's node values into Chebyshev coefficients, in place.
void fit_level(ifgf_plan_s* p, int d, cudaStream_t st) {
    const int P = p->P, Ps = p->Ps, Pa = p->Pa;
    LevelParams& L = p->lev[d].p;
    if (L.nseg == 0) return;
    const int fit_warps = std::max(1, std::min(4, (int)(48 * 1024 / (32 * P))));
    const size_t fit_smem = (size_t)fit_warps * 2 * P * sizeof(double2);
    if (fit_smem > 48 * 1024)
        IFGF_CUDA(cudaFuncSetAttribute(k_fit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fit_smem));
    Prof pr(p, st, 3);
    const unsigned nb8 = (unsigned)((L.nseg + 3) / 4);
    dispatch(
        Ps, Pa, [&] { k_fit_lines<3, 5><<<nb8, 64, 0, st>>>(L.nseg, p->cheb_Ms, p->cheb_Ma, p->vals[d & 1]); },
        [&] { k_fit_lines<5, 5><<<nb8, 64, 0, st>>>(L.nseg, p->cheb_Ms, p->cheb_Ma, p->vals[d & 1]); },
        [&] { k_fit_lines<5, 7><<<nb8, 64, 0, st>>>(L.nseg, p->cheb_Ms, p->cheb_Ma, p->vals[d & 1]); },
        [&] {
            k_fit<<<(int)((L.nseg + fit_warps - 1) / fit_warps), 32 * fit_warps, fit_smem, st>>>(
                L.nseg, Ps, Pa, p->cheb_Ms, p->cheb_Ma, p->vals[d & 1]);
        });
    pr.done();
}

// K6 of level d: out_sorted += cousin interpolation (Morton order).
void cousin_level(ifgf_plan_s* p, int d, cudaStream_t st) {
    LevelParams& L = p->lev[d].p;
    if (L.nseg == 0 || L.nwitems == 0) return;
    Prof pr(p, st, 4);
    const double2* vd = p->vals[d & 1];
    dim3 g(nblk(L.nwitems * L.nsplit_cou * 32));
    dispatch(
        p->Ps, p->Pa, [&] { Kern<3, 5>::cousin(g, st, L, p, vd, p->out_sorted, p->dev_bad); },
        [&] { Kern<5, 5>::cousin(g, st, L, p, vd, p->out_sorted, p->dev_bad); },
        [&] { Kern<5, 7>::cousin(g, st, L, p, vd, p->out_sorted, p->dev_bad); },
        [&] { Kern<0, 0>::cousin(g, st, L, p, vd, p->out_sorted, p->dev_bad); });
    pr.done();
}

// K7 d -> d-1 (+ the K5 fit of level d-1 when the kernel does not fuse it).
void upward_level(ifgf_plan_s* p, int d, cudaStream_t st) {
    LevelParams& L = p->lev[d].p;
    LevelParams& LP = p->lev[d - 1].p;
    if (LP.nseg == 0) return;
    bool fused = false;
    {
        Prof pr(p, st, 5);
        dim3 g(nblk(LP.nseg * p->P));
        const double2* vd = p->vals[d & 1];
        double2* vp = p->vals[(d - 1) & 1];
        dispatch(
            p->Ps, p->Pa, [&] { fused = Kern<3, 5>::upward(g, st, L, LP, p, vd, vp, p->dev_bad); },
            [&] { fused = Kern<5, 5>::upward(g, st, L, LP, p, vd, vp, p->dev_bad); },
            [&] { fused = Kern<5, 7>::upward(g, st, L, LP, p, vd, vp, p->dev_bad); },
            [&] { fused = Kern<0, 0>::upward(g, st, L, LP, p, vd, vp, p->dev_bad); });
        pr.done();
    }
    if (!fused) fit_level(p, d - 1, st);
}

// One apply (Algorithm 1).  The near field (K3) accumulates into its
// own buffer; the cousin interpolation (K6, levels D..3 in order) into out_sorted;
// the un-permute adds the two (the same order whether or not the kernels overlap).
// conc (graph capture): three streams -- K3 || (K4, K5, K7 chain) || K6 chain,
// with K6(d) after level d's values and K7(d -> d-1) after K6(d+1) (it overwrites
// level d+1's buffer); otherwise everything runs in order on st.
void run_apply(ifgf_plan_s* p, const double2* dens, double2* out, cudaStream_t st, bool conc) {
    const int D = p->D, Ps = p->Ps, Pa = p->Pa;
    const int64_t n = p->n;
    const unsigned mask = p->stage_mask;
    if (conc && !p->side[0]) {
        for (int i = 0; i < 2; ++i) IFGF_CUDA(cudaStreamCreateWithFlags(&p->side[i], cudaStreamNonBlocking));
        p->ev.resize(2 * (D + 2) + 2);
        for (auto& e : p->ev) IFGF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    cudaStream_t sN = conc ? p->side[0] : st, sU = conc ? p->side[1] : st;
    auto ev_lev = [&](int d) { return p->ev[d]; };
    auto ev_cou = [&](int d) { return p->ev[(D + 2) + d]; };
    cudaEvent_t ev_fork = conc ? p->ev[2 * (D + 2)] : nullptr, ev_near = conc ? p->ev[2 * (D + 2) + 1] : nullptr;
    {
        Prof pr(p, st, 0);
        k_permute<<<nblk(n, 256), 256, 0, st>>>(dens, p->perm, n, p->a_sorted);
        pr.done();
    }
    if (conc) {
        IFGF_CUDA(cudaEventRecord(ev_fork, st));
        IFGF_CUDA(cudaStreamWaitEvent(sN, ev_fork, 0));
        IFGF_CUDA(cudaStreamWaitEvent(sU, ev_fork, 0));
    }
    LevelHost& LD = p->lev[D];
    const bool near = mask & IFGF_STAGE_NEAR;
    if (near) {
        Prof pr(p, sN, 1);
        // targets without an owned neighbour get no near-field work item (multi-rank), and
        // with a split every part is a partial sum over its share of the neighbour boxes
        if (p->nranks > 1 || p->nparts_near > 1)
            IFGF_CUDA(cudaMemsetAsync(p->near_sorted, 0, sizeof(double2) * n * p->nparts_near, sN));
        const dim3 gn(nblk(LD.p.nwitems_near * LD.p.nsplit_near * 32));
        if (LD.p.nsplit_near > 1)
            k_near<true><<<gn, TPB, 0, sN>>>(LD.p, p->px, p->py, p->pz, p->a_sorted, p->k, p->near_sorted);
        else
            k_near<false><<<gn, TPB, 0, sN>>>(LD.p, p->px, p->py, p->pz, p->a_sorted, p->k, p->near_sorted);
        pr.done();
        if (conc) IFGF_CUDA(cudaEventRecord(ev_near, sN));
    }
    IFGF_CUDA(cudaMemsetAsync(p->out_sorted, 0, sizeof(double2) * n * p->nparts_cou, st));
    bool have = false;        // level d holds coefficients
    bool leaf_fused = false;  // K4 fused the leaf-level fit
    if (D >= 3 && (mask & (IFGF_STAGE_COUSIN | IFGF_STAGE_UPWARD)) && LD.p.b1 > LD.p.b0) {
        if (LD.p.nseg > 0) {
            Prof pr(p, sU, 2);
            const unsigned nb = (unsigned)((LD.p.b1 - LD.p.b0) * LD.p.nsplit_s2c);
            if (LD.p.ncell <= 8 && Ps == 3 && Pa == 5) {
                k_s2c<3, 5><<<nb, TPB, 0, sU>>>(LD.p, p->px, p->py, p->pz, p->a_sorted, p->k, Ps, Pa, p->vals[D & 1],
                                                p->cheb_Ms, p->cheb_Ma);
                leaf_fused = true;
            } else if (LD.p.ncell <= 8 && Ps == 5 && Pa == 5) {
                k_s2c<5, 5><<<nb, TPB, 0, sU>>>(LD.p, p->px, p->py, p->pz, p->a_sorted, p->k, Ps, Pa, p->vals[D & 1],
                                                p->cheb_Ms, p->cheb_Ma);
                leaf_fused = true;
            } else if (LD.p.ncell <= 8 && Ps == 5 && Pa == 7) {
                k_s2c<5, 7><<<nb, TPB, 0, sU>>>(LD.p, p->px, p->py, p->pz, p->a_sorted, p->k, Ps, Pa, p->vals[D & 1],
                                                p->cheb_Ms, p->cheb_Ma);
                leaf_fused = true;
            } else {
                k_s2c<0, 0><<<nb, TPB, 0, sU>>>(LD.p, p->px, p->py, p->pz, p->a_sorted, p->k, Ps, Pa, p->vals[D & 1],
                                                p->cheb_Ms, p->cheb_Ma);
            }
            pr.done();
        }
        have = true;
    }
    auto phase_dump = [&](int dl) {
        if (!p->phase_clk) return;
        unsigned long long h[16];
        IFGF_CUDA(cudaMemcpyAsync(h, p->phase_clk, sizeof(h), cudaMemcpyDeviceToHost, st));
        IFGF_CUDA(cudaStreamSynchronize(st));
        IFGF_CUDA(cudaMemsetAsync(p->phase_clk, 0, sizeof(h), st));
        double tot = 0;
        for (int i = 0; i < 7; ++i) tot += (double)h[i];
        fprintf(stderr, "[ifgf] level %d TC K7 phase clocks (block-thread-0 sums, %% of total %.3g):", dl, tot);
        for (int i = 0; i < 7; ++i) fprintf(stderr, " p%d=%.1f%%", i, 100.0 * (double)h[i] / (tot > 0 ? tot : 1));
        fprintf(stderr, "; task-loop warp utilisation %.1f%% (%d warps); per octant: %.2f cells, %.2f node tiles, "
                "%.1f segments; %.2f octants per chunk\n",
                100.0 * (double)h[8] / ((double)TcCfg<3, 5>::NWARP * (double)(h[5] > 0 ? h[5] : 1)),
                TcCfg<3, 5>::NWARP, (double)h[9] / std::max(1.0, (double)h[12]),
                (double)h[10] / std::max(1.0, (double)h[12]), (double)h[11] / std::max(1.0, (double)h[12]),
                (double)h[12] / std::max(1.0, (double)h[13]));
    };
    if (have && !leaf_fused) fit_level(p, D, sU);
    if (conc && have) IFGF_CUDA(cudaEventRecord(ev_lev(D), sU));
    for (int d = D; d >= 3 && have; --d) {
        if (mask & IFGF_STAGE_COUSIN) {
            if (conc) IFGF_CUDA(cudaStreamWaitEvent(st, ev_lev(d), 0));
            cousin_level(p, d, st);
        }
        if (conc) IFGF_CUDA(cudaEventRecord(ev_cou(d), st));
        if (d > 3 && (mask & IFGF_STAGE_UPWARD)) {
            // K7 (d -> d-1) overwrites level d+1's buffer: after K6(d+1)
            if (conc && d < D) IFGF_CUDA(cudaStreamWaitEvent(sU, ev_cou(d + 1), 0));
            upward_level(p, d, sU);
            if (conc) IFGF_CUDA(cudaEventRecord(ev_lev(d - 1), sU));
            phase_dump(d - 1);
        } else {
            have = false;
        }
    }
    if (conc) {  // join: the near field and the upward chain
        if (near) IFGF_CUDA(cudaStreamWaitEvent(st, ev_near, 0));
        IFGF_CUDA(cudaEventRecord(ev_fork, sU));
        IFGF_CUDA(cudaStreamWaitEvent(st, ev_fork, 0));
    }
    {
        Prof pr(p, st, 6);
        k_unpermute_sum<<<nblk(n, 256), 256, 0, st>>>(p->out_sorted, p->nparts_cou, p->near_sorted,
                                                      near ? p->nparts_near : 0, p->perm, n, out);
        pr.done();
    }
}

// Test hook (ifgf_debug_level_pass): one level's K5 / K6 / K7 in isolation on
// caller-supplied node values (SURVEY.md §8(c) exact pin 2, polynomial injection).
void debug_level_pass(ifgf_plan_s* p, int d, const double2* values_h, unsigned what, double2* field_h,
                      double2* parent_h) {
    const int P = p->P;
    const int64_t n = p->n;
    cudaStream_t st;
    IFGF_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamSynchronize(s); cudaStreamDestroy(s); }
    } sg{st};
    LevelParams& L = p->lev[d].p;
    IFGF_CUDA(cudaMemcpyAsync(p->vals[d & 1], values_h, sizeof(double2) * (size_t)L.nseg * P, cudaMemcpyHostToDevice, st));
    fit_level(p, d, st);
    if (what & 1) {
        IFGF_CUDA(cudaMemsetAsync(p->out_sorted, 0, sizeof(double2) * n * p->nparts_cou, st));
        cousin_level(p, d, st);
        double2* tmp = nullptr;
        IFGF_CUDA(cudaMallocAsync((void**)&tmp, sizeof(double2) * n, st));
        k_unpermute_sum<<<nblk(n, 256), 256, 0, st>>>(p->out_sorted, p->nparts_cou, nullptr, 0, p->perm, n, tmp);
        IFGF_CUDA(cudaMemcpyAsync(field_h, tmp, sizeof(double2) * n, cudaMemcpyDeviceToHost, st));
        IFGF_CUDA(cudaFreeAsync(tmp, st));
    }
    if ((what & 2) && d > 3) {
        upward_level(p, d, st);
        IFGF_CUDA(cudaMemcpyAsync(parent_h, p->vals[(d - 1) & 1], sizeof(double2) * (size_t)p->lev[d - 1].p.nseg * P,
                                  cudaMemcpyDeviceToHost, st));
    }
    IFGF_CUDA(cudaStreamSynchronize(st));
}

}  // namespace ifgf
