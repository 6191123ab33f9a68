// capi.cu -- the C ABI of libifgf (include/ifgf.h): argument validation,
// error mapping, plan lifetime, host-buffer apply, profiling, the direct-sum
// measurement kernel, the FP64 roofline microbenchmark and the partitioner.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include <nccl.h>

#include "ifgf_internal.cuh"

#define IFGF_NCCL(call)                                                                              \
    do {                                                                                             \
        ncclResult_t r_ = (call);                                                                    \
        if (r_ != ncclSuccess) throw ::ifgf::Error{IFGF_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)}; \
    } while (0)

namespace {
thread_local std::string g_last_error;

ifgf_status fail(ifgf_status s, const std::string& m) {
    g_last_error = m;
    return s;
}

template <class F>
ifgf_status guarded(ifgf_plan_s* p, F&& f) {
    try {
        f();
        return IFGF_OK;
    } catch (const ifgf::Error& e) {
        if (p && (e.st == IFGF_ECUDA || e.st == IFGF_ENCCL)) p->sticky_cuda_error = true;
        return fail(e.st, e.msg);
    } catch (const std::bad_alloc&) {
        return fail(IFGF_ENOMEM, "host allocation failed");
    } catch (...) {
        return fail(IFGF_EINTERNAL, "unexpected exception");
    }
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (dev >= 0 && cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
        else prev = -1;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

void free_plan(ifgf_plan_s* p) {
    if (!p) return;
    if (p->gexec) cudaGraphExecDestroy(p->gexec);
    if (p->cap_stream) cudaStreamDestroy(p->cap_stream);
    for (auto& sd : p->side)
        if (sd) cudaStreamDestroy(sd);
    for (auto& e : p->ev) cudaEventDestroy(e);
    for (void* a : p->allocs) cudaFree(a);
    for (auto& e : p->ev_pool) cudaEventDestroy(e);
    for (auto& e : p->pending) {
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
    }
    delete p;
}

// One apply on stream st: the kernels replayed from the plan's CUDA
// graph (captured on the first call for this (dens, out) pair; eager launches
// while profiling, with opts.no_graph, or if capture is not possible), then the
// in-place all-reduce of the ranks' partial fields when a communicator is set.
void apply_dispatch(ifgf_plan_s* p, const double2* dens, double2* out, cudaStream_t st) {
    const bool graph = p->use_graph && !p->graph_failed && !p->profile && !p->phase_clk;
    bool done = false;
    if (graph) {
        if (!p->gexec || p->g_dens != dens || p->g_out != out) {
            if (p->gexec) {
                IFGF_CUDA(cudaGraphExecDestroy(p->gexec));
                p->gexec = nullptr;
            }
            if (!p->cap_stream) IFGF_CUDA(cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking));
            IFGF_CUDA(cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal));
            cudaGraph_t g = nullptr;
            bool ok = true;
            try {
                ifgf::run_apply(p, dens, out, p->cap_stream, !p->no_concurrency);
            } catch (const ifgf::Error&) {
                ok = false;
            }
            cudaError_t e = cudaStreamEndCapture(p->cap_stream, &g);
            if (ok && e == cudaSuccess && g) e = cudaGraphInstantiate(&p->gexec, g, 0);
            else ok = false;
            if (g) cudaGraphDestroy(g);
            if (!ok || e != cudaSuccess) {  // not capturable here: launch eagerly from now on
                p->gexec = nullptr;
                p->graph_failed = true;
                cudaGetLastError();
            } else {
                p->g_dens = dens;
                p->g_out = out;
            }
        }
        if (p->gexec) {
            IFGF_CUDA(cudaGraphLaunch(p->gexec, st));
            p->stats.graph_applies++;
            done = true;
        }
    }
    if (!done) ifgf::run_apply(p, dens, out, st, false);
    if (p->nccl_comm)  // the one exchange step of the source partition
        IFGF_NCCL(ncclAllReduce(out, out, (size_t)2 * p->n, ncclDouble, ncclSum, (ncclComm_t)p->nccl_comm, st));
}

// ------------------------------------------------------------ direct sum
constexpr int DIR_TPB = 256;
__global__ void k_direct_partial(const double* __restrict__ pts, int64_t n, double k, const double2* __restrict__ a,
                                 const int64_t* __restrict__ tg, int64_t chunk, double2* part) {
    int64_t t = blockIdx.y;
    int64_t l = tg[t];
    const double x = pts[3 * l], y = pts[3 * l + 1], z = pts[3 * l + 2];
    int64_t m0 = blockIdx.x * chunk, m1 = min(n, m0 + chunk);
    double sr = 0.0, si = 0.0;
    for (int64_t m = m0 + threadIdx.x; m < m1; m += blockDim.x) {
        if (m == l) continue;
        double dx = x - pts[3 * m], dy = y - pts[3 * m + 1], dz = z - pts[3 * m + 2];
        double r = sqrt(dx * dx + dy * dy + dz * dz);
        double s, c;
        sincos(k * r, &s, &c);
        double w = 0.079577471545947667884 / r;
        double2 am = a[m];
        sr += (am.x * c - am.y * s) * w;
        si += (am.x * s + am.y * c) * w;
    }
    __shared__ double rs[DIR_TPB], is[DIR_TPB];
    rs[threadIdx.x] = sr;
    is[threadIdx.x] = si;
    __syncthreads();
    for (int w = DIR_TPB / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) {
            rs[threadIdx.x] += rs[threadIdx.x + w];
            is[threadIdx.x] += is[threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) part[t * gridDim.x + blockIdx.x] = make_double2(rs[0], is[0]);
}
__global__ void k_direct_reduce(const double2* __restrict__ part, int64_t m, int nchunk, double2* out) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= m) return;
    double sr = 0.0, si = 0.0;
    for (int c = 0; c < nchunk; ++c) {
        double2 v = part[t * nchunk + c];
        sr += v.x;
        si += v.y;
    }
    out[t] = make_double2(sr, si);
}

// ------------------------------------------------------------- DFMA peak
__global__ void k_dfma(int64_t iters, double seed, double* sink) {
    double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
           a7 = a0 + 7;
    const double b = 0.9999999, c = 1e-7;
    for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
            a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        }
    }
    double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 1.2345) sink[0] = s;  // never true; keeps the chains alive
}
// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) throughput probe: 8 independent
// accumulator tiles per warp.
__global__ void k_dmma(int64_t iters, double seed, double* sink) {
    double a = seed + threadIdx.x * 1e-3, b = 0.5 + threadIdx.x * 1e-4;
    double c[8][2];
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = t;
    for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
        for (int t = 0; t < 8; ++t)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[t][0]), "+d"(c[t][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
    if (s == 1.2345) sink[0] = s;
}
}  // namespace

extern "C" ifgf_status ifgf_bench_dmma(int64_t iters, double* flops, double* ms, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    return guarded(nullptr, [&] {
        int dev = 0, nsm = 0;
        IFGF_CUDA(cudaGetDevice(&dev));
        IFGF_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        double* sink = nullptr;
        IFGF_CUDA(cudaMallocAsync((void**)&sink, sizeof(double), st));
        int blocks = nsm * 8, tpb = 256;
        k_dmma<<<blocks, tpb, 0, st>>>(iters / 10 + 1, 1.0, sink);
        cudaEvent_t e0, e1;
        IFGF_CUDA(cudaEventCreate(&e0));
        IFGF_CUDA(cudaEventCreate(&e1));
        IFGF_CUDA(cudaEventRecord(e0, st));
        k_dmma<<<blocks, tpb, 0, st>>>(iters, 1.0, sink);
        IFGF_CUDA(cudaEventRecord(e1, st));
        IFGF_CUDA(cudaEventSynchronize(e1));
        float t = 0.f;
        IFGF_CUDA(cudaEventElapsedTime(&t, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        IFGF_CUDA(cudaFreeAsync(sink, st));
        // per warp per mma: 8 x 8 x 4 FMA = 512 flops
        double f = 512.0 * 8.0 * (double)iters * blocks * (tpb / 32);
        if (flops) *flops = f / (t * 1e-3);
        if (ms) *ms = t;
    });
}

namespace ifgf {
void set_error(const std::string& msg) { g_last_error = msg; }
void dev_free(ifgf_plan_s* p, void* ptr) {
    for (auto& a : p->allocs)
        if (a == ptr) {
            cudaFree(a);
            a = nullptr;
        }
}
}  // namespace ifgf

extern "C" {

const char* ifgf_version(void) { return "ifgf-b200 0.1 (sm_100a)"; }

const char* ifgf_status_string(ifgf_status s) {
    switch (s) {
        case IFGF_OK: return "IFGF_OK";
        case IFGF_EINVAL: return "IFGF_EINVAL";
        case IFGF_EDOMAIN: return "IFGF_EDOMAIN";
        case IFGF_ENOMEM: return "IFGF_ENOMEM";
        case IFGF_ECUDA: return "IFGF_ECUDA";
        case IFGF_ENCCL: return "IFGF_ENCCL";
        case IFGF_EINTERNAL: return "IFGF_EINTERNAL";
    }
    return "IFGF_UNKNOWN";
}

const char* ifgf_last_error_message(void) { return g_last_error.c_str(); }

ifgf_status ifgf_opts_init(ifgf_opts* o) {
    if (!o) return fail(IFGF_EINVAL, "null opts");
    std::memset(o, 0, sizeof(*o));
    o->device = -1;
    return IFGF_OK;
}

ifgf_status ifgf_plan(const double* points, int64_t n, double k, int levels, int P_s, int P_ang,
                      const ifgf_opts* opts, ifgf_plan_t* plan_out) {
    if (!plan_out) return fail(IFGF_EINVAL, "null plan_out");
    *plan_out = nullptr;
    if (!points) return fail(IFGF_EINVAL, "null points");
    if (n < 1 || n > 2000000000LL) return fail(IFGF_EINVAL, "n out of range");
    if (levels < 1 || levels > IFGF_MAX_LEVELS) return fail(IFGF_EINVAL, "levels must be in [1, 22]");
    if (P_s < 1 || P_ang < 1 || P_s > ifgf::kMaxP1 || P_ang > ifgf::kMaxP1)
        return fail(IFGF_EINVAL, "P_s and P_ang must be in [1, 16]");
    if (!(k >= 0.0) || !std::isfinite(k)) return fail(IFGF_EINVAL, "k must be finite and >= 0");
    ifgf_opts o;
    ifgf_opts_init(&o);
    if (opts) o = *opts;
    if (o.leaf_ns < 0 || o.leaf_nc < 0) return fail(IFGF_EINVAL, "negative leaf grid");
    if (o.has_root && !(o.root_side > 0.0 && std::isfinite(o.root_side)))
        return fail(IFGF_EINVAL, "root_side must be positive");
    if (o.nranks > 1 && (o.rank < 0 || o.rank >= o.nranks)) return fail(IFGF_EINVAL, "rank out of range");
    ifgf_plan_s* p = new (std::nothrow) ifgf_plan_s();
    if (!p) return fail(IFGF_ENOMEM, "host allocation failed");
    if (o.device >= 0) p->device = o.device;
    else if (cudaGetDevice(&p->device) != cudaSuccess) {
        delete p;
        return fail(IFGF_ECUDA, "no CUDA device");
    }
    DeviceGuard dg(p->device);
    p->n = n;
    p->k = k;
    p->D = levels;
    p->Ps = P_s;
    p->Pa = P_ang;
    p->P = P_s * P_ang * P_ang;
    if (const char* e = std::getenv("IFGF_LEGACY_UPWARD")) p->legacy_upward = std::atoi(e);
    if (const char* e = std::getenv("IFGF_NO_SYMMETRY")) p->no_symmetry = std::atoi(e);
    if (const char* e = std::getenv("IFGF_EXACT_CLASSIFY")) p->cls_exact = std::atoi(e);
    if (const char* e = std::getenv("IFGF_TC_UMAX")) p->tc_umax = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("IFGF_STAGE_SLOTS")) p->stage_slots = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("IFGF_LEGACY_COUSIN")) p->legacy_cousin = std::atoi(e);
    p->stage_mask = o.stage_mask ? o.stage_mask : IFGF_STAGE_ALL;
    p->rank = o.nranks > 1 ? o.rank : 0;
    p->nranks = o.nranks > 1 ? o.nranks : 1;
    p->use_graph = !o.no_graph && !std::getenv("IFGF_NO_GRAPH");
    p->no_concurrency = std::getenv("IFGF_NO_CONCURRENCY") != nullptr;
    if (o.nccl_comm) {
        int cnt = 0, rk = 0;
        if (ncclCommCount((ncclComm_t)o.nccl_comm, &cnt) != ncclSuccess ||
            ncclCommUserRank((ncclComm_t)o.nccl_comm, &rk) != ncclSuccess) {
            delete p;
            return fail(IFGF_ENCCL, "nccl_comm is not a valid communicator");
        }
        if (cnt != p->nranks || rk != p->rank) {
            delete p;
            return fail(IFGF_EINVAL, "nccl_comm size / rank differ from nranks / rank");
        }
        p->nccl_comm = o.nccl_comm;
    }
    ifgf_status st = guarded(p, [&] {
        p->dev_bad = ifgf::dev_alloc<int>(p, 1);
        IFGF_CUDA(cudaMemset(p->dev_bad, 0, sizeof(int)));
        ifgf::build_plan(p, points, o);
        if (std::getenv("IFGF_PHASE_PROF")) {
            p->phase_clk = ifgf::dev_alloc<unsigned long long>(p, 16);
            IFGF_CUDA(cudaMemset(p->phase_clk, 0, 16 * sizeof(unsigned long long)));
        }
    });
    if (st != IFGF_OK) {
        free_plan(p);
        return st;
    }
    *plan_out = p;
    return IFGF_OK;
}

ifgf_status ifgf_apply(ifgf_plan_t p, const double* densities, double* out, void* stream) {
    if (!p || !densities || !out) return fail(IFGF_EINVAL, "null argument");
    if (p->sticky_cuda_error) return fail(IFGF_ECUDA, "plan is in a failed CUDA state");
    DeviceGuard dg(p->device);
    return guarded(p, [&] {
        apply_dispatch(p, reinterpret_cast<const double2*>(densities), reinterpret_cast<double2*>(out),
                       (cudaStream_t)stream);
    });
}

ifgf_status ifgf_apply_host(ifgf_plan_t p, const double* dh, double* oh, void* stream) {
    if (!p || !dh || !oh) return fail(IFGF_EINVAL, "null argument");
    if (p->sticky_cuda_error) return fail(IFGF_ECUDA, "plan is in a failed CUDA state");
    DeviceGuard dg(p->device);
    cudaStream_t st = (cudaStream_t)stream;
    ifgf_status s = guarded(p, [&] {
        if (!p->host_stage_dev_in) {
            p->host_stage_dev_in = ifgf::dev_alloc<double2>(p, p->n);
            p->host_stage_dev_out = ifgf::dev_alloc<double2>(p, p->n);
        }
        IFGF_CUDA(cudaMemcpyAsync(p->host_stage_dev_in, dh, sizeof(double2) * p->n, cudaMemcpyHostToDevice, st));
        apply_dispatch(p, p->host_stage_dev_in, p->host_stage_dev_out, st);
        IFGF_CUDA(cudaMemcpyAsync(oh, p->host_stage_dev_out, sizeof(double2) * p->n, cudaMemcpyDeviceToHost, st));
        IFGF_CUDA(cudaStreamSynchronize(st));
        int bad = 0;
        IFGF_CUDA(cudaMemcpy(&bad, p->dev_bad, sizeof(int), cudaMemcpyDeviceToHost));
        if (bad) throw ifgf::Error{IFGF_EINTERNAL, "apply met a point outside the relevant cone segments"};
    });
    return s;
}

ifgf_status ifgf_debug_level_pass(ifgf_plan_t p, int d, const double* values, unsigned what, double* field,
                                  double* parent) {
    if (!p || !values) return fail(IFGF_EINVAL, "null argument");
    if (d < 3 || d > p->D) return fail(IFGF_EINVAL, "level must be in [3, levels]");
    if ((what & 1) && !field) return fail(IFGF_EINVAL, "null field");
    if ((what & 2) && d > 3 && !parent) return fail(IFGF_EINVAL, "null parent");
    if (p->sticky_cuda_error) return fail(IFGF_ECUDA, "plan is in a failed CUDA state");
    DeviceGuard dg(p->device);
    return guarded(p, [&] {
        ifgf::debug_level_pass(p, d, reinterpret_cast<const double2*>(values), what, reinterpret_cast<double2*>(field),
                               reinterpret_cast<double2*>(parent));
    });
}

ifgf_status ifgf_nccl_unique_id(void* id_out) {
    if (!id_out) return fail(IFGF_EINVAL, "null id_out");
    static_assert(sizeof(ncclUniqueId) == IFGF_NCCL_ID_BYTES, "ncclUniqueId size");
    return guarded(nullptr, [&] {
        ncclUniqueId id;
        IFGF_NCCL(ncclGetUniqueId(&id));
        std::memcpy(id_out, &id, sizeof(id));
    });
}

ifgf_status ifgf_nccl_comm_create(const void* id, int nranks, int rank, int device, void** comm_out) {
    if (!id || !comm_out) return fail(IFGF_EINVAL, "null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(IFGF_EINVAL, "rank out of range");
    *comm_out = nullptr;
    DeviceGuard dg(device);
    return guarded(nullptr, [&] {
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        ncclComm_t c = nullptr;
        IFGF_NCCL(ncclCommInitRank(&c, nranks, uid, rank));
        *comm_out = c;
    });
}

ifgf_status ifgf_nccl_comm_destroy(void* comm) {
    if (!comm) return IFGF_OK;
    return guarded(nullptr, [&] { IFGF_NCCL(ncclCommDestroy((ncclComm_t)comm)); });
}

ifgf_status ifgf_plan_destroy(ifgf_plan_t p) {
    if (!p) return IFGF_OK;
    DeviceGuard dg(p->device);
    free_plan(p);
    return IFGF_OK;
}

ifgf_status ifgf_plan_stats(ifgf_plan_t p, ifgf_stats* s) {
    if (!p || !s) return fail(IFGF_EINVAL, "null argument");
    DeviceGuard dg(p->device);
    *s = p->stats;
    int bad = 0;
    if (cudaMemcpy(&bad, p->dev_bad, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess)
        return fail(IFGF_ECUDA, "cannot read the invariant flag");
    if (bad) return fail(IFGF_EINTERNAL, "an apply met a point outside the relevant cone segments");
    return IFGF_OK;
}

ifgf_status ifgf_plan_level_segments(ifgf_plan_t p, int d, int64_t* out, int64_t cap, int64_t* count) {
    if (!p || !count) return fail(IFGF_EINVAL, "null argument");
    if (d < 1 || d > p->D) return fail(IFGF_EINVAL, "level out of range");
    DeviceGuard dg(p->device);
    const ifgf::LevelParams& L = p->lev[d].p;
    *count = L.nseg;
    if (!out || cap < L.nseg || L.nseg == 0) return IFGF_OK;
    return guarded(p, [&] {
        std::vector<int> sb(L.nseg), sc(L.nseg), ijk(3 * L.nbox);
        IFGF_CUDA(cudaMemcpy(sb.data(), L.seg_box, sizeof(int) * L.nseg, cudaMemcpyDeviceToHost));
        IFGF_CUDA(cudaMemcpy(sc.data(), L.seg_cell, sizeof(int) * L.nseg, cudaMemcpyDeviceToHost));
        IFGF_CUDA(cudaMemcpy(ijk.data(), L.box_ijk, sizeof(int) * 3 * L.nbox, cudaMemcpyDeviceToHost));
        for (int64_t s = 0; s < L.nseg; ++s) {
            out[4 * s] = ijk[3 * sb[s]];
            out[4 * s + 1] = ijk[3 * sb[s] + 1];
            out[4 * s + 2] = ijk[3 * sb[s] + 2];
            out[4 * s + 3] = sc[s];
        }
    });
}

ifgf_status ifgf_profile_enable(ifgf_plan_t p, int enable) {
    if (!p) return fail(IFGF_EINVAL, "null plan");
    p->profile = enable ? 1 : 0;
    return IFGF_OK;
}

ifgf_status ifgf_profile_read(ifgf_plan_t p, double* ms, int64_t* launches, int reset) {
    if (!p) return fail(IFGF_EINVAL, "null plan");
    DeviceGuard dg(p->device);
    return guarded(p, [&] {
        for (auto& e : p->pending) {
            IFGF_CUDA(cudaEventSynchronize(e.b));
            float t = 0.f;
            IFGF_CUDA(cudaEventElapsedTime(&t, e.a, e.b));
            p->prof_ms[e.cls] += t;
            p->prof_launches[e.cls] += 1;
            p->ev_pool.push_back(e.a);
            p->ev_pool.push_back(e.b);
        }
        p->pending.clear();
        for (int c = 0; c < IFGF_NUM_KCLASS; ++c) {
            if (ms) ms[c] = p->prof_ms[c];
            if (launches) launches[c] = p->prof_launches[c];
            if (reset) {
                p->prof_ms[c] = 0;
                p->prof_launches[c] = 0;
            }
        }
    });
}

ifgf_status ifgf_direct(const double* points, int64_t n, double k, const double* dens, const int64_t* targets,
                        int64_t m, double* out, void* stream) {
    if (!points || !dens || !targets || !out || n < 1 || m < 0) return fail(IFGF_EINVAL, "bad argument");
    if (m == 0) return IFGF_OK;
    cudaStream_t st = (cudaStream_t)stream;
    return guarded(nullptr, [&] {
        int64_t chunk = 1 << 16;
        int nchunk = (int)((n + chunk - 1) / chunk);
        double2* part = nullptr;
        IFGF_CUDA(cudaMallocAsync((void**)&part, sizeof(double2) * m * nchunk, st));
        for (int64_t t0 = 0; t0 < m; t0 += 65535) {
            int64_t mt = std::min<int64_t>(65535, m - t0);
            dim3 g(nchunk, (unsigned)mt);
            k_direct_partial<<<g, DIR_TPB, 0, st>>>(points, n, k, reinterpret_cast<const double2*>(dens),
                                                    targets + t0, chunk, part + t0 * nchunk);
            IFGF_CUDA(cudaGetLastError());
        }
        k_direct_reduce<<<(int)((m + 255) / 256), 256, 0, st>>>(part, m, nchunk, reinterpret_cast<double2*>(out));
        IFGF_CUDA(cudaGetLastError());
        IFGF_CUDA(cudaFreeAsync(part, st));
    });
}

ifgf_status ifgf_partition(const double* w, int64_t nleaf, int nranks, int64_t* bounds) {
    if (!w || !bounds || nleaf < 0 || nranks < 1) return fail(IFGF_EINVAL, "bad argument");
    double total = 0.0;
    for (int64_t i = 0; i < nleaf; ++i) {
        if (!(w[i] >= 0.0) || !std::isfinite(w[i])) return fail(IFGF_EINVAL, "weights must be finite and >= 0");
        total += w[i];
    }
    // bounds[r] = first leaf whose prefix weight (exclusive) reaches r/R of the total
    bounds[0] = 0;
    double acc = 0.0;
    int r = 1;
    for (int64_t i = 0; i < nleaf && r < nranks; ++i) {
        while (r < nranks && acc + 0.5 * w[i] >= total * r / nranks) bounds[r++] = i;
        acc += w[i];
    }
    while (r < nranks) bounds[r++] = nleaf;
    bounds[nranks] = nleaf;
    for (int q = 1; q <= nranks; ++q)
        if (bounds[q] < bounds[q - 1]) bounds[q] = bounds[q - 1];
    return IFGF_OK;
}

ifgf_status ifgf_bench_dfma(int64_t iters, double* flops, double* ms, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    return guarded(nullptr, [&] {
        int dev = 0, nsm = 0;
        IFGF_CUDA(cudaGetDevice(&dev));
        IFGF_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        double* sink = nullptr;
        IFGF_CUDA(cudaMallocAsync((void**)&sink, sizeof(double), st));
        int blocks = nsm * 8, tpb = 256;
        k_dfma<<<blocks, tpb, 0, st>>>(iters / 10 + 1, 1.0, sink);  // warm-up
        cudaEvent_t e0, e1;
        IFGF_CUDA(cudaEventCreate(&e0));
        IFGF_CUDA(cudaEventCreate(&e1));
        IFGF_CUDA(cudaEventRecord(e0, st));
        k_dfma<<<blocks, tpb, 0, st>>>(iters, 1.0, sink);
        IFGF_CUDA(cudaEventRecord(e1, st));
        IFGF_CUDA(cudaEventSynchronize(e1));
        float t = 0.f;
        IFGF_CUDA(cudaEventElapsedTime(&t, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        IFGF_CUDA(cudaFreeAsync(sink, st));
        double f = 2.0 * 8.0 * 8.0 * (double)iters * blocks * tpb;
        if (flops) *flops = f / (t * 1e-3);
        if (ms) *ms = t;
    });
}

}  // extern "C"
