/*
 * ifgf.h -- C ABI of the B200-native IFGF matvec library (libifgf.so).
 *
 * Computes, for N surface points x_l and complex densities a_m, the discrete
 * Helmholtz operator (PAPER.md eq. field1; eq. greensfunction,
 * P:305-307)
 *
 *     I(x_l) = sum_{m != l} a_m e^{i k |x_l - x_m|} / (4 pi |x_l - x_m|)
 *
 * by the Interpolated Factored Green Function method (Algorithm 1):
 * plan = box octree + cone-segment hierarchy + relevant segments;
 * apply = level-D near field and source-to-cone, then for d = D..3 cousin
 * interpolation and upward recentering.  Everything runs in
 * hand-written sm_100a CUDA kernels; all arithmetic is fp64 / complex128.
 *
 * Conventions
 *  - Every function returns ifgf_status (IFGF_OK == 0); no exception crosses
 *    the ABI.  ifgf_last_error_message() gives a human-readable reason
 *    (thread-local, valid until the next call on the same thread).
 *  - "device" pointers are CUDA device (or managed) pointers on the plan's
 *    device; "host" pointers are ordinary host memory.
 *  - Complex arrays are interleaved (re, im) fp64, i.e. complex128 layout.
 *  - Points are N x 3 row-major fp64 (x0, y0, z0, x1, ...).
 *  - A plan is immutable after ifgf_plan() returns and may be applied any
 *    number of times.  One apply at a time per plan (the plan
 *    owns the apply scratch); different plans may run concurrently.
 *  - IFGF_ECUDA is sticky: after it, only ifgf_plan_destroy() is meaningful.
 */
#ifndef IFGF_H_
#define IFGF_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ifgf_plan_s* ifgf_plan_t;

typedef enum {
    IFGF_OK = 0,
    IFGF_EINVAL = 1,    /* bad argument: n < 1, levels not in [1,22], P_s/P_ang < 1 or > 16,
                           k < 0 or non-finite, non-finite coordinates, null pointer   */
    IFGF_EDOMAIN = 2,   /* coincident points or a zero-extent cloud with n > 1 */
    IFGF_ENOMEM = 3,    /* device or host allocation failed; partial state freed         */
    IFGF_ECUDA = 4,     /* CUDA runtime error (sticky)                                   */
    IFGF_ENCCL = 5,     /* NCCL failure in the in-library all-reduce or communicator set-up
                           (sticky like IFGF_ECUDA)                                      */
    IFGF_EINTERNAL = 6  /* invariant violation (e.g. a cousin point or parent node whose
                           cone segment is not relevant); should be impossible          */
} ifgf_status;

/* Stage mask bits (debug / parity isolation).  0 means all stages. */
#define IFGF_STAGE_NEAR   1u  /* level-D near field                         */
#define IFGF_STAGE_COUSIN 2u  /* cousin-point interpolation at every level  */
#define IFGF_STAGE_UPWARD 4u  /* upward recentering d -> d-1                */
#define IFGF_STAGE_ALL    7u

typedef struct {
    int leaf_ns, leaf_nc;      /* leaf cone grid (n_s, n_C)_D; 0 -> (1, 2)       */
    int has_root;              /* nonzero: use root_center / root_side for the level-1 box     */
    double root_center[3];     /*   (P:1241-1245); else the bounding cube of reading R9        */
    double root_side;
    unsigned stage_mask;       /* IFGF_STAGE_* bits; 0 -> IFGF_STAGE_ALL                       */
    int device;                /* CUDA device ordinal; < 0 -> the current device               */
    int rank, nranks;          /* source partition (linearity of eq. field1,
                                  P:293-296): this process owns the rank-th contiguous,
                                  work-weighted Morton range of leaf boxes; nranks <= 1 -> all */
    void* nccl_comm;           /* ncclComm_t of the nranks processes (rank = its NCCL rank),
                                  borrowed: it must outlive the plan and is not destroyed by it
                                  (make one with ifgf_nccl_comm_create).  Non-null: ifgf_apply
                                  all-reduces the ranks' partial fields in place on cuda_stream,
                                  so every rank's out is the full field.  Null: out is this
                                  rank's partial field (the caller sums).                      */
    int no_graph;              /* nonzero: launch the apply's kernels one by one instead of
                                  replaying the plan's captured CUDA graph                      */
    int reserved[7];           /* must be zero                                                 */
} ifgf_opts;

/* Fill *opts with the defaults (all zero except device = -1). */
ifgf_status ifgf_opts_init(ifgf_opts* opts);

/*
 * Build a plan (T_pre of the paper) on the GPU.
 *   points : device, N x 3 row-major fp64, caller's order.  Copied; the caller
 *            may free it after the call returns.
 *   n      : number of points N >= 1.
 *   k      : wavenumber kappa >= 0 (kappa = 0 is the Laplace kernel 1/(4 pi r)).
 *   levels : number of octree levels D (root = level 1), 1 <= D <= 22.
 *   P_s, P_ang : Chebyshev nodes per cone segment in s and in each angle,
 *            1 <= P_s, P_ang <= 16; P = P_s * P_ang^2.
 *   opts   : nullable (defaults).
 *   plan_out : receives the plan handle (owned by the caller; destroy with
 *            ifgf_plan_destroy).
 * Synchronous: returns after the plan is complete on the device.
 */
ifgf_status ifgf_plan(const double* points, int64_t n, double k, int levels, int P_s, int P_ang,
                      const ifgf_opts* opts, ifgf_plan_t* plan_out);

/*
 * One operator application (T_acc): out = I(densities).
 *   densities : device, 2N fp64 (complex128), caller's point order. Borrowed
 *               until the work enqueued on cuda_stream completes.
 *   out       : device, 2N fp64 (complex128), caller's order; overwritten.
 *               With nranks > 1 and a communicator (opts.nccl_comm) it is the
 *               full field: the ranks' partial fields (sources of each owned
 *               leaf range) are summed by one in-place ncclAllReduce enqueued on
 *               cuda_stream after the kernels (every rank must call ifgf_apply).
 *               With nranks > 1 and no communicator it is this rank's partial
 *               field.
 *   cuda_stream : cudaStream_t to enqueue on (0 = legacy default stream).
 * Asynchronous with respect to the host.  The kernels of one apply are
 * captured once per (densities, out) pair into a CUDA graph owned by the plan
 * and replayed on cuda_stream (one launch instead of ~2 + 4(D-2); disabled by
 * opts.no_graph, while ifgf_profile_enable is on, or when capture is not
 * possible).  Errors: IFGF_EINVAL (null pointers), IFGF_ECUDA, IFGF_ENCCL
 * (sticky), IFGF_EINTERNAL is NOT detected here (the invariant flag is read by
 * ifgf_plan_stats and ifgf_apply_host).
 */
ifgf_status ifgf_apply(ifgf_plan_t plan, const double* densities, double* out, void* cuda_stream);

/*
 * End-to-end application from HOST buffers: copies densities (host, 2N fp64)
 * to the device, applies, copies the result back to out (host, 2N fp64) and
 * synchronises cuda_stream before returning.  Pinned host memory is faster
 * but not required.
 */
ifgf_status ifgf_apply_host(ifgf_plan_t plan, const double* densities_host, double* out_host, void* cuda_stream);

/*
 * NCCL communicator helpers (the library's own NCCL, so the communicator and
 * the all-reduce in ifgf_apply come from one NCCL instance).
 *   ifgf_nccl_unique_id  : id_out receives an ncclUniqueId (128 bytes, host);
 *                          call on one rank and broadcast the bytes (e.g. with
 *                          torch.distributed) to the others.
 *   ifgf_nccl_comm_create: collective over the nranks processes; device is the
 *                          CUDA ordinal this rank uses (< 0: current device);
 *                          *comm_out receives the ncclComm_t.
 *   ifgf_nccl_comm_destroy: releases it (after every plan using it is destroyed).
 * Errors: IFGF_EINVAL (null pointers, rank out of range), IFGF_ENCCL.
 */
#define IFGF_NCCL_ID_BYTES 128
ifgf_status ifgf_nccl_unique_id(void* id_out);
ifgf_status ifgf_nccl_comm_create(const void* id, int nranks, int rank, int device, void** comm_out);
ifgf_status ifgf_nccl_comm_destroy(void* comm);

/*
 * Test hook: one level's steps in isolation on caller-supplied node values
 * (SURVEY.md §8(c) exact pin 2, polynomial injection; Algorithm 1).
 *   d      : level, 3 <= d <= levels.
 *   values : host, nseg_d x P complex128 node values of level d's relevant
 *            segments in the order of ifgf_plan_level_segments, nodes s-fastest
 *            ((c P_ang + b) P_s + a for the a-th s, b-th theta, c-th phi
 *            first-kind Chebyshev node).  They replace the level's values and
 *            are fitted to Chebyshev coefficients (K5).
 *   what   : bit 0 -> K6 of level d alone: field (host, 2N fp64, caller order)
 *            = sum over (target, cousin box) pairs of Interp(x) G(x, c_B);
 *            bit 1 -> K7 d -> d-1 (d > 3): parent (host, nseg_{d-1} x P
 *            complex128) = level d-1's Chebyshev coefficients after the
 *            upward pass from these values alone (plus its fit).
 * Synchronous.  Overwrites the plan's apply scratch (not thread-safe with a
 * concurrent apply).  Errors: IFGF_EINVAL, IFGF_ECUDA.
 */
ifgf_status ifgf_debug_level_pass(ifgf_plan_t plan, int d, const double* values, unsigned what, double* field,
                                  double* parent);

/* Release every device and host resource of the plan.  Null is allowed. */
ifgf_status ifgf_plan_destroy(ifgf_plan_t plan);

/* Per-level algorithmic work counts (the roofline report divides these by time). */
#define IFGF_MAX_LEVELS 22
typedef struct {
    int64_t n;                 /* points                                                       */
    int levels, P_s, P_ang, P;
    double k, root_center[3], root_side;
    int64_t owned_leaf_begin, owned_leaf_end;          /* leaf-box range of this rank          */
    int64_t nbox[IFGF_MAX_LEVELS + 1];                 /* relevant boxes |R_B^d|               */
    int64_t nseg[IFGF_MAX_LEVELS + 1];                 /* relevant segments |R_C^d| (owned)   */
    int ns[IFGF_MAX_LEVELS + 1], nC[IFGF_MAX_LEVELS + 1]; /* cone grid (n_s, n_C) per level    */
    int64_t near_pairs;                                /* level-D (target, source) pairs       */
    int64_t s2c_pairs;                                 /* (leaf node, source) pairs            */
    int64_t cousin_evals[IFGF_MAX_LEVELS + 1];         /* (target, source box) interpolations  */
    int64_t upward_evals[IFGF_MAX_LEVELS + 1];         /* (parent node, child) d -> d-1        */
    int64_t segment_bytes[IFGF_MAX_LEVELS + 1];        /* 16 P |R_C^d|                         */
    int64_t plan_device_bytes;                         /* device memory held by the plan       */
    double plan_ms;                                    /* wall time of ifgf_plan               */
    int upward_kernel[IFGF_MAX_LEVELS + 1];            /* K7 kernel of the pass d -> d-1:
                                                          0 cell-grouped staged DFMA, 1 FP64
                                                          tensor-core GEMM, 2 per-evaluation
                                                          DFMA, 3 register-basis FP64 tensor-core
                                                          GEMM, -1 no pass (chosen at plan time) */
    uint64_t owned_morton_begin, owned_morton_end;     /* leaf Morton keys of the owned range,
                                                          half-open (key bit 3b+2/3b+1/3b = bit b
                                                          of i/j/k); [0, 2^64-1) with nranks <= 1 */
    int64_t graph_applies;                             /* applies replayed from the captured graph */
    double partition_weight_total, partition_weight_owned; /* work-weight units (ns, model) */
} ifgf_stats;

ifgf_status ifgf_plan_stats(ifgf_plan_t plan, ifgf_stats* stats);

/*
 * Relevant segments of level d (plan-diff against the oracle), host output:
 * out[4*s + 0..3] = (i, j, k, cell) with (i, j, k) the 0-based box multi-index
 * and cell = (i_phi * n_C + i_theta) * n_s + i_s.  Boxes in Morton order,
 * cells increasing within a box.  If out is null or cap < count, only *count
 * is written.
 */
ifgf_status ifgf_plan_level_segments(ifgf_plan_t plan, int d, int64_t* out, int64_t cap, int64_t* count);

/*
 * Per-kernel-class device time of the applies since the last reset, measured
 * with CUDA events recorded on the apply stream around each launch (enabled by
 * ifgf_profile_enable(plan, 1); disabled by default).  Classes:
 *   0 permute, 1 near (K3), 2 s2c (K4), 3 fit (K5), 4 cousin (K6),
 *   5 upward (K7), 6 unpermute.
 * ms[c] = total milliseconds, launches[c] = number of launches.
 */
#define IFGF_NUM_KCLASS 7
ifgf_status ifgf_profile_enable(ifgf_plan_t plan, int enable);
ifgf_status ifgf_profile_read(ifgf_plan_t plan, double* ms, int64_t* launches, int reset);

/*
 * Direct sum (measurement harness, PAPER.md eq. field1) at M target indices:
 * out[t] = sum_{m != targets[t]} a_m G(x_targets[t], x_m).
 *   points (device, N x 3), densities (device, 2N), targets (device, int64 M),
 *   out (device, 2M).  Asynchronous on cuda_stream.
 */
ifgf_status ifgf_direct(const double* points, int64_t n, double k, const double* densities,
                        const int64_t* targets, int64_t m, double* out, void* cuda_stream);

/*
 * Host-only: split nleaf work weights into nranks contiguous ranges of
 * near-equal weight.  bounds[0..nranks] (bounds[0] = 0, bounds[nranks] = nleaf).
 * Needs no GPU.
 */
ifgf_status ifgf_partition(const double* weights, int64_t nleaf, int nranks, int64_t* bounds);

/*
 * FP64 FMA throughput microbenchmark on the current device (the FP64 roofline
 * denominator): runs a DFMA-only kernel for ~iters iterations per thread and
 * returns achieved FP64 FLOP/s (FMA = 2 flops) and the kernel time.
 */
ifgf_status ifgf_bench_dfma(int64_t iters, double* flops_per_s, double* ms, void* cuda_stream);

/* Same for the FP64 tensor core (mma.sync m8n8k4 f64, DMMA): achieved FLOP/s. */
ifgf_status ifgf_bench_dmma(int64_t iters, double* flops_per_s, double* ms, void* cuda_stream);

const char* ifgf_status_string(ifgf_status s);
const char* ifgf_last_error_message(void);
const char* ifgf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* IFGF_H_ */
