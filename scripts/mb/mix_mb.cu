// Do DMMA (FP64 tensor core) and DFMA share one pipe on B200?  Blocks of 8 warps:
// mode 0: all warps DFMA; mode 1: all warps DMMA; mode 2: warps 0-3 DFMA, 4-7 DMMA
// (same per-warp work as in modes 0/1).  If the pipes were separate, mode 2 would
// take about half of (mode 0 + mode 1) time; if shared, about the sum of halves.
#include <cstdio>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void k(int mode, long iters_f, long iters_m, double* sink) {
    const int w = threadIdx.x >> 5;
    const bool do_m = mode == 1 || (mode == 2 && w >= 4);
    double s = 0;
    if (!do_m) {
        double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
        for (long i = 0; i < iters_f; ++i) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                a0 = fma(a0, 0.9999, 1e-7); a1 = fma(a1, 0.9999, 1e-7); a2 = fma(a2, 0.9999, 1e-7); a3 = fma(a3, 0.9999, 1e-7);
                a4 = fma(a4, 0.9999, 1e-7); a5 = fma(a5, 0.9999, 1e-7); a6 = fma(a6, 0.9999, 1e-7); a7 = fma(a7, 0.9999, 1e-7);
            }
        }
        s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    } else {
        double c[8][2];
        for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = t;
        double a = threadIdx.x * 1e-3, b = 0.5;
        for (long i = 0; i < iters_m; ++i) {
#pragma unroll
            for (int t = 0; t < 8; ++t) dmma(c[t][0], c[t][1], a, b);
        }
        for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
    }
    if (s == 1.2345) sink[0] = s;
}
int main() {
    double* sink;
    cudaMalloc(&sink, 8);
    // per warp: DFMA work = iters_f * 64 FMA instr (warp) = 64 * 32 FMAs; DMMA work = iters_m * 8 * 256 FMA
    long itf = 20000, itm = 20000 * 64 * 32 / (8 * 256);  // equal FMA counts per warp
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 3; ++mode) {
        k<<<148 * 4, 256>>>(mode, itf / 10, itm / 10, sink);
        cudaEventRecord(e0);
        k<<<148 * 4, 256>>>(mode, itf, itm, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double fma = (double)148 * 4 * 8 * (double)itf * 64 * 32;  // same FMA count in every mode
        printf("mode %d (%s): %.3f ms, %.2f TFLOP/s\n", mode, mode == 0 ? "DFMA" : mode == 1 ? "DMMA" : "half/half",
               ms, 2 * fma / (ms * 1e-3) / 1e12);
    }
    return 0;
}
