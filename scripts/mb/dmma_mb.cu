#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k(int iters, double* out, double a0, double b0) {
    double d[CH][2];
    for (int c = 0; c < CH; ++c) { d[c][0] = threadIdx.x; d[c][1] = c; }
    double a = a0 + threadIdx.x * 1e-9, b = b0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) dmma(d[c][0], d[c][1], a, b);
    }
    double s = 0; for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH>
__global__ void kf(int iters, double* out, double a0, double b0) {  // DFMA chains
    double d[CH];
    for (int c = 0; c < CH; ++c) d[c] = threadIdx.x + c;
    double a = a0 + threadIdx.x * 1e-9, b = b0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) d[c] = fma(d[c], a, b);
    }
    double s = 0; for (int c = 0; c < CH; ++c) s += d[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH> void run(int warps, bool f) {
    double* o; cudaMalloc(&o, 148 * 32 * 64 * 8);
    int iters = 4000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    if (f) kf<CH><<<148, 32 * warps>>>(iters, o, 0.999999, 1e-7); else k<CH><<<148, 32 * warps>>>(iters, o, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)148 * warps * iters * CH;  // warp-level instrs
    double clk = ms * 1e-3 * 1.965e9;
    if (rep) printf("%s chains=%d warps/SM=%2d : %.3f instr/clk/SM  (latency-est %.1f clk)\n", f ? "DFMA" : "DMMA", CH, warps, ops / 148 / clk, clk / iters);
    }
    cudaFree(o);
}
int main() {
    for (int w : {1, 2, 4, 8, 16, 32}) { run<1>(w, false); run<2>(w, false); run<4>(w, false); run<8>(w, false); }
    for (int w : {1, 4, 8, 16}) { run<1>(w, true); run<4>(w, true); run<8>(w, true); }
    return 0;
}
