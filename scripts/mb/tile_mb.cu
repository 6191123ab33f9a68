// Microbenchmark of the TC K7 tile loop: A fragments from shared memory (LDS.64,
// row stride KP), B fragments (complex) held in registers, 4 accumulator chains,
// 38 DMMA per tile.  Reports DMMA per clock per SM (peak 0.25).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
constexpr int KS = 19, KP = 76, NW = 64;
template <int EPI>
__global__ void k(int tiles, double* out, const double2* gb) {
    __shared__ double sW[NW * KP];
    __shared__ double2 sV[8 * 75];
    for (int i = threadIdx.x; i < NW * KP; i += blockDim.x) sW[i] = 1e-3 * (i % 97);
    for (int i = threadIdx.x; i < 8 * 75; i += blockDim.x) sV[i] = make_double2(0, 0);
    __syncthreads();
    const int lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
    double2 b[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) b[ks] = gb[(threadIdx.x * KS + ks) % 4096];
    double sum = 0;
    for (int t = 0; t < tiles; ++t) {
        const int tile = t % 8;
        const double* wr = sW + (tile * 8 + gid) * KP + tig;
        double dr0 = 0, dr1 = 0, di0 = 0, di1 = 0, er0 = 0, er1 = 0, ei0 = 0, ei1 = 0;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            const double a = wr[4 * ks];
            if (ks & 1) { dmma(er0, er1, a, b[ks].x); dmma(ei0, ei1, a, b[ks].y); }
            else { dmma(dr0, dr1, a, b[ks].x); dmma(di0, di1, a, b[ks].y); }
        }
        if (EPI) {
            const int n = (tile * 8 + gid) % 75;
            double2 acc = sV[(2 * tig) * 75 + n];
            acc.x = fma(0.5, dr0 + er0, fma(-0.25, di0 + ei0, acc.x));
            acc.y = fma(0.5, di0 + ei0, fma(0.25, dr0 + er0, acc.y));
            sV[(2 * tig) * 75 + n] = acc;
            acc = sV[(2 * tig + 1) * 75 + n];
            acc.x = fma(0.5, dr1 + er1, fma(-0.25, di1 + ei1, acc.x));
            acc.y = fma(0.5, di1 + ei1, fma(0.25, dr1 + er1, acc.y));
            sV[(2 * tig + 1) * 75 + n] = acc;
        } else {
            sum += dr0 + dr1 + di0 + di1 + er0 + er1 + ei0 + ei1;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = sum + sV[threadIdx.x % 600].x;
}
template <int EPI> void run(int warps) {
    double* o; cudaMalloc(&o, 148 * 1024 * 8);
    double2* gb; cudaMalloc(&gb, 4096 * 16); cudaMemset(gb, 0, 4096 * 16);
    int tiles = 2000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k<EPI><<<148, 32 * warps>>>(tiles, o, gb);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double dmma = 148.0 * warps * tiles * 38;
        if (rep) printf("epilogue=%d warps/SM=%2d: %.3f DMMA/clk/SM (peak 0.25)\n", EPI, warps, dmma / 148 / (ms * 1e-3 * 1.965e9));
    }
}
int main() { for (int w : {4, 8, 12, 16}) { run<0>(w); run<1>(w); } return 0; }
