// fastmath.cuh -- lean FP64 atan2 and sincos for the IFGF kernels.
//
// The classification contract makes every DISCRETE decision from
// IEEE-rounded + - * / sqrt against host-libm tables; the transcendental
// functions below only produce VALUES (local interpolation coordinates, phases),
// where the paper's method tolerates ulp-level differences (reading R12).  CUDA's
// libdevice atan2 / sincos spend ~125 / ~80 instructions on special cases (inf,
// NaN, denormals, Payne-Hanek reduction) that cannot occur here; these versions
// are branch-light polynomials:
//   fm_atan2: octant reduction to |t| <= tan(pi/8) with ONE division, then an odd
//             polynomial of degree 23 (near-minimax, Chebyshev-interpolated in
//             high precision; rel. error < 5e-18 before rounding), and one fused
//             k pi/4 +- p reconstruction; atan2_2pi maps to [0, 2 pi] directly.
//   fm_sincos: Cody-Waite reduction by pi/2 with a 3-part constant (FMA), then
//             degree-15 / degree-16 polynomials on |r| <= pi/4 (abs. error < 1e-17
//             before rounding); |x| >= 2^30 falls back to libdevice sincos.
// Coefficients were generated with mpmath (60 digits) by Chebyshev interpolation
// of (atan(t) - t)/t^3, (sin(r) - r)/r^3 and (cos(r) - 1 + r^2/2)/r^4 in t^2 / r^2.
// Both functions compile for host and device so that the CPU unit test
// (tests/test_fastmath_cpu.py) can check them against mpmath without a GPU.
#pragma once

#include <cmath>

#ifdef __CUDACC__
#define IFGF_HD __host__ __device__ __forceinline__
#else
#define IFGF_HD inline
#endif

namespace ifgf {
namespace fm {

constexpr double kTanPi8 = 0.41421356237309503;
constexpr double kPi4 = 0.7853981633974483, kPi4Lo = 3.061616997868383e-17;
constexpr double k2OverPi = 0.6366197723675814;
constexpr double kPio2_1 = 1.5707963267948966, kPio2_2 = 6.123233995736766e-17, kPio2_3 = -1.4973849048591698e-33;

// Polynomial coefficients (highest degree first), see the header comment.  On the
// device they live in constant memory so each DFMA reads its coefficient straight
// from the constant bank (no per-use 64-bit immediate materialisation).
#ifdef __CUDACC__
static __constant__ double kAtanQ_d[11] = {
    -0.019176887119062258989,
    0.039231658295587191303,
    -0.050854497379402598613,
    0.058581489128022098816,
    -0.066645114473819480001,
    0.076921831908260865637,
    -0.090909045781239018905,
    0.11111111015256361727,
    -0.14285714284666542922,
    0.19999999999995520678,
    -0.3333333333333333016};
#endif
static constexpr double kAtanQ_h[11] = {
    -0.019176887119062258989,
    0.039231658295587191303,
    -0.050854497379402598613,
    0.058581489128022098816,
    -0.066645114473819480001,
    0.076921831908260865637,
    -0.090909045781239018905,
    0.11111111015256361727,
    -0.14285714284666542922,
    0.19999999999995520678,
    -0.3333333333333333016};
#ifdef __CUDACC__
static __constant__ double kSinS_d[7] = {
    -7.5866970028175042058e-13,
    1.6058531617037151954e-10,
    -2.5052106232435281095e-8,
    2.7557319219339131119e-6,
    -0.00019841269841265064901,
    0.0083333333333333314921,
    -0.16666666666666666666};
#endif
static constexpr double kSinS_h[7] = {
    -7.5866970028175042058e-13,
    1.6058531617037151954e-10,
    -2.5052106232435281095e-8,
    2.7557319219339131119e-6,
    -0.00019841269841265064901,
    0.0083333333333333314921,
    -0.16666666666666666666};
#ifdef __CUDACC__
static __constant__ double kCosC_d[6] = {
    -1.1382632258093614476e-11,
    2.0876146266079308857e-9,
    -2.7557317271718642711e-7,
    0.000024801587298765666432,
    -0.0013888888888887397222,
    0.041666666666666665389};
#endif
static constexpr double kCosC_h[6] = {
    -1.1382632258093614476e-11,
    2.0876146266079308857e-9,
    -2.7557317271718642711e-7,
    0.000024801587298765666432,
    -0.0013888888888887397222,
    0.041666666666666665389};
#ifdef __CUDA_ARCH__
#define IFGF_FMC(name, i) name##_d[i]
#else
#define IFGF_FMC(name, i) name##_h[i]
#endif

// 1/sqrt(x) for finite x > 0 (values only): hardware approximation refined by one
// third-order step y (1 + e/2 + 3e^2/8), e = 1 - x y^2 (error ~e^3: ~1 ulp), without
// the special-case handling of the library rsqrt.
IFGF_HD double rsqrt_fast(double x) {
#ifdef __CUDA_ARCH__
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = std::fma(-x * y, y, 1.0);
    return std::fma(y * e, std::fma(0.375, e, 0.5), y);
#else
    return 1.0 / std::sqrt(x);
#endif
}

// Flip the sign of x when flip is true (one integer xor on the high word).
IFGF_HD double flip_sign(double x, bool flip) {
#ifdef __CUDA_ARCH__
    return __hiloint2double(__double2hiint(x) ^ (flip ? (int)0x80000000 : 0), __double2loint(x));
#else
    return flip ? -x : x;
#endif
}

// Shared core of atan2 / atan2_2pi: for (x, y) != (0, 0) returns p = atan(t) of the
// reduced argument |t| <= tan(pi/8) and the octant data such that
//   atan2(|y|, x) = k pi/4 + sg p,  k in {0, ..., 4}, sg = +-1.
// One compare replaces fmax/fmin (no NaN handling needed); the octant fix-ups are
// integer selects and ONE fused k pi/4 add (k * kPi4 is exact for k <= 4: the
// significand of kPi4 ends in three zero bits), instead of three hi/lo additions.
IFGF_HD double atan2_core(double y, double x, int* kq, bool* neg) {
    const double ax = std::fabs(x), ay = std::fabs(y);
    const bool sw = ay > ax;
    const double mx = sw ? ay : ax, mn = sw ? ax : ay;
    const bool big = mn > kTanPi8 * mx;  // reduce via atan(t) = pi/4 + atan((t-1)/(t+1))
    const double num = big ? mn - mx : mn, den = big ? mn + mx : mx;
#ifdef __CUDA_ARCH__
    // value only: hardware reciprocal + two Newton steps (~1 ulp) instead of an IEEE division
    double rd;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rd) : "d"(den));
    double e = std::fma(-den, rd, 1.0);
    rd = std::fma(rd, e, rd);
    e = std::fma(-den, rd, 1.0);
    rd = std::fma(rd, e, rd);
    const double t = num * rd;
#else
    const double t = num / den;
#endif
    const double s = t * t;
    double q = IFGF_FMC(kAtanQ, 0);
    q = std::fma(q, s, IFGF_FMC(kAtanQ, 1));
    q = std::fma(q, s, IFGF_FMC(kAtanQ, 2));
    q = std::fma(q, s, IFGF_FMC(kAtanQ, 3));
    q = std::fma(q, s, IFGF_FMC(kAtanQ, 4));
    q = std::fma(q, s, IFGF_FMC(kAtanQ, 5));
    q = std::fma(q, s, IFGF_FMC(kAtanQ, 6));
    q = std::fma(q, s, IFGF_FMC(kAtanQ, 7));
    q = std::fma(q, s, IFGF_FMC(kAtanQ, 8));
    q = std::fma(q, s, IFGF_FMC(kAtanQ, 9));
    q = std::fma(q, s, IFGF_FMC(kAtanQ, 10));
    // atan(mn/mx) = big pi/4 + p; swapped: pi/2 - that; x < 0: pi - that
    int k = big ? 1 : 0;
    bool ng = false;
    if (sw) {
        k = 2 - k;
        ng = true;
    }
    if (x < 0.0) {
        k = 4 - k;
        ng = !ng;
    }
    *kq = k;
    *neg = ng;
    return std::fma(t * s, q, t);
}

IFGF_HD double octant_sum(int k, bool neg, double p) {
    const double kd = (double)k;
    return std::fma(kd, kPi4, std::fma(kd, kPi4Lo, flip_sign(p, neg)));
}

// atan2(y, x) in [-pi, pi]; (x, y) != (0, 0).
IFGF_HD double atan2(double y, double x) {
    int k;
    bool ng;
    const double p = atan2_core(y, x, &k, &ng);
    return std::copysign(octant_sum(k, ng, p), y);
}

// atan2(y, x) mapped to [0, 2 pi] (y < 0: 2 pi - |atan2|); (x, y) != (0, 0).
IFGF_HD double atan2_2pi(double y, double x) {
    int k;
    bool ng;
    const double p = atan2_core(y, x, &k, &ng);
    if (y < 0.0) {
        k = 8 - k;
        ng = !ng;
    }
    return octant_sum(k, ng, p);
}

// sin and cos of x (any finite x).
IFGF_HD void sincos(double x, double* sp, double* cp) {
    const double q = std::rint(x * k2OverPi);
    if (!(std::fabs(q) < 1073741824.0)) {  // |x| >~ 1.7e9 (or non-finite): full reduction
#ifdef __CUDA_ARCH__
        ::sincos(x, sp, cp);
#else
        *sp = std::sin(x);
        *cp = std::cos(x);
#endif
        return;
    }
    double r = std::fma(-q, kPio2_1, x);
    r = std::fma(-q, kPio2_2, r);
    r = std::fma(-q, kPio2_3, r);
    const double s = r * r;
    double ps = IFGF_FMC(kSinS, 0);
    ps = std::fma(ps, s, IFGF_FMC(kSinS, 1));
    ps = std::fma(ps, s, IFGF_FMC(kSinS, 2));
    ps = std::fma(ps, s, IFGF_FMC(kSinS, 3));
    ps = std::fma(ps, s, IFGF_FMC(kSinS, 4));
    ps = std::fma(ps, s, IFGF_FMC(kSinS, 5));
    ps = std::fma(ps, s, IFGF_FMC(kSinS, 6));
    double pc = IFGF_FMC(kCosC, 0);
    pc = std::fma(pc, s, IFGF_FMC(kCosC, 1));
    pc = std::fma(pc, s, IFGF_FMC(kCosC, 2));
    pc = std::fma(pc, s, IFGF_FMC(kCosC, 3));
    pc = std::fma(pc, s, IFGF_FMC(kCosC, 4));
    pc = std::fma(pc, s, IFGF_FMC(kCosC, 5));
    const double sn = std::fma(r * s, ps, r);
    const double cs = std::fma(s * s, pc, std::fma(-0.5, s, 1.0));
    const int iq = (int)(long long)q & 3;
    const double a = (iq & 1) ? cs : sn, b = (iq & 1) ? sn : cs;
    *sp = flip_sign(a, iq & 2);
    *cp = flip_sign(b, (iq + 1) & 2);
}

}  // namespace fm
}  // namespace ifgf
