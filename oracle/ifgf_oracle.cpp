// =============================================================================
// ifgf_oracle.cpp -- plain fp64 CPU oracle of the IFGF operator evaluation
// (Bauinger & Bruno, arXiv 2010.02857); serial, or OpenMP with bitwise the
// serial result.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load this library.
// The product path (paper_2010_02857_b200/, libifgf.so) never links, imports
// or executes anything under oracle/.  The two share NO code: no headers, no
// tables, no helpers.  Where both must take the same discrete decision (box
// membership, cone-segment classification) they implement the same written
// specification independently.
//
// Citations "P:n" are lines of /root/reference/PAPER.md (with the equation /
// section label they fall in).  Readings of silent/garbled passages are the
// "R<n>" entries of DESIGN.md (same numbering as SURVEY.md §8(c)).
//
// Build: g++ -O2 -std=c++17 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
// (FMA contraction off so that every discrete decision is the IEEE result of
// the written formula).
//
// Loop order and threads (SURVEY.md §8(c) "Oracle data layout and cost"): the
// near field and the cousin evaluations are TARGET-major (for each target box,
// its neighbour / cousin source boxes in increasing box order; both relations
// are symmetric), the upward pass is PARENT-SEGMENT-major (for each
// parent segment and node, its children in increasing box order).  Every output
// (I(x_l), a parent node value) therefore has exactly one owner and receives its
// terms in the same order as the source-major serial loops of Algorithm 1
// -- the sums are bitwise those of the literal loop nest, at any
// thread count.  OpenMP only distributes owners over threads
// (oracle_set_threads; 1 = serial).  Work that the paper defines per box but
// that is box-independent (node offsets, and a parent node's child cell,
// local coordinates and recentering factor per (level, parent cell, child
// octant)) is computed once and reused: same calls, same bits.
//
// Parity pins (tests/test_oracle_*.py): closed forms of G and g_S, the
// factorisation identity, Chebyshev node reproduction / polynomial exactness /
// eq. 19 bound, brute-force tree relations, bypass mode == direct sum,
// exact-recentering check, centred-source exact case, convergence in (P_s,P_ang),
// metamorphic rotation symmetry; the parallel mode equals the serial mode
// bitwise, the fast classification equals the literal interval scans
// (incl. boundary ties), and a source-partitioned plan equals the masked
// densities exactly (tests/test_oracle_parallel.py).  Every function below is
// pinned by at least one of those; none is "parity unpinned".
// =============================================================================
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <omp.h>
#include <parallel/algorithm>
#include <string>
#include <tuple>
#include <vector>

namespace {

using cplx = std::complex<double>;

enum Status { OK = 0, EINVAL_ = 1, EDOMAIN_ = 2, ENOMEM_ = 3, EINTERNAL_ = 6 };

const double PI = 3.14159265358979323846;

// ---------------------------------------------------------------------------
// L0: kernel math
// ---------------------------------------------------------------------------

// Helmholtz Green function, eq. greensfunction:
//   G(x,x') = e^{i kappa |x-x'|} / (4 pi |x-x'|)
cplx green_r(double r, double k) {
    return cplx(std::cos(k * r), std::sin(k * r)) / (4.0 * PI * r);
}

double norm3(const double v[3]) { return std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]); }

// |v - w| - |v| without cancellation, via the identity a - b = (a^2 - b^2)/(a + b)
// with |v-w|^2 - |v|^2 = w.w - 2 v.w.  (Reading R17: the phase of the analytic
// factor / recentering ratio is evaluated in this algebraically identical form
// because |v| can exceed |w| by 10^4 at coarse levels.)
double dist_minus_norm(const double v[3], const double w[3], double* dvw) {
    double d[3] = {v[0] - w[0], v[1] - w[1], v[2] - w[2]};
    double a = norm3(d), b = norm3(v);
    double num = (w[0] * w[0] + w[1] * w[1] + w[2] * w[2]) - 2.0 * (v[0] * w[0] + v[1] * w[1] + v[2] * w[2]);
    if (dvw) *dvw = a;
    return num / (a + b);
}

// Analytic factor, eq. factored_f, centred at c, written with
// v = x - c and w = x' - c:   g_S = (|v| / |v - w|) e^{i kappa (|v-w| - |v|)}.
// (Reading R3: the 1/(4 pi) of eqs factor_r / factor_r_eps is
// spurious; G = G(x,c) g_S holds exactly with this form.)
cplx analytic_factor_rel(const double v[3], const double w[3], double k) {
    double dvw;
    double diff = dist_minus_norm(v, w, &dvw);
    double ratio = norm3(v) / dvw;
    return ratio * cplx(std::cos(k * diff), std::sin(k * diff));
}

// ---------------------------------------------------------------------------
// L1: Chebyshev interpolation
// ---------------------------------------------------------------------------

// First-kind Chebyshev nodes x_k = cos((2k+1) pi / (2n)), k = 0..n-1.
std::vector<double> cheb_nodes(int n) {
    std::vector<double> t(n);
    for (int k = 0; k < n; ++k) t[k] = std::cos((2.0 * k + 1.0) * PI / (2.0 * n));
    return t;
}

// T_i(x) = cos(i arccos x), via the three-term recurrence (identical
// polynomial; valid for x a few ulps outside [-1,1]).
void cheb_T(int n, double x, double* T) {
    if (n > 0) T[0] = 1.0;
    if (n > 1) T[1] = x;
    for (int i = 2; i < n; ++i) T[i] = 2.0 * x * T[i - 1] - T[i - 2];
}

// Reading R1: eq. defchebyshevcoeffsandpoints is garbled (it mixes
// first-kind nodes with Lobatto weights and does not reproduce node values).
// The interpolant at the first-kind nodes is unique; its coefficients are
//   a_i = ((2 - delta_{i0}) / n) sum_k u(x_k) T_i(x_k).
const int MAXP = 16;  // P_s, P_ang <= 16 (include/ifgf.h)

// T_i(x_k) at the first-kind nodes of every n <= MAXP, computed once (the same
// calls as computing them per fit, so the same bits).
struct ChebTables {
    double T[MAXP + 1][MAXP][MAXP];
    ChebTables() {
        for (int n = 1; n <= MAXP; ++n) {
            std::vector<double> t = cheb_nodes(n);
            for (int k = 0; k < n; ++k) cheb_T(n, t[k], T[n][k]);
        }
    }
};
const ChebTables& cheb_tables() {
    static const ChebTables tb;  // thread-safe one-time initialisation
    return tb;
}

void cheb_fit1d(int n, const cplx* u, cplx* a) {
    const ChebTables& tb = cheb_tables();
    for (int i = 0; i < n; ++i) a[i] = 0.0;
    for (int k = 0; k < n; ++k) {
        const double* T = tb.T[n][k];
        for (int i = 0; i < n; ++i) a[i] += u[k] * T[i];
    }
    for (int i = 0; i < n; ++i) a[i] *= (i == 0 ? 1.0 : 2.0) / n;
}

// I_n u(x) = sum_{i<n} a_i T_i(x)  (eq. defchebyshevinterpooperator).
cplx cheb_eval1d(int n, const cplx* a, double x) {
    std::vector<double> T(n);
    cheb_T(n, x, T.data());
    cplx s = 0.0;
    for (int i = 0; i < n; ++i) s += a[i] * T[i];
    return s;
}

// Node values / coefficients of one cone segment are stored s-fastest:
//   index(ks, it, jp) = (jp * Pang + it) * Ps + ks.
// Nested 1-D fits along s, then theta, then phi (Theorem
// errorestimatenested P:732-746; reading R2: order irrelevant on a tensor grid).
void tensor_fit(int Ps, int Pa, const cplx* V, cplx* C) {
    cplx A[MAXP * MAXP * MAXP], in[MAXP], out[MAXP];
    std::copy(V, V + Ps * Pa * Pa, A);
    for (int jp = 0; jp < Pa; ++jp)  // along s
        for (int it = 0; it < Pa; ++it) {
            for (int ks = 0; ks < Ps; ++ks) in[ks] = A[(jp * Pa + it) * Ps + ks];
            cheb_fit1d(Ps, in, out);
            for (int ks = 0; ks < Ps; ++ks) A[(jp * Pa + it) * Ps + ks] = out[ks];
        }
    for (int jp = 0; jp < Pa; ++jp)  // along theta
        for (int ks = 0; ks < Ps; ++ks) {
            for (int it = 0; it < Pa; ++it) in[it] = A[(jp * Pa + it) * Ps + ks];
            cheb_fit1d(Pa, in, out);
            for (int it = 0; it < Pa; ++it) A[(jp * Pa + it) * Ps + ks] = out[it];
        }
    for (int it = 0; it < Pa; ++it)  // along phi
        for (int ks = 0; ks < Ps; ++ks) {
            for (int jp = 0; jp < Pa; ++jp) in[jp] = A[(jp * Pa + it) * Ps + ks];
            cheb_fit1d(Pa, in, out);
            for (int jp = 0; jp < Pa; ++jp) A[(jp * Pa + it) * Ps + ks] = out[jp];
        }
    std::copy(A, A + Ps * Pa * Pa, C);
}

// Plain triple sum ("simple evaluations of triple sums"), from the
// three 1-D Chebyshev vectors T_i(u_s), T_i(u_theta), T_i(u_phi).
cplx tensor_eval_T(int Ps, int Pa, const cplx* C, const double* Ts, const double* Tt, const double* Tp) {
    cplx s = 0.0;
    for (int jp = 0; jp < Pa; ++jp)
        for (int it = 0; it < Pa; ++it)
            for (int ks = 0; ks < Ps; ++ks) s += C[(jp * Pa + it) * Ps + ks] * (Ts[ks] * Tt[it] * Tp[jp]);
    return s;
}

cplx tensor_eval(int Ps, int Pa, const cplx* C, double us, double ut, double up) {
    double Ts[MAXP], Tt[MAXP], Tp[MAXP];
    cheb_T(Ps, us, Ts);
    cheb_T(Pa, ut, Tt);
    cheb_T(Pa, up, Tp);
    return tensor_eval_T(Ps, Pa, C, Ts, Tt, Tp);
}

// ---------------------------------------------------------------------------
// Cone grids and classification (reading R7 +
// DESIGN.md "Classification contract")
// ---------------------------------------------------------------------------
struct Grid {
    int ns = 1, nC = 2;
    double H = 0, h = 0, ds = 0, dth = 0;  // box side H_d, radius h_d (eq. def_eps), spans
    std::vector<double> cos_tb;            // cos(k dtheta), k = 0..nC    (theta boundaries)
    std::vector<double> cos_pb, sin_pb;    // cos/sin(j dphi), j = 0..2nC (phi boundaries)
    // Node tables of eq. interp_pts, filled by node_tables():
    // r(is, ks) = h / s_k, sin/cos theta_i (ith, it), cos/sin phi_j (iph, jp).
    std::vector<double> nr, nst, nct, ncp, nsp;
};

// (c, s) rotated by q quarter turns about z: (c, s) -> (-s, c) per turn (exact).
void quarter_turns(double c, double s, int q, double* co, double* so) {
    switch (q & 3) {
        case 0: *co = c; *so = s; break;
        case 1: *co = -s; *so = c; break;
        case 2: *co = -c; *so = -s; break;
        default: *co = s; *so = -c; break;
    }
}

void grid_tables(Grid& g) {
    const double eta = std::sqrt(3.0) / 3.0;  // eta = sqrt(3)/3
    g.h = std::sqrt(3.0) / 2.0 * g.H;         // h = (sqrt(3)/2) H (eq. def_eps)
    g.ds = eta / g.ns;                        // Delta_s = eta / n_s
    g.dth = PI / g.nC;                        // Delta_theta = Delta_phi = pi / n_C
    g.cos_tb.assign(g.nC + 1, 0.0);
    for (int k = 0; k <= g.nC; ++k) g.cos_tb[k] = std::cos((double)k * PI / (double)g.nC);
    g.cos_pb.assign(2 * g.nC + 1, 0.0);
    g.sin_pb.assign(2 * g.nC + 1, 0.0);
    if (g.nC % 2 == 0) {
        // n_C even: exact quarter-turn symmetry of the boundary rays (reading R18):
        // phi_j = q pi/2 + phi_jr with jr < n_C/2; (cos, sin) of phi_jr from libm,
        // rotated by q quarter turns ((c, s) -> (-s, c)), which is exact.
        const int hq = g.nC / 2;
        for (int j = 0; j <= 2 * g.nC; ++j) {
            const int q = (j / hq) & 3, jr = j % hq;
            const double a = (double)jr * PI / (double)g.nC;
            quarter_turns(std::cos(a), std::sin(a), q, &g.cos_pb[j], &g.sin_pb[j]);
        }
        return;
    }
    for (int j = 0; j < g.nC; ++j) {
        double a = (double)j * PI / (double)g.nC;
        g.cos_pb[j] = std::cos(a);
        g.sin_pb[j] = std::sin(a);
        g.cos_pb[j + g.nC] = -g.cos_pb[j];  // exact half-turn symmetry of the boundary rays
        g.sin_pb[j + g.nC] = -g.sin_pb[j];
    }
    g.cos_pb[2 * g.nC] = g.cos_pb[0];
    g.sin_pb[2 * g.nC] = g.sin_pb[0];
}

struct Cls {
    int is, it, ip;        // interval indices (0-based gamma - 1)
    double us, ut, up;     // local coordinates in [-1,1] of (s, theta, phi)
    double r, s;
};

// phi interval by its definition: the unique j with cross_j >= 0 > cross_{j+1},
// cross_j = v_y cos(j dphi) - v_x sin(j dphi); no such j (poles) -> 0.
bool phi_sector_is(const Grid& g, const double v[3], int j) {
    double cj = v[1] * g.cos_pb[j] - v[0] * g.sin_pb[j];
    double cj1 = v[1] * g.cos_pb[j + 1] - v[0] * g.sin_pb[j + 1];
    return cj >= 0.0 && cj1 < 0.0;
}

int phi_sector_scan(const Grid& g, const double v[3]) {
    for (int j = 0; j < 2 * g.nC; ++j)
        if (phi_sector_is(g, v, j)) return j;
    return 0;
}

// phi = atan2(y, x) in [0, 2 pi) (reading R13).
double phi_of(const double v[3]) {
    double ph = std::atan2(v[1], v[0]);
    if (ph < 0.0) ph += 2.0 * PI;
    return ph;
}

// Local coordinates (reading R13: theta = atan2(rho, z), phi as phi_of).
void local_coords(const Grid& g, const double v[3], double ph, Cls& c) {
    double rho = std::sqrt(v[0] * v[0] + v[1] * v[1]);
    double th = std::atan2(rho, v[2]);
    if (v[0] == 0.0 && v[1] == 0.0) ph = 0.0;  // poles: phi := 0 (reading R7)
    c.us = 2.0 * (c.s - c.is * g.ds) / g.ds - 1.0;
    c.ut = 2.0 * (th - c.it * g.dth) / g.dth - 1.0;
    c.up = 2.0 * (ph - c.ip * g.dth) / g.dth - 1.0;
}

// Cone segment containing the point with relative vector v = x - x_k^d
// ("simple arithmetic operations in spherical coordinates"), by the
// literal interval scans of the classification contract.
// Intervals are half-open lower-closed (eq. defconedomain, reading R7).
Cls classify_scan(const Grid& g, const double v[3]) {
    Cls c;
    c.r = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    c.s = g.h / c.r;  // s = h / r (eq. defparametrizationins)
    c.is = (int)std::floor(c.s / g.ds);
    if (c.is > g.ns - 1) c.is = g.ns - 1;  // s = eta closes the last interval
    // theta interval: theta >= k dtheta  <=>  cos(theta) <= cos(k dtheta)
    double ct = v[2] / c.r;
    c.it = 0;
    for (int k = 1; k < g.nC; ++k)
        if (ct <= g.cos_tb[k]) c.it = k;
    c.ip = phi_sector_scan(g, v);
    local_coords(g, v, phi_of(v), c);
    return c;
}

// The same decisions, found faster (tests/test_oracle_units.py pins equality
// with classify_scan on random and boundary-tie vectors):
//  - i_theta = #{k in 1..nC-1 : v_z/r <= cos(k dtheta)}; cos(k dtheta) is
//    decreasing in k, so that set is a prefix {1..K} and K is found by bisection;
//  - i_phi: the defining condition is tested at the atan2 guess and its two
//    neighbours; the sector is unique, so a hit is the scan's answer; no hit
//    (poles, or a guess off by more than one) falls back to the scan.
Cls classify(const Grid& g, const double v[3]) {
    Cls c;
    c.r = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    c.s = g.h / c.r;
    c.is = (int)std::floor(c.s / g.ds);
    if (c.is > g.ns - 1) c.is = g.ns - 1;
    double ct = v[2] / c.r;
    int lo = 0, hi = g.nC - 1;  // invariant: all k <= lo satisfy (k = 0 vacuous), all k > hi fail
    while (lo < hi) {
        int mid = (lo + hi + 1) / 2;
        if (ct <= g.cos_tb[mid]) lo = mid; else hi = mid - 1;
    }
    c.it = lo;
    const int n2 = 2 * g.nC;
    const double ph = phi_of(v);
    int guess = (int)std::floor(ph / g.dth);
    if (guess < 0) guess = 0;
    if (guess > n2 - 1) guess = n2 - 1;
    c.ip = -1;
    const int cand[3] = {guess, (guess + n2 - 1) % n2, (guess + 1) % n2};
    for (int j : cand)
        if (phi_sector_is(g, v, j)) { c.ip = j; break; }
    if (c.ip < 0) c.ip = phi_sector_scan(g, v);
    local_coords(g, v, ph, c);
    return c;
}

int64_t cell_lin(const Grid& g, int is, int it, int ip) { return ((int64_t)ip * g.nC + it) * g.ns + is; }

// ---------------------------------------------------------------------------
// L2: box octree
// ---------------------------------------------------------------------------
struct Box {
    int64_t i, j, k;          // 0-based multi-index (the paper's k - 1)
    std::vector<int> pts;     // point indices, increasing
    int parent = -1;
    std::vector<int> children, nbrs, cousins;
    std::vector<int64_t> segs;  // relevant cone segments R_C B (sorted cell_lin)
    bool active = true;         // has an owned leaf (source partition)
};

// Morton key of a leaf multi-index (bit b of i, j, k -> bits 3b+2, 3b+1, 3b);
// the source partition owns a half-open range of these keys.
uint64_t morton_key(int64_t i, int64_t j, int64_t k) {
    uint64_t r = 0;
    for (int b = 0; b < 21; ++b)
        r |= ((uint64_t)((i >> b) & 1) << (3 * b + 2)) | ((uint64_t)((j >> b) & 1) << (3 * b + 1)) |
             ((uint64_t)((k >> b) & 1) << (3 * b));
    return r;
}

// Box multi-index packed into one key, (i, j, k) lexicographic = key order
// (0 <= i, j, k < 2^21 since D <= 22).
uint64_t box_key(int64_t i, int64_t j, int64_t k) { return ((uint64_t)i << 42) | ((uint64_t)j << 21) | (uint64_t)k; }

struct Level {
    std::vector<Box> boxes;     // relevant boxes in (i, j, k) lexicographic order
    std::vector<uint64_t> keys; // box_key of boxes[b] (increasing)
    int64_t side = 1;           // 2^{d-1} boxes per axis
    Grid g;
    int find(int64_t i, int64_t j, int64_t k) const {
        if (i < 0 || j < 0 || k < 0 || i >= side || j >= side || k >= side) return -1;
        uint64_t key = box_key(i, j, k);
        auto it = std::lower_bound(keys.begin(), keys.end(), key);
        return (it == keys.end() || *it != key) ? -1 : (int)(it - keys.begin());
    }
};

}  // namespace

struct oracle_plan {
    int64_t n = 0;
    double k = 0;
    int D = 1, Ps = 3, Pa = 5, P = 75;
    double x0[3] = {0, 0, 0}, H1 = 1;
    std::vector<double> pts;   // n x 3
    std::vector<Level> lev;    // index 1..D
    std::vector<double> ts, ta;  // reference nodes for P_s and P_ang
    double last_check = 0.0;
    // Source partition: only the sources in leaves whose Morton
    // key lies in [own_lo, own_hi) contribute; apply() then returns the partial
    // field over all targets (by linearity, the field of the densities zeroed
    // outside those leaves).  Default: everything.
    uint64_t own_lo = 0, own_hi = ~(uint64_t)0;
};

namespace {

int g_threads = 0;  // oracle_set_threads(); 0 = all processors
int nthreads() { return g_threads > 0 ? g_threads : omp_get_num_procs(); }

// ORACLE_VERBOSE=1: wall time of each phase on stderr (diagnostics only).
void phase(const char* what, int d = 0) {
    static const bool on = std::getenv("ORACLE_VERBOSE") && std::getenv("ORACLE_VERBOSE")[0] == '1';
    static double t_last = 0.0;
    if (!on) return;
    double t = omp_get_wtime();
    if (what) std::fprintf(stderr, "[oracle] %-18s d=%-2d %8.3f s\n", what, d, t - t_last);
    t_last = t;
}

double centre(const oracle_plan& p, int d, int64_t k, int axis) {
    // eq. defboxsizesandcenters, 0-based k: x0 + (k + 1/2) H_d
    return p.x0[axis] + ((double)k + 0.5) * p.lev[d].g.H;
}

void box_centre(const oracle_plan& p, int d, const Box& b, double c[3]) {
    c[0] = centre(p, d, b.i, 0);
    c[1] = centre(p, d, b.j, 1);
    c[2] = centre(p, d, b.k, 2);
}

// Separable node tables of a level (eq. interp_pts, eq.
// parametrizationleveldependent P:1290-1292):
//   s_k = (i_s + (1 + t_k)/2) Delta_s,  r = h_d / s_k,
//   theta_i = (i_theta + (1 + t_i)/2) Delta_theta,  phi_j likewise (for n_C even
//   from the first-quadrant sector rotated by quarter turns, reading R18).
void node_tables(const oracle_plan& p, Grid& g) {
    const int Ps = p.Ps, Pa = p.Pa;
    g.nr.assign((size_t)g.ns * Ps, 0.0);
    for (int is = 0; is < g.ns; ++is)
        for (int ks = 0; ks < Ps; ++ks) {
            double s = ((double)is + (1.0 + p.ts[ks]) / 2.0) * g.ds;
            g.nr[is * Ps + ks] = g.h / s;
        }
    g.nst.assign((size_t)g.nC * Pa, 0.0);
    g.nct.assign((size_t)g.nC * Pa, 0.0);
    for (int ith = 0; ith < g.nC; ++ith)
        for (int it = 0; it < Pa; ++it) {
            double th = ((double)ith + (1.0 + p.ta[it]) / 2.0) * g.dth;
            g.nst[ith * Pa + it] = std::sin(th);
            g.nct[ith * Pa + it] = std::cos(th);
        }
    g.ncp.assign((size_t)2 * g.nC * Pa, 0.0);
    g.nsp.assign((size_t)2 * g.nC * Pa, 0.0);
    for (int iph = 0; iph < 2 * g.nC; ++iph)
        for (int jp = 0; jp < Pa; ++jp) {
            double cp, sp;
            if (g.nC % 2 == 0) {  // quarter-turn reduction of the phi sector (reading R18)
                const int hq = g.nC / 2;
                const double ph = ((double)(iph % hq) + (1.0 + p.ta[jp]) / 2.0) * g.dth;
                quarter_turns(std::cos(ph), std::sin(ph), iph / hq, &cp, &sp);
            } else {
                const double ph = ((double)iph + (1.0 + p.ta[jp]) / 2.0) * g.dth;
                sp = std::sin(ph);
                cp = std::cos(ph);
            }
            g.ncp[iph * Pa + jp] = cp;
            g.nsp[iph * Pa + jp] = sp;
        }
}

// Offset from the box centre of node (ks, it, jp) of cell (is, ith, iph):
// x^d(s_k, theta_i, phi_j) = r (sin th cos ph, sin th sin ph, cos th), left to right.
void node_offset(const oracle_plan& p, const Grid& g, int is, int ith, int iph, int ks, int it, int jp,
                 double off[3], double* r_out) {
    const double r = g.nr[is * p.Ps + ks];
    const double st = g.nst[ith * p.Pa + it], ct = g.nct[ith * p.Pa + it];
    const double cp = g.ncp[iph * p.Pa + jp], sp = g.nsp[iph * p.Pa + jp];
    off[0] = r * st * cp;
    off[1] = r * st * sp;
    off[2] = r * ct;
    if (r_out) *r_out = r;
}

void decode_cell(const Grid& g, int64_t lin, int* is, int* it, int* ip) {
    *is = (int)(lin % g.ns);
    *it = (int)((lin / g.ns) % g.nC);
    *ip = (int)(lin / ((int64_t)g.ns * g.nC));
}

// Exact analytic factor F_B at relative position v (eq. I_k).
cplx exact_F(const oracle_plan& p, int d, const Box& b, const double* a2, const double v[3]) {
    double c[3];
    box_centre(p, d, b, c);
    cplx F = 0.0;
    for (int m : b.pts) {
        double w[3] = {p.pts[3 * m] - c[0], p.pts[3 * m + 1] - c[1], p.pts[3 * m + 2] - c[2]};
        F += cplx(a2[2 * m], a2[2 * m + 1]) * analytic_factor_rel(v, w, p.k);
    }
    return F;
}

// Recentering factor G(y, c_B) / G(y, c_Q) (Algorithm 1 line
// P:1858) for y = c_Q + off = c_B + (off + delta):
//   (r_Q / r_B) e^{i kappa (r_B - r_Q)}.
cplx recenter(const double off[3], const double delta[3], double k) {
    double mdelta[3] = {-delta[0], -delta[1], -delta[2]};
    double rB;
    double diff = dist_minus_norm(off, mdelta, &rB);  // |off + delta| - |off|
    double rQ = norm3(off);
    return (rQ / rB) * cplx(std::cos(k * diff), std::sin(k * diff));
}

// Child octant of box b (parity of its multi-index) and delta = c_Q - c_B =
// +-H_d/2 per axis (exact; DESIGN.md contract): + for an even index.
int octant(const Box& b) { return (int)((b.i & 1) | ((b.j & 1) << 1) | ((b.k & 1) << 2)); }
void octant_delta(int o, double H, double delta[3]) {
    for (int a = 0; a < 3; ++a) delta[a] = ((o >> a) & 1) ? -H / 2.0 : H / 2.0;
}

// Sorted, duplicate-free copy of v (the set of its values).
template <class T>
void sort_unique(std::vector<T>& v) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
}

int build_plan(oracle_plan& p, const double* pts, int64_t n, double k, int D, int Ps, int Pa, int leaf_ns,
               int leaf_nc, int has_root, const double* root_c, double root_H, uint64_t own_lo, uint64_t own_hi) {
    if (n < 1 || D < 1 || D > 22 || Ps < 1 || Pa < 1 || Ps > MAXP || Pa > MAXP || !(k >= 0.0) ||
        !std::isfinite(k) || !pts)
        return EINVAL_;
    if (leaf_ns < 1) leaf_ns = 1;
    if (leaf_nc < 1) leaf_nc = 2;
    for (int64_t i = 0; i < 3 * n; ++i)
        if (!std::isfinite(pts[i])) return EINVAL_;
    const int nt = nthreads();
    p.n = n; p.k = k; p.D = D; p.Ps = Ps; p.Pa = Pa; p.P = Ps * Pa * Pa;
    p.own_lo = own_lo; p.own_hi = own_hi;
    p.pts.assign(pts, pts + 3 * n);
    p.ts = cheb_nodes(Ps);
    p.ta = cheb_nodes(Pa);
    phase(nullptr);

    // Pairwise-different points.
    {
        std::vector<std::tuple<double, double, double>> s(n);
        for (int64_t i = 0; i < n; ++i) s[i] = std::make_tuple(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
        __gnu_parallel::sort(s.begin(), s.end());
        for (int64_t i = 1; i < n; ++i)
            if (s[i] == s[i - 1]) return EDOMAIN_;
    }
    // Root box B^1 containing Gamma_N (eq. deffirstbox; reading R9).
    double c1[3], H1;
    if (has_root) {
        if (!root_c || !(root_H > 0.0)) return EINVAL_;
        c1[0] = root_c[0]; c1[1] = root_c[1]; c1[2] = root_c[2];
        H1 = root_H;
    } else {
        double lo[3], hi[3];
        for (int a = 0; a < 3; ++a) { lo[a] = pts[a]; hi[a] = pts[a]; }
        for (int64_t i = 1; i < n; ++i)
            for (int a = 0; a < 3; ++a) {
                lo[a] = std::min(lo[a], pts[3 * i + a]);
                hi[a] = std::max(hi[a], pts[3 * i + a]);
            }
        double ext = 0.0;
        for (int a = 0; a < 3; ++a) {
            c1[a] = (lo[a] + hi[a]) / 2.0;
            ext = std::max(ext, hi[a] - lo[a]);
        }
        if (ext == 0.0) {
            if (n > 1) return EDOMAIN_;
            ext = 1.0;
        }
        H1 = (1.0 + std::ldexp(1.0, -20)) * ext;
    }
    p.H1 = H1;
    for (int a = 0; a < 3; ++a) p.x0[a] = c1[a] - H1 / 2.0;
    if (has_root)  // B^1 must contain Gamma_N (eq. deffirstbox)
        for (int64_t i = 0; i < n; ++i)
            for (int a = 0; a < 3; ++a)
                if (!(pts[3 * i + a] >= p.x0[a] && pts[3 * i + a] <= p.x0[a] + H1)) return EDOMAIN_;

    // Levels and cone grids.  Reading R8: (n_s, n_C)_D = (leaf_ns, leaf_nc);
    // readings R5/R6: counts double from d to d-1 iff kappa H_{d-1} > 1
    // (the "/a_d" of P:1329 contradicts the spans halving).
    p.lev.assign(D + 1, Level());
    for (int d = 1; d <= D; ++d) p.lev[d].g.H = std::ldexp(H1, -(d - 1));  // H_d = H_1 / 2^{d-1}
    p.lev[D].g.ns = leaf_ns;
    p.lev[D].g.nC = leaf_nc;
    for (int d = D; d >= 2; --d) {
        bool refine = k * p.lev[d - 1].g.H > 1.0;
        p.lev[d - 1].g.ns = refine ? 2 * p.lev[d].g.ns : p.lev[d].g.ns;
        p.lev[d - 1].g.nC = refine ? 2 * p.lev[d].g.nC : p.lev[d].g.nC;
    }
    for (int d = 1; d <= D; ++d) {
        grid_tables(p.lev[d].g);
        node_tables(p, p.lev[d].g);
        p.lev[d].side = (int64_t)1 << (d - 1);
    }

    // Relevant boxes via the integer parts of the coordinate
    // quotients: q = floor((x - x0)/H_D), level d: q >> (D - d).
    const int64_t nmax = (int64_t)1 << (D - 1);
    std::vector<int64_t> q(3 * n);
#pragma omp parallel for num_threads(nt) schedule(static)
    for (int64_t m = 0; m < n; ++m)
        for (int a = 0; a < 3; ++a) {
            double t = std::floor((pts[3 * m + a] - p.x0[a]) / p.lev[D].g.H);
            int64_t qi = t < 0.0 ? 0 : (t >= (double)nmax ? nmax - 1 : (int64_t)t);
            q[3 * m + a] = qi;
        }
    {
        std::vector<std::pair<uint64_t, int>> kv(n);
        for (int d = 1; d <= D; ++d) {
            Level& L = p.lev[d];
            const int sh = D - d;
#pragma omp parallel for num_threads(nt) schedule(static)
            for (int64_t m = 0; m < n; ++m)
                kv[m] = {box_key(q[3 * m] >> sh, q[3 * m + 1] >> sh, q[3 * m + 2] >> sh), (int)m};
            // (key, point) pairs are distinct: every correct sort gives the same order,
            // boxes by key and each box's points increasing.
            __gnu_parallel::sort(kv.begin(), kv.end());
            for (int64_t m = 0; m < n;) {
                int64_t e = m;
                while (e < n && kv[e].first == kv[m].first) ++e;
                Box b;
                b.i = (int64_t)(kv[m].first >> 42);
                b.j = (int64_t)((kv[m].first >> 21) & ((1u << 21) - 1));
                b.k = (int64_t)(kv[m].first & ((1u << 21) - 1));
                b.pts.resize(e - m);
                for (int64_t t = m; t < e; ++t) b.pts[t - m] = kv[t].second;
                L.keys.push_back(kv[m].first);
                L.boxes.push_back(std::move(b));
                m = e;
            }
        }
    }
    phase("plan: boxes");
    // Parent / children; children in increasing box order.
    for (int d = 2; d <= D; ++d) {
        Level& L = p.lev[d];
        int bad = 0;
#pragma omp parallel for num_threads(nt) schedule(static) reduction(| : bad)
        for (int64_t bi = 0; bi < (int64_t)L.boxes.size(); ++bi) {
            Box& b = L.boxes[bi];
            b.parent = p.lev[d - 1].find(b.i >> 1, b.j >> 1, b.k >> 1);
            if (b.parent < 0) bad = 1;
        }
        if (bad) return EINTERNAL_;
        for (int bi = 0; bi < (int)L.boxes.size(); ++bi) p.lev[d - 1].boxes[L.boxes[bi].parent].children.push_back(bi);
    }
    // Owned leaves, and the boxes with an owned leaf below them.
    for (Box& b : p.lev[D].boxes) {
        const uint64_t mk = morton_key(b.i, b.j, b.k);
        b.active = mk >= own_lo && mk < own_hi;
    }
    for (int d = D - 1; d >= 1; --d)
        for (Box& b : p.lev[d].boxes) {
            b.active = false;
            for (int ch : b.children) b.active = b.active || p.lev[d + 1].boxes[ch].active;
        }
    // Neighbours N B: relevant, ||a - k||_inf <= 1, B included;
    // increasing box order.
    for (int d = 1; d <= D; ++d) {
        Level& L = p.lev[d];
#pragma omp parallel for num_threads(nt) schedule(dynamic, 256)
        for (int64_t bi = 0; bi < (int64_t)L.boxes.size(); ++bi) {
            Box& b = L.boxes[bi];
            for (int64_t di = -1; di <= 1; ++di)
                for (int64_t dj = -1; dj <= 1; ++dj)
                    for (int64_t dk = -1; dk <= 1; ++dk) {
                        int a = L.find(b.i + di, b.j + dj, b.k + dk);
                        if (a >= 0) b.nbrs.push_back(a);
                    }
        }
    }
    // Cousins M B = (R_B^d \ N B) cap Q N P B (eq. defcousinboxes),
    // increasing box order.
    for (int d = 2; d <= D; ++d) {
        Level& L = p.lev[d];
        Level& LP = p.lev[d - 1];
#pragma omp parallel for num_threads(nt) schedule(dynamic, 256)
        for (int64_t bi = 0; bi < (int64_t)L.boxes.size(); ++bi) {
            Box& b = L.boxes[bi];
            std::vector<int> c;
            for (int pn : LP.boxes[b.parent].nbrs)
                for (int ch : LP.boxes[pn].children) {
                    const Box& a = L.boxes[ch];
                    int64_t dist = std::max({std::llabs(a.i - b.i), std::llabs(a.j - b.j), std::llabs(a.k - b.k)});
                    if (dist > 1) c.push_back(ch);
                }
            sort_unique(c);
            b.cousins = std::move(c);
        }
    }
    phase("plan: lists");
    // Relevant cone segments, single sweep d = 3..D (eq. defallrelevantconesegments
    // P:1509-1522): (i) segments containing a cousin point; (ii) for
    // d >= 4, segments containing a node of a relevant parent segment.
    for (int d = 3; d <= D; ++d) {
        Level& L = p.lev[d];
        const int64_t ncell = (int64_t)2 * L.g.ns * L.g.nC * L.g.nC;
        // (ii) is box-independent given (parent cell, child octant): the set
        // S(gamma', o) of child cells hit by the nodes of gamma' (SURVEY.md §8(c)
        // "child-code set").  Computed once for every pair that occurs.
        std::vector<uint64_t> pairs;  // parent cell * 8 + octant, sorted
        std::vector<int64_t> s_off;   // CSR over pairs
        std::vector<int64_t> s_cells;
        if (d >= 4) {
            const Level& LP = p.lev[d - 1];
            for (const Box& b : L.boxes)
                if (b.active)
                    for (int64_t gq : LP.boxes[b.parent].segs) pairs.push_back((uint64_t)gq * 8 + octant(b));
            __gnu_parallel::sort(pairs.begin(), pairs.end());
            pairs.erase(std::unique(pairs.begin(), pairs.end()), pairs.end());
            std::vector<std::vector<int64_t>> S(pairs.size());
#pragma omp parallel for num_threads(nt) schedule(dynamic, 64)
            for (int64_t pi = 0; pi < (int64_t)pairs.size(); ++pi) {
                int is, ith, iph;
                decode_cell(LP.g, (int64_t)(pairs[pi] / 8), &is, &ith, &iph);
                double delta[3];
                octant_delta((int)(pairs[pi] % 8), L.g.H, delta);
                std::vector<int64_t>& out = S[pi];
                for (int jp = 0; jp < p.Pa; ++jp)
                    for (int it = 0; it < p.Pa; ++it)
                        for (int ks = 0; ks < p.Ps; ++ks) {
                            double off[3];
                            node_offset(p, LP.g, is, ith, iph, ks, it, jp, off, nullptr);
                            double v[3] = {off[0] + delta[0], off[1] + delta[1], off[2] + delta[2]};
                            Cls cl = classify(L.g, v);
                            out.push_back(cell_lin(L.g, cl.is, cl.it, cl.ip));
                        }
                sort_unique(out);
            }
            s_off.assign(pairs.size() + 1, 0);
            for (size_t pi = 0; pi < pairs.size(); ++pi) s_off[pi + 1] = s_off[pi] + (int64_t)S[pi].size();
            s_cells.resize(s_off.back());
            for (size_t pi = 0; pi < pairs.size(); ++pi) std::copy(S[pi].begin(), S[pi].end(), s_cells.begin() + s_off[pi]);
        }
#pragma omp parallel num_threads(nt)
        {
            std::vector<uint8_t> flag(ncell, 0);
            std::vector<int64_t> touched;
#pragma omp for schedule(dynamic, 16)
            for (int64_t bi = 0; bi < (int64_t)L.boxes.size(); ++bi) {
                Box& b = L.boxes[bi];
                if (!b.active) continue;  // its cone data is never formed on this partition
                touched.clear();
                auto mark = [&](int64_t cell) {
                    if (!flag[cell]) { flag[cell] = 1; touched.push_back(cell); }
                };
                double c[3];
                box_centre(p, d, b, c);
                for (int ci : b.cousins)
                    for (int m : L.boxes[ci].pts) {
                        double v[3] = {p.pts[3 * m] - c[0], p.pts[3 * m + 1] - c[1], p.pts[3 * m + 2] - c[2]};
                        Cls cl = classify(L.g, v);
                        mark(cell_lin(L.g, cl.is, cl.it, cl.ip));
                    }
                if (d >= 4) {
                    const int o = octant(b);
                    for (int64_t gq : p.lev[d - 1].boxes[b.parent].segs) {
                        uint64_t key = (uint64_t)gq * 8 + o;
                        int64_t pi = std::lower_bound(pairs.begin(), pairs.end(), key) - pairs.begin();
                        for (int64_t t = s_off[pi]; t < s_off[pi + 1]; ++t) mark(s_cells[t]);
                    }
                }
                std::sort(touched.begin(), touched.end());
                for (int64_t cell : touched) flag[cell] = 0;
                b.segs = touched;
            }
        }
        phase("plan: relevance", d);
    }
    return OK;
}

int seg_slot(const Box& b, int64_t lin) {
    auto it = std::lower_bound(b.segs.begin(), b.segs.end(), lin);
    if (it == b.segs.end() || *it != lin) return -1;
    return (int)(it - b.segs.begin());
}

enum { ST_NEAR = 1, ST_COUSIN = 2, ST_UPWARD = 4 };
enum { MODE_NORMAL = 0, MODE_BYPASS = 1 };

// Operator application, Algorithm 1.  Loop order: see the file
// header (target-major near / cousin loops, parent-segment-major upward loop;
// every output has one owner and receives its terms in increasing source-box
// order, exactly as in the source-major loop nest of Algorithm 1).
int apply(oracle_plan& p, const double* a2, double* out2, unsigned stage_mask, int mode) {
    const int D = p.D, P = p.P, Ps = p.Ps, Pa = p.Pa;
    const int nt = nthreads();
    if (mode == MODE_BYPASS && (p.own_lo != 0 || p.own_hi != ~(uint64_t)0))
        return EINVAL_;  // the bypass check is defined on the full source set only
    std::vector<cplx> I(p.n, 0.0);
    const double* X = p.pts.data();
    int bad = 0;
    phase(nullptr);

    // Direct evaluations on level D, neighbouring surface points:
    // I(x_l) += sum_{m in B, m != l} a_m G(x_l, x_m) over the neighbours B of
    // x_l's leaf (raw kernel, reading R11).
    if (stage_mask & ST_NEAR) {
        const Level& L = p.lev[D];
#pragma omp parallel for num_threads(nt) schedule(dynamic, 16)
        for (int64_t ti = 0; ti < (int64_t)L.boxes.size(); ++ti) {
            const Box& t = L.boxes[ti];
            for (int l : t.pts) {
                cplx acc = I[l];
                for (int nb : t.nbrs) {
                    if (!L.boxes[nb].active) continue;  // sources outside the partition
                    for (int m : L.boxes[nb].pts) {
                        if (m == l) continue;
                        double d3[3] = {X[3 * l] - X[3 * m], X[3 * l + 1] - X[3 * m + 1], X[3 * l + 2] - X[3 * m + 2]};
                        acc += cplx(a2[2 * m], a2[2 * m + 1]) * green_r(norm3(d3), p.k);
                    }
                }
                I[l] = acc;
            }
        }
    }

    phase("apply: near");
    // Node values V (per level, per box, per relevant segment, P values); after
    // the fit of level d they hold that level's Chebyshev coefficients.
    std::vector<std::vector<std::vector<cplx>>> V(D + 1);
    // Level D: F_B at all interpolation points of relevant leaf segments.
    if (D >= 3 && mode == MODE_NORMAL && (stage_mask & (ST_COUSIN | ST_UPWARD))) {
        const Level& L = p.lev[D];
        V[D].resize(L.boxes.size());
#pragma omp parallel for num_threads(nt) schedule(dynamic, 16)
        for (int64_t bi = 0; bi < (int64_t)L.boxes.size(); ++bi) {
            const Box& b = L.boxes[bi];
            if (!b.active) continue;
            V[D][bi].assign(b.segs.size() * P, 0.0);
            for (size_t si = 0; si < b.segs.size(); ++si) {
                int is, ith, iph;
                decode_cell(L.g, b.segs[si], &is, &ith, &iph);
                for (int jp = 0; jp < Pa; ++jp)
                    for (int it = 0; it < Pa; ++it)
                        for (int ks = 0; ks < Ps; ++ks) {
                            double off[3];
                            node_offset(p, L.g, is, ith, iph, ks, it, jp, off, nullptr);
                            V[D][bi][si * P + (jp * Pa + it) * Ps + ks] = exact_F(p, D, b, a2, off);
                        }
            }
        }
    }

    phase("apply: s2c");
    // Interpolation onto surface points and parent interpolation points,
    // d = D, ..., 3.
    for (int d = D; d >= 3; --d) {
        const Level& L = p.lev[d];
        // Chebyshev coefficients of every relevant segment, in place.
        std::vector<std::vector<cplx>>& C = V[d];
        const bool have = mode == MODE_NORMAL && !C.empty();
        if (have) {
#pragma omp parallel for num_threads(nt) schedule(dynamic, 16)
            for (int64_t bi = 0; bi < (int64_t)L.boxes.size(); ++bi)
                for (size_t si = 0; si < L.boxes[bi].segs.size(); ++si)
                    tensor_fit(Ps, Pa, &C[bi][si * P], &C[bi][si * P]);
        }
        phase("apply: fit", d);
        // Cousin surface points: I(x) += G(x, x_k^d) Interp F_k^d(x),
        // for each target x_l, over the cousins x_k^d of its level-d box.
        if ((stage_mask & ST_COUSIN) && (have || mode == MODE_BYPASS)) {
            // work items: (target box, up to 64 of its points); each point has one owner
            std::vector<std::pair<int, int>> items;
            for (int ti = 0; ti < (int)L.boxes.size(); ++ti)
                for (int s = 0; s < (int)L.boxes[ti].pts.size(); s += 64) items.emplace_back(ti, s);
#pragma omp parallel for num_threads(nt) schedule(dynamic, 8) reduction(| : bad)
            for (int64_t wi = 0; wi < (int64_t)items.size(); ++wi) {
                const Box& t = L.boxes[items[wi].first];
                const int s0 = items[wi].second, s1 = std::min(s0 + 64, (int)t.pts.size());
                for (int sp = s0; sp < s1; ++sp) {
                    const int l = t.pts[sp];
                    cplx acc = I[l];
                    for (int bi : t.cousins) {
                        const Box& b = L.boxes[bi];
                        if (!b.active) continue;  // sources outside the partition
                        double c[3];
                        box_centre(p, d, b, c);
                        double v[3] = {X[3 * l] - c[0], X[3 * l + 1] - c[1], X[3 * l + 2] - c[2]};
                        cplx F;
                        if (mode == MODE_BYPASS) {
                            F = exact_F(p, d, b, a2, v);
                        } else {
                            Cls cl = classify(L.g, v);
                            int sl = seg_slot(b, cell_lin(L.g, cl.is, cl.it, cl.ip));
                            if (sl < 0) { bad = 1; continue; }  // cousin point outside R_C B (impossible)
                            F = tensor_eval(Ps, Pa, &C[bi][sl * P], cl.us, cl.ut, cl.up);
                        }
                        acc += green_r(norm3(v), p.k) * F;
                    }
                    I[l] = acc;
                }
            }
            if (bad) return EINTERNAL_;
        }
        phase("apply: cousin", d);
        // Parent interpolation points with re-centering:
        //   V_Q[gamma', y] = sum over children B of Q (increasing box order) of
        //   Interp_{B, gamma(y - c_B)}(y) G(y, c_B) / G(y, c_Q).
        // The child cell, local coordinates and recentering factor of node y
        // depend only on (gamma', octant of B): computed once per occurring pair.
        if (d > 3 && (stage_mask & ST_UPWARD) && have) {
            const Level& LP = p.lev[d - 1];
            V[d - 1].resize(LP.boxes.size());
            std::vector<std::tuple<int64_t, int, int>> segs;  // (cell, Q, slot): parent segments by cell
            for (size_t qi = 0; qi < LP.boxes.size(); ++qi) {
                if (!LP.boxes[qi].active) continue;
                V[d - 1][qi].assign(LP.boxes[qi].segs.size() * P, 0.0);
                for (size_t sq = 0; sq < LP.boxes[qi].segs.size(); ++sq)
                    segs.emplace_back(LP.boxes[qi].segs[sq], (int)qi, (int)sq);
            }
            __gnu_parallel::sort(segs.begin(), segs.end());
            std::vector<int64_t> gstart;  // runs of equal cell
            for (size_t e = 0; e < segs.size(); ++e)
                if (e == 0 || std::get<0>(segs[e]) != std::get<0>(segs[e - 1])) gstart.push_back((int64_t)e);
            gstart.push_back((int64_t)segs.size());
            struct NodeGeo {
                int64_t cell;
                double Ts[MAXP], Tt[MAXP], Tp[MAXP];
                cplx rec;
            };
            const int64_t ngroups = (int64_t)gstart.size() - 1;
#pragma omp parallel num_threads(nt)
            {
                std::vector<NodeGeo> geo(8 * (size_t)P);
#pragma omp for schedule(dynamic, 4) reduction(| : bad)
                for (int64_t gi = 0; gi < ngroups; ++gi) {
                    const int64_t cellq = std::get<0>(segs[gstart[gi]]);
                    int is, ith, iph;
                    decode_cell(LP.g, cellq, &is, &ith, &iph);
                    unsigned need = 0;
                    for (int64_t e = gstart[gi]; e < gstart[gi + 1]; ++e)
                        for (int ch : LP.boxes[std::get<1>(segs[e])].children)
                            if (L.boxes[ch].active) need |= 1u << octant(L.boxes[ch]);
                    for (int o = 0; o < 8; ++o) {
                        if (!(need & (1u << o))) continue;
                        double delta[3];
                        octant_delta(o, L.g.H, delta);
                        for (int jp = 0; jp < Pa; ++jp)
                            for (int it = 0; it < Pa; ++it)
                                for (int ks = 0; ks < Ps; ++ks) {
                                    const int y = (jp * Pa + it) * Ps + ks;
                                    double off[3];
                                    node_offset(p, LP.g, is, ith, iph, ks, it, jp, off, nullptr);
                                    double v[3] = {off[0] + delta[0], off[1] + delta[1], off[2] + delta[2]};
                                    Cls cl = classify(L.g, v);
                                    NodeGeo& G = geo[o * P + y];
                                    G.cell = cell_lin(L.g, cl.is, cl.it, cl.ip);
                                    cheb_T(Ps, cl.us, G.Ts);
                                    cheb_T(Pa, cl.ut, G.Tt);
                                    cheb_T(Pa, cl.up, G.Tp);
                                    G.rec = recenter(off, delta, p.k);
                                }
                    }
                    for (int64_t e = gstart[gi]; e < gstart[gi + 1]; ++e) {
                        const int qi = std::get<1>(segs[e]), sq = std::get<2>(segs[e]);
                        const Box& Q = LP.boxes[qi];
                        cplx* out = &V[d - 1][qi][(size_t)sq * P];
                        int64_t last_cell[8];
                        int last_slot[8];
                        for (int c = 0; c < 8; ++c) last_cell[c] = -1;
                        for (int y = 0; y < P; ++y)
                            for (size_t c = 0; c < Q.children.size(); ++c) {
                                const int ch = Q.children[c];
                                const Box& b = L.boxes[ch];
                                if (!b.active) continue;
                                const NodeGeo& G = geo[octant(b) * P + y];
                                if (G.cell != last_cell[c]) {  // same cell as the previous node: same slot
                                    last_cell[c] = G.cell;
                                    last_slot[c] = seg_slot(b, G.cell);
                                }
                                const int sl = last_slot[c];
                                if (sl < 0) { bad = 1; continue; }  // parent node outside R_C B (impossible)
                                cplx F = tensor_eval_T(Ps, Pa, &C[ch][(size_t)sl * P], G.Ts, G.Tt, G.Tp);
                                out[y] += F * G.rec;
                            }
                    }
                }
            }
            if (bad) return EINTERNAL_;
        }
        phase("apply: upward", d);
        V[d].clear();  // level d values freed once level d-1 is filled
        V[d].shrink_to_fit();
    }
    for (int64_t l = 0; l < p.n; ++l) {
        out2[2 * l] = I[l].real();
        out2[2 * l + 1] = I[l].imag();
    }
    return OK;
}

// Exact-recentering check (pins P:1754-1757 / P:1858 algebra): for every level
// d = D..4, parent Q, relevant (Q, gamma'), node y:
//   | sum_{B in Q Q} F_B(y) G(y,c_B)/G(y,c_Q) - F_Q(y) | / |F_Q(y)|,
// with F exact (eq. I_k).  Returns the maximum.
double recentering_check(const oracle_plan& p, const double* a2) {
    double worst = 0.0;
    for (int d = p.D; d >= 4; --d) {
        const Level& L = p.lev[d];
        const Level& LP = p.lev[d - 1];
        for (const Box& Q : LP.boxes)
            for (int64_t gq : Q.segs) {
                int is, ith, iph;
                decode_cell(LP.g, gq, &is, &ith, &iph);
                for (int jp = 0; jp < p.Pa; ++jp)
                    for (int it = 0; it < p.Pa; ++it)
                        for (int ks = 0; ks < p.Ps; ++ks) {
                            double off[3];
                            node_offset(p, LP.g, is, ith, iph, ks, it, jp, off, nullptr);
                            cplx acc = 0.0;
                            for (int ch : Q.children) {
                                const Box& b = L.boxes[ch];
                                double delta[3] = {(b.i & 1) ? -L.g.H / 2.0 : L.g.H / 2.0,
                                                   (b.j & 1) ? -L.g.H / 2.0 : L.g.H / 2.0,
                                                   (b.k & 1) ? -L.g.H / 2.0 : L.g.H / 2.0};
                                double v[3] = {off[0] + delta[0], off[1] + delta[1], off[2] + delta[2]};
                                acc += exact_F(p, d, b, a2, v) * recenter(off, delta, p.k);
                            }
                            cplx direct = exact_F(p, d - 1, Q, a2, off);
                            double e = std::abs(acc - direct) / std::abs(direct);
                            worst = std::max(worst, e);
                        }
            }
    }
    return worst;
}

}  // namespace

// =============================================================================
// C ABI (ctypes).  Status codes follow include/ifgf.h numbering by value only.
// =============================================================================
extern "C" {

// Threads of the parallel loops (0 = all processors, 1 = serial).  Results do
// not depend on it (see the file header).
void oracle_set_threads(int n) { g_threads = n < 0 ? 0 : n; }
int oracle_get_threads(void) { return nthreads(); }

// own_lo / own_hi: half-open Morton-key range of the owned leaves (source
// partition); 0 / ~0 = all sources.
int oracle_plan_create_part(const double* pts, int64_t n, double k, int D, int Ps, int Pa, int leaf_ns, int leaf_nc,
                            int has_root, const double* root_c, double root_H, uint64_t own_lo, uint64_t own_hi,
                            oracle_plan** out) {
    if (!out) return EINVAL_;
    *out = nullptr;
    oracle_plan* p = new (std::nothrow) oracle_plan();
    if (!p) return ENOMEM_;
    int st;
    try {
        st = build_plan(*p, pts, n, k, D, Ps, Pa, leaf_ns, leaf_nc, has_root, root_c, root_H, own_lo, own_hi);
    } catch (const std::bad_alloc&) {
        st = ENOMEM_;
    }
    if (st != OK) {
        delete p;
        return st;
    }
    *out = p;
    return OK;
}

int oracle_plan_create(const double* pts, int64_t n, double k, int D, int Ps, int Pa, int leaf_ns, int leaf_nc,
                       int has_root, const double* root_c, double root_H, oracle_plan** out) {
    return oracle_plan_create_part(pts, n, k, D, Ps, Pa, leaf_ns, leaf_nc, has_root, root_c, root_H, 0,
                                   ~(uint64_t)0, out);
}

void oracle_plan_destroy(oracle_plan* p) { delete p; }

int oracle_apply(oracle_plan* p, const double* dens, double* out, unsigned stage_mask, int mode) {
    if (!p || !dens || !out) return EINVAL_;
    try {
        return apply(*p, dens, out, stage_mask, mode);
    } catch (const std::bad_alloc&) {
        return ENOMEM_;
    }
}

double oracle_recentering_check(oracle_plan* p, const double* dens) { return recentering_check(*p, dens); }

// info[0..9]: nbox, nseg, ns, nC, H, h, x0[3] (levels d < 1 or > D: error)
int oracle_level_info(const oracle_plan* p, int d, double* info) {
    if (!p || d < 1 || d > p->D) return EINVAL_;
    const Level& L = p->lev[d];
    int64_t nseg = 0;
    for (const Box& b : L.boxes) nseg += (int64_t)b.segs.size();
    info[0] = (double)L.boxes.size();
    info[1] = (double)nseg;
    info[2] = L.g.ns;
    info[3] = L.g.nC;
    info[4] = L.g.H;
    info[5] = L.g.h;
    info[6] = p->x0[0];
    info[7] = p->x0[1];
    info[8] = p->x0[2];
    return OK;
}

// Boxes of level d in the oracle's (lexicographic) order: out[5*b..] = i, j, k, npts, ncousins.
int64_t oracle_level_boxes(const oracle_plan* p, int d, int64_t* out, int64_t cap) {
    if (!p || d < 1 || d > p->D) return -1;
    const Level& L = p->lev[d];
    int64_t nb = (int64_t)L.boxes.size();
    if (out && cap >= nb)
        for (int64_t b = 0; b < nb; ++b) {
            const Box& x = L.boxes[b];
            out[5 * b] = x.i; out[5 * b + 1] = x.j; out[5 * b + 2] = x.k;
            out[5 * b + 3] = (int64_t)x.pts.size();
            out[5 * b + 4] = (int64_t)x.cousins.size();
        }
    return nb;
}

// Relevant segments of level d: out[4*s..] = i, j, k, cell_lin (cell_lin = (ip*nC + it)*ns + is).
int64_t oracle_level_segments(const oracle_plan* p, int d, int64_t* out, int64_t cap) {
    if (!p || d < 1 || d > p->D) return -1;
    const Level& L = p->lev[d];
    int64_t ns = 0;
    for (const Box& b : L.boxes) ns += (int64_t)b.segs.size();
    if (out && cap >= ns) {
        int64_t s = 0;
        for (const Box& b : L.boxes)
            for (int64_t g : b.segs) {
                out[4 * s] = b.i; out[4 * s + 1] = b.j; out[4 * s + 2] = b.k; out[4 * s + 3] = g;
                ++s;
            }
    }
    return ns;
}

// Neighbour / cousin lists of box index b at level d (indices into oracle_level_boxes order).
int64_t oracle_box_list(const oracle_plan* p, int d, int64_t b, int which, int64_t* out, int64_t cap) {
    if (!p || d < 1 || d > p->D || b < 0 || b >= (int64_t)p->lev[d].boxes.size()) return -1;
    const Box& x = p->lev[d].boxes[b];
    const std::vector<int>& v = which == 0 ? x.nbrs : (which == 1 ? x.cousins : x.children);
    if (out && cap >= (int64_t)v.size())
        for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
    return (int64_t)v.size();
}

// Direct sum I(x_l) = sum_{m != l} a_m G(x_l, x_m) (eq. field1) at
// targets[0..M), with Kahan-compensated accumulation of re and im.
int oracle_direct(const double* pts, int64_t n, double k, const double* dens, const int64_t* targets, int64_t M,
                  double* out) {
    for (int64_t t = 0; t < M; ++t)
        if (targets[t] < 0 || targets[t] >= n) return EINVAL_;
#pragma omp parallel for num_threads(nthreads()) schedule(dynamic, 1)
    for (int64_t t = 0; t < M; ++t) {
        int64_t l = targets[t];
        double sr = 0, cr = 0, si = 0, ci = 0;
        for (int64_t m = 0; m < n; ++m) {
            if (m == l) continue;
            double d3[3] = {pts[3 * l] - pts[3 * m], pts[3 * l + 1] - pts[3 * m + 1], pts[3 * l + 2] - pts[3 * m + 2]};
            cplx v = cplx(dens[2 * m], dens[2 * m + 1]) * green_r(norm3(d3), k);
            double y = v.real() - cr, tt = sr + y;
            cr = (tt - sr) - y; sr = tt;
            y = v.imag() - ci; tt = si + y;
            ci = (tt - si) - y; si = tt;
        }
        out[2 * t] = sr;
        out[2 * t + 1] = si;
    }
    return OK;
}

// ---- unit entry points for the pins ---------------------------------------
void oracle_green(const double* x, const double* y, double k, double* out2) {
    double d3[3] = {x[0] - y[0], x[1] - y[1], x[2] - y[2]};
    cplx g = green_r(norm3(d3), k);
    out2[0] = g.real(); out2[1] = g.imag();
}

void oracle_analytic_factor(const double* x, const double* xp, const double* c, double k, double* out2) {
    double v[3] = {x[0] - c[0], x[1] - c[1], x[2] - c[2]};
    double w[3] = {xp[0] - c[0], xp[1] - c[1], xp[2] - c[2]};
    cplx g = analytic_factor_rel(v, w, k);
    out2[0] = g.real(); out2[1] = g.imag();
}

void oracle_recenter(const double* off, const double* delta, double k, double* out2) {
    cplx g = recenter(off, delta, k);
    out2[0] = g.real(); out2[1] = g.imag();
}

void oracle_cheb_nodes(int n, double* t) {
    std::vector<double> v = cheb_nodes(n);
    std::copy(v.begin(), v.end(), t);
}

void oracle_cheb_fit1d(int n, const double* u2, double* a2) {
    std::vector<cplx> u(n), a(n);
    for (int i = 0; i < n; ++i) u[i] = cplx(u2[2 * i], u2[2 * i + 1]);
    cheb_fit1d(n, u.data(), a.data());
    for (int i = 0; i < n; ++i) { a2[2 * i] = a[i].real(); a2[2 * i + 1] = a[i].imag(); }
}

void oracle_cheb_eval1d(int n, const double* a2, double x, double* out2) {
    std::vector<cplx> a(n);
    for (int i = 0; i < n; ++i) a[i] = cplx(a2[2 * i], a2[2 * i + 1]);
    cplx v = cheb_eval1d(n, a.data(), x);
    out2[0] = v.real(); out2[1] = v.imag();
}

void oracle_tensor_fit(int Ps, int Pa, const double* V2, double* C2) {
    int P = Ps * Pa * Pa;
    std::vector<cplx> V(P), C(P);
    for (int i = 0; i < P; ++i) V[i] = cplx(V2[2 * i], V2[2 * i + 1]);
    tensor_fit(Ps, Pa, V.data(), C.data());
    for (int i = 0; i < P; ++i) { C2[2 * i] = C[i].real(); C2[2 * i + 1] = C[i].imag(); }
}

void oracle_tensor_eval(int Ps, int Pa, const double* C2, double us, double ut, double up, double* out2) {
    int P = Ps * Pa * Pa;
    std::vector<cplx> C(P);
    for (int i = 0; i < P; ++i) C[i] = cplx(C2[2 * i], C2[2 * i + 1]);
    cplx v = tensor_eval(Ps, Pa, C.data(), us, ut, up);
    out2[0] = v.real(); out2[1] = v.imag();
}

// Classification of relative vector v for a grid (H, ns, nC):
// cell[0..2] = is, it, ip; loc[0..5] = us, ut, up, r, s, unused.
void oracle_classify(double H, int ns, int nC, const double* v, int* cell, double* loc) {
    Grid g;
    g.H = H; g.ns = ns; g.nC = nC;
    grid_tables(g);
    Cls c = classify(g, v);
    Cls s = classify_scan(g, v);  // the literal interval scans must agree
    if (s.is != c.is || s.it != c.it || s.ip != c.ip) { cell[0] = cell[1] = cell[2] = -1; return; }
    cell[0] = c.is; cell[1] = c.it; cell[2] = c.ip;
    loc[0] = c.us; loc[1] = c.ut; loc[2] = c.up; loc[3] = c.r; loc[4] = c.s;
}

// Node offset from the box centre for level grid (H, ns, nC), cell (is,it,ip), node (ks,kt,kp).
void oracle_node_offset(double H, int ns, int nC, int Ps, int Pa, const int* cell, const int* node, double* off) {
    oracle_plan p;
    p.Ps = Ps; p.Pa = Pa;
    p.ts = cheb_nodes(Ps);
    p.ta = cheb_nodes(Pa);
    Grid g;
    g.H = H; g.ns = ns; g.nC = nC;
    grid_tables(g);
    node_tables(p, g);
    node_offset(p, g, cell[0], cell[1], cell[2], node[0], node[1], node[2], off, nullptr);
}

}  // extern "C"
