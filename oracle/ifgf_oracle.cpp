// =============================================================================
// ifgf_oracle.cpp -- plain, serial, fp64 CPU oracle of the IFGF operator
// evaluation (Bauinger & Bruno, arXiv 2010.02857).
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
// Build: g++ -O2 -std=c++17 -ffp-contract=off -fno-fast-math -shared -fPIC
// (FMA contraction off so that every discrete decision is the IEEE result of
// the written formula).
//
// Parity pins (tests/test_oracle_*.py): closed forms of G and g_S, the
// factorisation identity, Chebyshev node reproduction / polynomial exactness /
// eq. 19 bound, brute-force tree relations, bypass mode == direct sum,
// exact-recentering check, centred-source exact case, convergence in (P_s,P_ang),
// metamorphic rotation symmetry.  Every function below is pinned by at least
// one of those; none is "parity unpinned".
// =============================================================================
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <map>
#include <new>
#include <set>
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
void cheb_fit1d(int n, const cplx* u, cplx* a) {
    std::vector<double> t = cheb_nodes(n), T(n);
    for (int i = 0; i < n; ++i) a[i] = 0.0;
    for (int k = 0; k < n; ++k) {
        cheb_T(n, t[k], T.data());
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
    std::vector<cplx> A(V, V + Ps * Pa * Pa), in(std::max(Ps, Pa)), out(std::max(Ps, Pa));
    for (int jp = 0; jp < Pa; ++jp)  // along s
        for (int it = 0; it < Pa; ++it) {
            for (int ks = 0; ks < Ps; ++ks) in[ks] = A[(jp * Pa + it) * Ps + ks];
            cheb_fit1d(Ps, in.data(), out.data());
            for (int ks = 0; ks < Ps; ++ks) A[(jp * Pa + it) * Ps + ks] = out[ks];
        }
    for (int jp = 0; jp < Pa; ++jp)  // along theta
        for (int ks = 0; ks < Ps; ++ks) {
            for (int it = 0; it < Pa; ++it) in[it] = A[(jp * Pa + it) * Ps + ks];
            cheb_fit1d(Pa, in.data(), out.data());
            for (int it = 0; it < Pa; ++it) A[(jp * Pa + it) * Ps + ks] = out[it];
        }
    for (int it = 0; it < Pa; ++it)  // along phi
        for (int ks = 0; ks < Ps; ++ks) {
            for (int jp = 0; jp < Pa; ++jp) in[jp] = A[(jp * Pa + it) * Ps + ks];
            cheb_fit1d(Pa, in.data(), out.data());
            for (int jp = 0; jp < Pa; ++jp) A[(jp * Pa + it) * Ps + ks] = out[jp];
        }
    std::copy(A.begin(), A.end(), C);
}

// Plain triple sum ("simple evaluations of triple sums").
cplx tensor_eval(int Ps, int Pa, const cplx* C, double us, double ut, double up) {
    std::vector<double> Ts(Ps), Tt(Pa), Tp(Pa);
    cheb_T(Ps, us, Ts.data());
    cheb_T(Pa, ut, Tt.data());
    cheb_T(Pa, up, Tp.data());
    cplx s = 0.0;
    for (int jp = 0; jp < Pa; ++jp)
        for (int it = 0; it < Pa; ++it)
            for (int ks = 0; ks < Ps; ++ks) s += C[(jp * Pa + it) * Ps + ks] * (Ts[ks] * Tt[it] * Tp[jp]);
    return s;
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

// Cone segment containing the point with relative vector v = x - x_k^d
// ("simple arithmetic operations in spherical coordinates").
// Intervals are half-open lower-closed (eq. defconedomain, reading R7).
Cls classify(const Grid& g, const double v[3]) {
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
    // phi interval: the unique j with cross_j >= 0 > cross_{j+1}, where
    // cross_j = v_y cos(j dphi) - v_x sin(j dphi); poles (no such j) -> j = 0.
    c.ip = 0;
    for (int j = 0; j < 2 * g.nC; ++j) {
        double cj = v[1] * g.cos_pb[j] - v[0] * g.sin_pb[j];
        double cj1 = v[1] * g.cos_pb[j + 1] - v[0] * g.sin_pb[j + 1];
        if (cj >= 0.0 && cj1 < 0.0) { c.ip = j; break; }
    }
    // Local coordinates (reading R13: theta = atan2(rho, z), phi = atan2(y, x) in [0, 2 pi)).
    double rho = std::sqrt(v[0] * v[0] + v[1] * v[1]);
    double th = std::atan2(rho, v[2]);
    double ph = std::atan2(v[1], v[0]);
    if (ph < 0.0) ph += 2.0 * PI;
    if (v[0] == 0.0 && v[1] == 0.0) ph = 0.0;  // poles: phi := 0 (reading R7)
    c.us = 2.0 * (c.s - c.is * g.ds) / g.ds - 1.0;
    c.ut = 2.0 * (th - c.it * g.dth) / g.dth - 1.0;
    c.up = 2.0 * (ph - c.ip * g.dth) / g.dth - 1.0;
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
};

struct Level {
    std::vector<Box> boxes;
    std::map<std::tuple<int64_t, int64_t, int64_t>, int> index;
    Grid g;
    int find(int64_t i, int64_t j, int64_t k) const {
        auto it = index.find(std::make_tuple(i, j, k));
        return it == index.end() ? -1 : it->second;
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
};

namespace {

double centre(const oracle_plan& p, int d, int64_t k, int axis) {
    // eq. defboxsizesandcenters, 0-based k: x0 + (k + 1/2) H_d
    return p.x0[axis] + ((double)k + 0.5) * p.lev[d].g.H;
}

void box_centre(const oracle_plan& p, int d, const Box& b, double c[3]) {
    c[0] = centre(p, d, b.i, 0);
    c[1] = centre(p, d, b.j, 1);
    c[2] = centre(p, d, b.k, 2);
}

// Offset from the box centre of node (ks, it, jp) of cell (is, ith, iph):
// x^d(s_k, theta_i, phi_j) (eq. interp_pts, eq.
// parametrizationleveldependent P:1290-1292): r = h_d / s_k.
void node_offset(const oracle_plan& p, const Grid& g, int is, int ith, int iph, int ks, int it, int jp,
                 double off[3], double* r_out) {
    double s = ((double)is + (1.0 + p.ts[ks]) / 2.0) * g.ds;
    double th = ((double)ith + (1.0 + p.ta[it]) / 2.0) * g.dth;
    double r = g.h / s;
    double st = std::sin(th), ct = std::cos(th), sp, cp;
    if (g.nC % 2 == 0) {  // quarter-turn reduction of the phi sector (reading R18)
        const int hq = g.nC / 2;
        const double ph = ((double)(iph % hq) + (1.0 + p.ta[jp]) / 2.0) * g.dth;
        quarter_turns(std::cos(ph), std::sin(ph), iph / hq, &cp, &sp);
    } else {
        const double ph = ((double)iph + (1.0 + p.ta[jp]) / 2.0) * g.dth;
        sp = std::sin(ph);
        cp = std::cos(ph);
    }
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

int build_plan(oracle_plan& p, const double* pts, int64_t n, double k, int D, int Ps, int Pa, int leaf_ns,
               int leaf_nc, int has_root, const double* root_c, double root_H) {
    if (n < 1 || D < 1 || D > 22 || Ps < 1 || Pa < 1 || !(k >= 0.0) || !std::isfinite(k) || !pts)
        return EINVAL_;
    if (leaf_ns < 1) leaf_ns = 1;
    if (leaf_nc < 1) leaf_nc = 2;
    for (int64_t i = 0; i < 3 * n; ++i)
        if (!std::isfinite(pts[i])) return EINVAL_;
    p.n = n; p.k = k; p.D = D; p.Ps = Ps; p.Pa = Pa; p.P = Ps * Pa * Pa;
    p.pts.assign(pts, pts + 3 * n);
    p.ts = cheb_nodes(Ps);
    p.ta = cheb_nodes(Pa);

    // Pairwise-different points.
    {
        std::vector<std::tuple<double, double, double>> s(n);
        for (int64_t i = 0; i < n; ++i) s[i] = std::make_tuple(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
        std::sort(s.begin(), s.end());
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
    for (int d = 1; d <= D; ++d) grid_tables(p.lev[d].g);

    // Relevant boxes via the integer parts of the coordinate
    // quotients: q = floor((x - x0)/H_D), level d: q >> (D - d).
    const int64_t nmax = (int64_t)1 << (D - 1);
    std::vector<int64_t> q(3 * n);
    for (int64_t m = 0; m < n; ++m)
        for (int a = 0; a < 3; ++a) {
            double t = std::floor((pts[3 * m + a] - p.x0[a]) / p.lev[D].g.H);
            int64_t qi = t < 0.0 ? 0 : (t >= (double)nmax ? nmax - 1 : (int64_t)t);
            q[3 * m + a] = qi;
        }
    for (int d = 1; d <= D; ++d) {
        Level& L = p.lev[d];
        int sh = D - d;
        std::map<std::tuple<int64_t, int64_t, int64_t>, std::vector<int>> tmp;
        for (int64_t m = 0; m < n; ++m)
            tmp[std::make_tuple(q[3 * m] >> sh, q[3 * m + 1] >> sh, q[3 * m + 2] >> sh)].push_back((int)m);
        for (auto& kv : tmp) {
            Box b;
            std::tie(b.i, b.j, b.k) = kv.first;
            b.pts = std::move(kv.second);
            L.index[kv.first] = (int)L.boxes.size();
            L.boxes.push_back(std::move(b));
        }
    }
    // Parent / children.
    for (int d = 2; d <= D; ++d)
        for (int bi = 0; bi < (int)p.lev[d].boxes.size(); ++bi) {
            Box& b = p.lev[d].boxes[bi];
            int pa = p.lev[d - 1].find(b.i >> 1, b.j >> 1, b.k >> 1);
            if (pa < 0) return EINTERNAL_;
            b.parent = pa;
            p.lev[d - 1].boxes[pa].children.push_back(bi);
        }
    // Neighbours N B: relevant, ||a - k||_inf <= 1, B included.
    for (int d = 1; d <= D; ++d) {
        Level& L = p.lev[d];
        for (Box& b : L.boxes)
            for (int64_t di = -1; di <= 1; ++di)
                for (int64_t dj = -1; dj <= 1; ++dj)
                    for (int64_t dk = -1; dk <= 1; ++dk) {
                        int a = L.find(b.i + di, b.j + dj, b.k + dk);
                        if (a >= 0) b.nbrs.push_back(a);
                    }
    }
    // Cousins M B = (R_B^d \ N B) cap Q N P B (eq. defcousinboxes).
    for (int d = 2; d <= D; ++d) {
        Level& L = p.lev[d];
        Level& LP = p.lev[d - 1];
        for (Box& b : L.boxes) {
            std::set<int> c;
            for (int pn : LP.boxes[b.parent].nbrs)
                for (int ch : LP.boxes[pn].children) {
                    const Box& a = L.boxes[ch];
                    int64_t dist = std::max({std::llabs(a.i - b.i), std::llabs(a.j - b.j), std::llabs(a.k - b.k)});
                    if (dist > 1) c.insert(ch);
                }
            b.cousins.assign(c.begin(), c.end());
        }
    }
    // Relevant cone segments, single sweep d = 3..D (eq. defallrelevantconesegments
    // P:1509-1522): (i) segments containing a cousin point; (ii) for
    // d >= 4, segments containing a node of a relevant parent segment.
    for (int d = 3; d <= D; ++d) {
        Level& L = p.lev[d];
        for (Box& b : L.boxes) {
            std::set<int64_t> R;
            double c[3];
            box_centre(p, d, b, c);
            for (int ci : b.cousins)
                for (int m : L.boxes[ci].pts) {
                    double v[3] = {p.pts[3 * m] - c[0], p.pts[3 * m + 1] - c[1], p.pts[3 * m + 2] - c[2]};
                    Cls cl = classify(L.g, v);
                    R.insert(cell_lin(L.g, cl.is, cl.it, cl.ip));
                }
            if (d >= 4) {
                const Level& LP = p.lev[d - 1];
                const Box& Q = LP.boxes[b.parent];
                // delta = c_Q - c_B = +-H_d/2 per axis (exact; DESIGN.md contract)
                double delta[3] = {(b.i & 1) ? -L.g.H / 2.0 : L.g.H / 2.0, (b.j & 1) ? -L.g.H / 2.0 : L.g.H / 2.0,
                                   (b.k & 1) ? -L.g.H / 2.0 : L.g.H / 2.0};
                for (int64_t gq : Q.segs) {
                    int is, ith, iph;
                    decode_cell(LP.g, gq, &is, &ith, &iph);
                    for (int jp = 0; jp < p.Pa; ++jp)
                        for (int it = 0; it < p.Pa; ++it)
                            for (int ks = 0; ks < p.Ps; ++ks) {
                                double off[3];
                                node_offset(p, LP.g, is, ith, iph, ks, it, jp, off, nullptr);
                                double v[3] = {off[0] + delta[0], off[1] + delta[1], off[2] + delta[2]};
                                Cls cl = classify(L.g, v);
                                R.insert(cell_lin(L.g, cl.is, cl.it, cl.ip));
                            }
                }
            }
            b.segs.assign(R.begin(), R.end());
        }
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

// Operator application, Algorithm 1.
int apply(oracle_plan& p, const double* a2, double* out2, unsigned stage_mask, int mode) {
    const int D = p.D, P = p.P, Ps = p.Ps, Pa = p.Pa;
    std::vector<cplx> I(p.n, 0.0);
    const double* X = p.pts.data();

    // Direct evaluations on level D, neighbouring surface points:
    // I(x) += sum_{m in B, m != l} a_m G(x_l, x_m)  (raw kernel, reading R11).
    if (stage_mask & ST_NEAR) {
        const Level& L = p.lev[D];
        for (const Box& b : L.boxes)
            for (int nb : b.nbrs)
                for (int l : L.boxes[nb].pts)
                    for (int m : b.pts) {
                        if (m == l) continue;
                        double d3[3] = {X[3 * l] - X[3 * m], X[3 * l + 1] - X[3 * m + 1], X[3 * l + 2] - X[3 * m + 2]};
                        I[l] += cplx(a2[2 * m], a2[2 * m + 1]) * green_r(norm3(d3), p.k);
                    }
    }

    // Node values V (per level, per box, per relevant segment, P values).
    std::vector<std::vector<std::vector<cplx>>> V(D + 1);
    // Level D: F_B at all interpolation points of relevant leaf segments.
    if (D >= 3 && mode == MODE_NORMAL && (stage_mask & (ST_COUSIN | ST_UPWARD))) {
        const Level& L = p.lev[D];
        V[D].resize(L.boxes.size());
        for (size_t bi = 0; bi < L.boxes.size(); ++bi) {
            const Box& b = L.boxes[bi];
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

    // Interpolation onto surface points and parent interpolation points,
    // d = D, ..., 3.
    for (int d = D; d >= 3; --d) {
        const Level& L = p.lev[d];
        // Chebyshev coefficients of every relevant segment.
        std::vector<std::vector<cplx>> C(L.boxes.size());
        if (mode == MODE_NORMAL && !V[d].empty())
            for (size_t bi = 0; bi < L.boxes.size(); ++bi) {
                C[bi].assign(V[d][bi].size(), 0.0);
                for (size_t si = 0; si < L.boxes[bi].segs.size(); ++si)
                    tensor_fit(Ps, Pa, &V[d][bi][si * P], &C[bi][si * P]);
            }
        // Cousin surface points: I(x) += G(x, x_k^d) Interp F_k^d(x).
        if (stage_mask & ST_COUSIN)
            for (size_t bi = 0; bi < L.boxes.size(); ++bi) {
                const Box& b = L.boxes[bi];
                double c[3];
                box_centre(p, d, b, c);
                for (int ci : b.cousins)
                    for (int l : L.boxes[ci].pts) {
                        double v[3] = {X[3 * l] - c[0], X[3 * l + 1] - c[1], X[3 * l + 2] - c[2]};
                        cplx F;
                        if (mode == MODE_BYPASS) {
                            F = exact_F(p, d, b, a2, v);
                        } else {
                            if (C[bi].empty()) continue;  // level without values (stage mask)
                            Cls cl = classify(L.g, v);
                            int sl = seg_slot(b, cell_lin(L.g, cl.is, cl.it, cl.ip));
                            if (sl < 0) return EINTERNAL_;  // cousin point outside R_C B (impossible)
                            F = tensor_eval(Ps, Pa, &C[bi][sl * P], cl.us, cl.ut, cl.up);
                        }
                        I[l] += green_r(norm3(v), p.k) * F;
                    }
            }
        // Parent interpolation points with re-centering.
        if (d > 3 && (stage_mask & ST_UPWARD) && mode == MODE_NORMAL && !V[d].empty()) {
            const Level& LP = p.lev[d - 1];
            V[d - 1].resize(LP.boxes.size());
            for (size_t qi = 0; qi < LP.boxes.size(); ++qi) V[d - 1][qi].assign(LP.boxes[qi].segs.size() * P, 0.0);
            for (size_t bi = 0; bi < L.boxes.size(); ++bi) {
                const Box& b = L.boxes[bi];
                const Box& Q = LP.boxes[b.parent];
                double delta[3] = {(b.i & 1) ? -L.g.H / 2.0 : L.g.H / 2.0, (b.j & 1) ? -L.g.H / 2.0 : L.g.H / 2.0,
                                   (b.k & 1) ? -L.g.H / 2.0 : L.g.H / 2.0};
                for (size_t sq = 0; sq < Q.segs.size(); ++sq) {
                    int is, ith, iph;
                    decode_cell(LP.g, Q.segs[sq], &is, &ith, &iph);
                    for (int jp = 0; jp < Pa; ++jp)
                        for (int it = 0; it < Pa; ++it)
                            for (int ks = 0; ks < Ps; ++ks) {
                                double off[3];
                                node_offset(p, LP.g, is, ith, iph, ks, it, jp, off, nullptr);
                                double v[3] = {off[0] + delta[0], off[1] + delta[1], off[2] + delta[2]};
                                Cls cl = classify(L.g, v);
                                int sl = seg_slot(b, cell_lin(L.g, cl.is, cl.it, cl.ip));
                                if (sl < 0) return EINTERNAL_;  // parent node outside R_C B (impossible)
                                cplx F = tensor_eval(Ps, Pa, &C[bi][sl * P], cl.us, cl.ut, cl.up);
                                V[d - 1][b.parent][sq * P + (jp * Pa + it) * Ps + ks] += F * recenter(off, delta, p.k);
                            }
                }
            }
        }
        V[d].clear();  // level d values freed once level d-1 is filled
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

int oracle_plan_create(const double* pts, int64_t n, double k, int D, int Ps, int Pa, int leaf_ns, int leaf_nc,
                       int has_root, const double* root_c, double root_H, oracle_plan** out) {
    if (!out) return EINVAL_;
    *out = nullptr;
    oracle_plan* p = new (std::nothrow) oracle_plan();
    if (!p) return ENOMEM_;
    int st;
    try {
        st = build_plan(*p, pts, n, k, D, Ps, Pa, leaf_ns, leaf_nc, has_root, root_c, root_H);
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
    for (int64_t t = 0; t < M; ++t) {
        int64_t l = targets[t];
        if (l < 0 || l >= n) return EINVAL_;
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
    node_offset(p, g, cell[0], cell[1], cell[2], node[0], node[1], node[2], off, nullptr);
}

}  // extern "C"
