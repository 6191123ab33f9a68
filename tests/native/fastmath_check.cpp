// CPU harness for paper_2010_02857_b200/csrc/fastmath.cuh (compiled as plain C++):
// reads "a y x" (atan2), "b y x" (atan2_2pi) or "s x" (sincos) lines, prints results with %.17g.
#include <cstdio>
#include <cstring>
#include "../../paper_2010_02857_b200/csrc/fastmath.cuh"
int main() {
    char op[8];
    double u, v;
    while (std::scanf("%7s", op) == 1) {
        if (!std::strcmp(op, "a")) {
            if (std::scanf("%lf %lf", &u, &v) != 2) return 1;
            std::printf("%.17g\n", ifgf::fm::atan2(u, v));
        } else if (!std::strcmp(op, "b")) {
            if (std::scanf("%lf %lf", &u, &v) != 2) return 1;
            std::printf("%.17g\n", ifgf::fm::atan2_2pi(u, v));
        } else {
            if (std::scanf("%lf", &u) != 1) return 1;
            double s, c;
            ifgf::fm::sincos(u, &s, &c);
            std::printf("%.17g %.17g\n", s, c);
        }
    }
    return 0;
}
