// rad_table.h — host-side construction of the Box-Muller radius table RT
// (spec/RNG.md §3, revision R10c): 736 rows x 4 binary32 coefficients of the
// cubic interpolating sqrt(-2 ln u1) at four dyadic nodes per segment, built
// in binary64 in the spec's operation order.  The CPU checker carries out the
// same construction with its own code; the two share none.  Used by
// distill.cu (uploaded once per device) and tools/.
#pragma once
#include <cmath>
#include <cuda_runtime.h>

namespace distill {

inline void build_rad_table(float4* rt) {
    const double nodes[4] = {-3.0 / 128.0, -1.0 / 128.0, 1.0 / 128.0, 3.0 / 128.0};
    for (int reg = 0; reg < 2; ++reg) {
        for (int oct = 0; oct < 23; ++oct) {
            for (int sub = 0; sub < 16; ++sub) {
                const double centre = 1.0 + (2.0 * sub + 1.0) / 32.0;
                double f[4];
                for (int k = 0; k < 4; ++k) {
                    const double x = (centre + nodes[k]) * std::ldexp(1.0, oct);
                    const double n = reg ? 16777216.0 - x : x;
                    f[k] = std::sqrt(-2.0 * std::log(n * 0x1p-24));
                }
                const double d01 = (f[1] - f[0]) / (nodes[1] - nodes[0]);
                const double d12 = (f[2] - f[1]) / (nodes[2] - nodes[1]);
                const double d23 = (f[3] - f[2]) / (nodes[3] - nodes[2]);
                const double d012 = (d12 - d01) / (nodes[2] - nodes[0]);
                const double d123 = (d23 - d12) / (nodes[3] - nodes[1]);
                const double a3 = (d123 - d012) / (nodes[3] - nodes[0]);
                const double p01 = nodes[0] * nodes[1];
                const double a2 = d012 - a3 * ((nodes[0] + nodes[1]) + nodes[2]);
                const double a1 = (d01 - d012 * (nodes[0] + nodes[1])) + a3 * ((p01 + nodes[0] * nodes[2]) + nodes[1] * nodes[2]);
                const double a0 = ((f[0] - d01 * nodes[0]) + d012 * p01) - a3 * (p01 * nodes[2]);
                rt[368 * reg + 16 * oct + sub] = make_float4((float)a0, (float)a1, (float)a2, (float)a3);
            }
        }
    }
}

}  // namespace distill
