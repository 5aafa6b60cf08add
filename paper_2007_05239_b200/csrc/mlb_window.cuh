// Kaiser-Bessel window of the reference (fastsum.py:158-167) as polynomials.
//
// phi(t) = sinh(b sqrt(m^2-t^2)) / (pi sqrt(m^2-t^2)) (and its sin / b/pi
// branches) is ONE entire function of z = m^2 - t^2, so for the 2m+1 stencil
// offsets o = -m..m the values phi(f - o), f in [0,1), are entire functions
// of s = 2f - 1 and are reproduced to ~1e-15 of max(phi) by degree-14/16
// polynomials (fitted on the host, checked at plan build).  The symmetry
// phi(t) = phi(-t) gives P_{1-q}(s) = P_q(-s), so q = 1..m share one even
// part E_q(s^2) and one odd part O_q(s^2): two windows for one polynomial.
#pragma once
#include "mlb_internal.cuh"

namespace mlb {

template <int M>
struct WinDeg {
    static constexpr int deg = (M <= 3) ? 16 : 14;
    static constexpr int ne = deg / 2 + 1;  // s^0, s^2, ..., s^deg
    static constexpr int no = deg / 2;      // s^1, s^3, ..., s^(deg-1)
};

// w[o + M] = phi(f - o), o = -M..M
template <int M>
__device__ __forceinline__ void kb_windows(double f, const WinCoef& c, double* w) {
    constexpr int NE = WinDeg<M>::ne;
    constexpr int NO = WinDeg<M>::no;
    constexpr int DM = WinDeg<M>::deg;
    const double s = 2.0 * f - 1.0;
    const double s2 = s * s;
#pragma unroll
    for (int q = 1; q <= M; ++q) {
        double e = c.e[q - 1][NE - 1];
#pragma unroll
        for (int j = NE - 2; j >= 0; --j) e = fma(e, s2, c.e[q - 1][j]);
        double od = c.o[q - 1][NO - 1];
#pragma unroll
        for (int j = NO - 2; j >= 0; --j) od = fma(od, s2, c.o[q - 1][j]);
        od *= s;
        w[q + M] = e + od;        // o = q
        w[1 - q + M] = e - od;    // o = 1 - q
    }
    double p = c.mm[DM];
#pragma unroll
    for (int j = DM - 1; j >= 0; --j) p = fma(p, s, c.mm[j]);
    w[0] = p;                      // o = -M
}

}  // namespace mlb
