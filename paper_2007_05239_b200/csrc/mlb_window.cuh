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

// The same windows for K offsets at once (several axes and / or points of a
// lane): every coefficient is read once and feeds K FMAs.  The window
// coefficients are ~(2m+1)(deg/2+1) doubles, more than the uniform register
// file holds, so each Horner step otherwise costs a per-thread constant load
// (LDC) next to its DFMA -- on the d <= 2 gather that saturated the memory
// pipe.  Per offset the arithmetic is kb_windows' (bitwise the same values).
template <int M, int K>
__device__ __forceinline__ void kb_windows_k(const double (&f)[K], const WinCoef& c, double (&w)[K][2 * M + 1]) {
    constexpr int NE = WinDeg<M>::ne;
    constexpr int NO = WinDeg<M>::no;
    constexpr int DM = WinDeg<M>::deg;
    double s[K], s2[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        s[k] = 2.0 * f[k] - 1.0;
        s2[k] = s[k] * s[k];
    }
#pragma unroll
    for (int q = 1; q <= M; ++q) {
        double e[K], od[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            e[k] = c.e[q - 1][NE - 1];
            od[k] = c.o[q - 1][NO - 1];
        }
#pragma unroll
        for (int j = NE - 2; j >= 0; --j) {
            const double cj = c.e[q - 1][j];
#pragma unroll
            for (int k = 0; k < K; ++k) e[k] = fma(e[k], s2[k], cj);
        }
#pragma unroll
        for (int j = NO - 2; j >= 0; --j) {
            const double cj = c.o[q - 1][j];
#pragma unroll
            for (int k = 0; k < K; ++k) od[k] = fma(od[k], s2[k], cj);
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const double o = od[k] * s[k];
            w[k][q + M] = e[k] + o;
            w[k][1 - q + M] = e[k] - o;
        }
    }
    double pm[K];
#pragma unroll
    for (int k = 0; k < K; ++k) pm[k] = c.mm[DM];
#pragma unroll
    for (int j = DM - 1; j >= 0; --j) {
        const double cj = c.mm[j];
#pragma unroll
        for (int k = 0; k < K; ++k) pm[k] = fma(pm[k], s[k], cj);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) w[k][0] = pm[k];
}

// acc[o] += sum_k phi(f_k - o) sv_k for K points of a lane, windows consumed
// as they are formed (no K x (2m+1) window array held): the d = 1 streaming
// spread.  Same per-point window arithmetic as kb_windows.
template <int M, int K>
__device__ __forceinline__ void kb_accumulate_k(const double (&f)[K], const double (&sv)[K], const WinCoef& c,
                                                double (&acc)[2 * M + 1]) {
    constexpr int NE = WinDeg<M>::ne;
    constexpr int NO = WinDeg<M>::no;
    constexpr int DM = WinDeg<M>::deg;
    double s[K], s2[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        s[k] = 2.0 * f[k] - 1.0;
        s2[k] = s[k] * s[k];
    }
#pragma unroll
    for (int q = 1; q <= M; ++q) {
        double e[K], od[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            e[k] = c.e[q - 1][NE - 1];
            od[k] = c.o[q - 1][NO - 1];
        }
#pragma unroll
        for (int j = NE - 2; j >= 0; --j) {
            const double cj = c.e[q - 1][j];
#pragma unroll
            for (int k = 0; k < K; ++k) e[k] = fma(e[k], s2[k], cj);
        }
#pragma unroll
        for (int j = NO - 2; j >= 0; --j) {
            const double cj = c.o[q - 1][j];
#pragma unroll
            for (int k = 0; k < K; ++k) od[k] = fma(od[k], s2[k], cj);
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const double o = od[k] * s[k];
            acc[q + M] = fma(e[k] + o, sv[k], acc[q + M]);
            acc[1 - q + M] = fma(e[k] - o, sv[k], acc[1 - q + M]);
        }
    }
    double pm[K];
#pragma unroll
    for (int k = 0; k < K; ++k) pm[k] = c.mm[DM];
#pragma unroll
    for (int j = DM - 1; j >= 0; --j) {
        const double cj = c.mm[j];
#pragma unroll
        for (int k = 0; k < K; ++k) pm[k] = fma(pm[k], s[k], cj);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) acc[0] = fma(pm[k], sv[k], acc[0]);
}

// acc[k] += sum_o phi(f_k - o) g_k[o] for K points of a lane (g_k: the
// (2m+1) grid values of point k's stencil), windows consumed as formed: the
// d = 1 streaming gather.
template <int M, int K>
__device__ __forceinline__ void kb_dot_k(const double (&f)[K], const WinCoef& c, const double* __restrict__ gbase,
                                         const int (&cell)[K], double (&acc)[K]) {
    constexpr int NE = WinDeg<M>::ne;
    constexpr int NO = WinDeg<M>::no;
    constexpr int DM = WinDeg<M>::deg;
    double s[K], s2[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        s[k] = 2.0 * f[k] - 1.0;
        s2[k] = s[k] * s[k];
    }
#pragma unroll
    for (int q = 1; q <= M; ++q) {
        double e[K], od[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            e[k] = c.e[q - 1][NE - 1];
            od[k] = c.o[q - 1][NO - 1];
        }
#pragma unroll
        for (int j = NE - 2; j >= 0; --j) {
            const double cj = c.e[q - 1][j];
#pragma unroll
            for (int k = 0; k < K; ++k) e[k] = fma(e[k], s2[k], cj);
        }
#pragma unroll
        for (int j = NO - 2; j >= 0; --j) {
            const double cj = c.o[q - 1][j];
#pragma unroll
            for (int k = 0; k < K; ++k) od[k] = fma(od[k], s2[k], cj);
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const double o = od[k] * s[k];
            acc[k] = fma(e[k] + o, gbase[cell[k] + q + M], acc[k]);
            acc[k] = fma(e[k] - o, gbase[cell[k] + 1 - q + M], acc[k]);
        }
    }
    double pm[K];
#pragma unroll
    for (int k = 0; k < K; ++k) pm[k] = c.mm[DM];
#pragma unroll
    for (int j = DM - 1; j >= 0; --j) {
        const double cj = c.mm[j];
#pragma unroll
        for (int k = 0; k < K; ++k) pm[k] = fma(pm[k], s[k], cj);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = fma(pm[k], gbase[cell[k]], acc[k]);
}

}  // namespace mlb
