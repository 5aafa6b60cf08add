// Kaiser-Bessel window of the reference (fastsum.py:158-167) as polynomials.
//
// phi(t) = sinh(b sqrt(m^2-t^2)) / (pi sqrt(m^2-t^2)) (and its sin / b/pi
// branches) is ONE entire function of z = m^2 - t^2, so for the 2m+1 stencil
// offsets o = -m..m the values phi(f - o), f in [0,1), are entire functions
// of s = 2f - 1 and are reproduced to ~1e-15 of max(phi) by degree-13/15
// polynomials (fitted on the host, checked at plan build).  The symmetry
// phi(t) = phi(-t) gives P_{1-q}(s) = P_q(-s), so q = 1..m share one even
// part E_q(s^2) and one odd part O_q(s^2): two windows for one polynomial.
#pragma once
#include "mlb_internal.cuh"

namespace mlb {

// Odd degrees: P = E(s^2) + s O(s^2) with equally many even and odd terms.
// Degree 13 (m >= 4) / 15 (m <= 3) fits as tightly as 14 / 16 did (<= 5e-15
// of max phi through float64 Horner) and saves one FMA per polynomial.
template <int M>
struct WinDeg {
    static constexpr int deg = (M <= 3) ? 15 : 13;
    static constexpr int ne = deg / 2 + 1;        // s^0, s^2, ..., s^(deg-1)
    static constexpr int no = (deg + 1) / 2;      // s^1, s^3, ..., s^deg
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

// The d = 1 streaming kernels never need the window VALUES, only their sums
// against sv (spread) or the grid (gather), and the pair P_q(s) = E_q + s O_q,
// P_{1-q}(s) = E_q - s O_q shares E_q and O_q.  So the spread keeps the even
// and odd sums apart -- ae[q] += E_q sv, ao[q] += O_q (s sv), a0 += P_{-m} sv:
// two FMAs per pair instead of the product, two adds and two FMAs -- and the
// cell's window sums are formed at the flush: acc[q+m] = ae + ao, acc[1-q+m]
// = ae - ao.  Same arithmetic as kb_windows up to that association.
template <int M, int K>
__device__ __forceinline__ void kb_accumulate_k(const double (&f)[K], const double (&sv)[K], const WinCoef& c,
                                                double (&ae)[M], double (&ao)[M], double& a0) {
    constexpr int NE = WinDeg<M>::ne;
    constexpr int NO = WinDeg<M>::no;
    constexpr int DM = WinDeg<M>::deg;
    double s[K], s2[K], ssv[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        s[k] = 2.0 * f[k] - 1.0;
        s2[k] = s[k] * s[k];
        ssv[k] = s[k] * sv[k];
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
            ae[q - 1] = fma(e[k], sv[k], ae[q - 1]);
            ao[q - 1] = fma(od[k], ssv[k], ao[q - 1]);
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
    for (int k = 0; k < K; ++k) a0 = fma(pm[k], sv[k], a0);
}

// Gather counterpart: acc_k = P_{-m} g[c] + sum_q E_q GS[c][q] + s sum_q O_q
// GD[c][q] with the per-cell pair sums GS = g[c+q+m] + g[c+1-q+m] and
// differences GD = g[c+q+m] - g[c+1-q+m] precomputed (tab: per cell, 2m + 1
// doubles: g[c], then (GS, GD) per q).  2m + 3 FP64 ops per point besides the
// Horner steps, instead of 5m + 1.
template <int M, int K>
__device__ __forceinline__ void kb_dot_k(const double (&f)[K], const WinCoef& c, const double* __restrict__ tab,
                                         const int (&cell)[K], double (&acc)[K]) {
    constexpr int NE = WinDeg<M>::ne;
    constexpr int NO = WinDeg<M>::no;
    constexpr int DM = WinDeg<M>::deg;
    constexpr int TS = 2 * M + 1;
    double s[K], s2[K], ao[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        s[k] = 2.0 * f[k] - 1.0;
        s2[k] = s[k] * s[k];
        ao[k] = 0.0;
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
            const double* t = tab + cell[k] * TS + 2 * q - 1;
            acc[k] = fma(e[k], t[0], acc[k]);
            ao[k] = fma(od[k], t[1], ao[k]);
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
    for (int k = 0; k < K; ++k) acc[k] = fma(s[k], ao[k], fma(pm[k], tab[cell[k] * TS], acc[k]));
}

}  // namespace mlb
