// Exact complex arithmetic and traversal-order rules shared by the sm_100a
// kernels of the "exact" precision mode.
//
// Every operation is an explicit IEEE round-to-nearest intrinsic so that no
// FMA contraction can happen: the reference is compiled for x86-64 without
// -march (proj/CMakeLists.txt), so std::complex<double> products are
// (ar*br - ai*bi, ar*bi + ai*br) with every product rounded, and complex
// division is libgcc's __divdc3.  Reproducing those expression trees and the
// summation orders fixed by the spacetree traversal makes every iterate
// bit-identical to the reference (up to the sign of exact zeros).
#pragma once

#include <cuda_runtime.h>

namespace tmg {
namespace dev {

__device__ __forceinline__ double2 cz() { return make_double2(0.0, 0.0); }
__device__ __forceinline__ double2 xadd(double2 a, double2 b) {
    return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ double2 xsub(double2 a, double2 b) {
    return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}
__device__ __forceinline__ double2 xneg(double2 a) { return make_double2(-a.x, -a.y); }
// std::complex<double> operator* (GCC lowering, no FMA)
__device__ __forceinline__ double2 xmul(double2 a, double2 b) {
    return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                        __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
// double * std::complex<double>
__device__ __forceinline__ double2 xscale(double w, double2 a) {
    return make_double2(__dmul_rn(w, a.x), __dmul_rn(w, a.y));
}
__device__ __forceinline__ bool xzero(double2 a) { return a.x == 0.0 && a.y == 0.0; }

// Per-level constants of libgcc's __divdc3 (GCC >= 12 algorithm with
// underflow/overflow scaling) for a division by the level's constant
// operator diagonal (c, d).  The host evaluates every branch that depends on
// (c, d) only; the kernel keeps the data-dependent ones.
struct DivConst {
    double c, d;       // divisor after the uniform pre-scaling
    double ratio;      // c/d (swap == 0) or d/c (swap == 1)
    double denom;      // denominator without / with the small-numerator scaling
    double denomTiny;
    int swap;          // 0: |c| < |d| branch, 1: else branch
    int pre;           // 0: none, 1: halved (|big| >= RBIG), 2: scaled up (|big| < RMIN2)
    int sub;           // |ratio| <= RMIN: alternate evaluation order
};

constexpr double kRBIG = 8.98846567431157953865e+307;   // DBL_MAX / 2
constexpr double kRMIN = 2.22507385850720138309e-308;   // DBL_MIN
constexpr double kRMIN2 = 2.220446049250313080847e-16;  // DBL_EPSILON
constexpr double kRMINSCAL = 4503599627370496.0;        // 1 / DBL_EPSILON
constexpr double kRMAX2 = kRBIG * kRMIN2;

// (a + ib) / (c + id), bit-identical to libgcc __divdc3.
__device__ __forceinline__ double2 divdc3(double a, double b, const DivConst& k) {
    double c = k.c, d = k.d, denom = k.denom;
    if (k.pre == 1) {
        a = __dmul_rn(a, 0.5);
        b = __dmul_rn(b, 0.5);
    }
    if (k.pre == 2) {
        a = __dmul_rn(a, kRMINSCAL);
        b = __dmul_rn(b, kRMINSCAL);
    } else {
        const double big = k.swap ? fabs(c) : fabs(d);
        if (((fabs(a) < kRMIN) && (fabs(b) < kRMAX2) && (big < kRMAX2)) ||
            ((fabs(b) < kRMIN) && (fabs(a) < kRMAX2) && (big < kRMAX2))) {
            a = __dmul_rn(a, kRMINSCAL);
            b = __dmul_rn(b, kRMINSCAL);
            c = __dmul_rn(c, kRMINSCAL);
            d = __dmul_rn(d, kRMINSCAL);
            denom = k.denomTiny;
        }
    }
    const double ratio = k.ratio;
    double x, y;
    if (!k.swap) {
        if (!k.sub) {
            x = __ddiv_rn(__dadd_rn(__dmul_rn(a, ratio), b), denom);
            y = __ddiv_rn(__dsub_rn(__dmul_rn(b, ratio), a), denom);
        } else {
            x = __ddiv_rn(__dadd_rn(__dmul_rn(c, __ddiv_rn(a, d)), b), denom);
            y = __ddiv_rn(__dsub_rn(__dmul_rn(c, __ddiv_rn(b, d)), a), denom);
        }
    } else {
        if (!k.sub) {
            x = __ddiv_rn(__dadd_rn(__dmul_rn(b, ratio), a), denom);
            y = __ddiv_rn(__dsub_rn(b, __dmul_rn(a, ratio)), denom);
        } else {
            x = __ddiv_rn(__dadd_rn(a, __dmul_rn(d, __ddiv_rn(b, c))), denom);
            y = __ddiv_rn(__dsub_rn(b, __dmul_rn(d, __ddiv_rn(a, c))), denom);
        }
    }
    if (isnan(x) && isnan(y)) {  // libgcc's recovery of infinities and zeros
        const double inf = __longlong_as_double(0x7ff0000000000000ll);
        if (c == 0.0 && d == 0.0 && (!isnan(a) || !isnan(b))) {
            x = __dmul_rn(copysign(inf, c), a);
            y = __dmul_rn(copysign(inf, c), b);
        } else if ((isinf(a) || isinf(b)) && isfinite(c) && isfinite(d)) {
            a = copysign(isinf(a) ? 1.0 : 0.0, a);
            b = copysign(isinf(b) ? 1.0 : 0.0, b);
            x = __dmul_rn(inf, __dadd_rn(__dmul_rn(a, c), __dmul_rn(b, d)));
            y = __dmul_rn(inf, __dsub_rn(__dmul_rn(b, c), __dmul_rn(a, d)));
        } else if ((isinf(c) || isinf(d)) && isfinite(a) && isfinite(b)) {
            c = copysign(isinf(c) ? 1.0 : 0.0, c);
            d = copysign(isinf(d) ? 1.0 : 0.0, d);
            x = __dmul_rn(0.0, __dadd_rn(__dmul_rn(a, c), __dmul_rn(b, d)));
            y = __dmul_rn(0.0, __dsub_rn(__dmul_rn(b, c), __dmul_rn(a, d)));
        }
    }
    return make_double2(x, y);
}

__device__ __forceinline__ double unit_rand(unsigned long long x) {  // cycles.cpp:802-808
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    x = x ^ (x >> 31);
    return __dsub_rn(__ddiv_rn(__dmul_rn(2.0, static_cast<double>(x >> 11)), 9007199254740992.0), 1.0);
}

// DivConst of a divisor known only on the device (per-vertex diagonals of
// cell-varying operators): the host div_const (hierarchy.cu) with explicit
// round-to-nearest operations.
__device__ __forceinline__ DivConst div_const_dev(double c, double d) {
    DivConst k{};
    const bool swap = !(fabs(c) < fabs(d));
    k.swap = swap ? 1 : 0;
    const double big = swap ? fabs(c) : fabs(d);
    k.pre = 0;
    if (big >= kRBIG) {
        c = __ddiv_rn(c, 2.0);
        d = __ddiv_rn(d, 2.0);
        k.pre = 1;
    }
    const double big2 = swap ? fabs(c) : fabs(d);
    if (big2 < kRMIN2) {
        c = __dmul_rn(c, kRMINSCAL);
        d = __dmul_rn(d, kRMINSCAL);
        k.pre = k.pre == 1 ? 1 : 2;
    }
    k.c = c;
    k.d = d;
    if (!swap) {
        k.ratio = __ddiv_rn(c, d);
        k.denom = __dadd_rn(__dmul_rn(c, k.ratio), d);
        k.denomTiny = __dadd_rn(__dmul_rn(__dmul_rn(c, kRMINSCAL), k.ratio), __dmul_rn(d, kRMINSCAL));
    } else {
        k.ratio = __ddiv_rn(d, c);
        k.denom = __dadd_rn(__dmul_rn(d, k.ratio), c);
        k.denomTiny = __dadd_rn(__dmul_rn(__dmul_rn(d, kRMINSCAL), k.ratio), __dmul_rn(c, kRMINSCAL));
    }
    k.sub = fabs(k.ratio) > kRMIN ? 0 : 1;
    return k;
}

// Per-level constants of the exact kernels (constant theta and phi).
struct LevelConst {
    double2 A[8];   // element operator entry for XOR pattern of (a, b)
    double M[8];    // reference mass entry for XOR pattern
    double2 massScale;
    DivConst div;
    double2 wRaw;   // omega_unmasked(pol, succ = L - l, n)
};

// ---- traversal orders ---------------------------------------------------
//
// The spacetree traversal (proj/src/spacetree.cpp:394-424) enters the 3^p
// children of a cell with axis 0 fastest, depth first; cells of one level are
// therefore visited in base-3 Morton order with axis p-1 the most significant
// within a digit.  Two consequences fix the floating-point summation orders:
//
// (1) cells around vertex v (c = v - 1 + e, e in {0,1}^p): the pair of cells
//     differing on axis d first differs at the digit where v_d has its lowest
//     non-zero base-3 digit, so the cells are ordered lexicographically in e
//     with the axes prioritised by (tz3(v_d), d) descending;
// (2) interior vertices are touched last in Morton order of the cell they are
//     the lower corner of, so the fine vertices 3W+k restricted into coarse
//     vertex W are grouped by their parent cell W-1+f (ordered by rule (1) at
//     the coarse level) and lexicographic (axis p-1 slowest) within a group.
// Both rules were checked against brute-force Morton sorting for p <= 3.

__device__ __forceinline__ int tz3(int x) {
    if (x == 0) return 31;
    int t = 0;
    while (x % 3 == 0) {
        x /= 3;
        ++t;
    }
    return t;
}

// Axis priority list of a permutation id (P=3: id = 2*pr0 + (pr1 > pr2)).
__host__ __device__ constexpr int perm_axis(int P, int id, int j) {
    return P == 1 ? 0
         : P == 2 ? (id == 0 ? (j == 0 ? 1 : 0) : (j == 0 ? 0 : 1))
                  : (j == 0 ? id / 2
                     : j == 1 ? ((id % 2 == 0) ? (id / 2 == 0 ? 1 : 0) : (id / 2 == 2 ? 1 : 2))
                              : ((id % 2 == 0) ? (id / 2 == 2 ? 1 : 2) : (id / 2 == 0 ? 1 : 0)));
}

// i-th cell (as e bitmask) around a vertex for permutation id.
__host__ __device__ constexpr int perm_cell(int P, int id, int i) {
    int e = 0;
    for (int j = 0; j < P; ++j) e |= ((i >> (P - 1 - j)) & 1) << perm_axis(P, id, j);
    return e;
}

// Permutation id from the per-axis base-3 trailing-zero counts.
template <int P>
__device__ __forceinline__ int perm_id(const int* idx) {
    if (P == 1) return 0;
    if (P == 2) {
        // id 0: axis 1 first (t1 > t0, or tie -> higher axis first)
        return (tz3(idx[1]) >= tz3(idx[0])) ? 0 : 1;
    }
    const int k0 = tz3(idx[0]) * 4 + 0, k1 = tz3(idx[1]) * 4 + 1, k2 = tz3(idx[2]) * 4 + 2;
    int pr0, pr1, pr2;
    if (k0 > k1 && k0 > k2) {
        pr0 = 0;
        pr1 = k1 > k2 ? 1 : 2;
        pr2 = k1 > k2 ? 2 : 1;
    } else if (k1 > k2) {
        pr0 = 1;
        pr1 = k0 > k2 ? 0 : 2;
        pr2 = k0 > k2 ? 2 : 0;
    } else {
        pr0 = 2;
        pr1 = k0 > k1 ? 0 : 1;
        pr2 = k0 > k1 ? 1 : 0;
    }
    return 2 * pr0 + (pr1 > pr2 ? 1 : 0);
}

}  // namespace dev
}  // namespace tmg
