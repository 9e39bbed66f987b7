// Fused fine pass for 2D (see fused2.cuh).

#include "fused2.cuh"

#include <algorithm>
#include <type_traits>

#include "lattice.cuh"

namespace tmg {
namespace fused2 {

namespace {

// ---- complex arithmetic on double2 (complex128) and float2 (complex64), as fused3.cu ----
template <class S> struct Cx;
template <> struct Cx<double> { using T = double2; };
template <> struct Cx<float> { using T = float2; };
__device__ __forceinline__ double2 mk(double x, double y) { return make_double2(x, y); }
__device__ __forceinline__ float2 mk(float x, float y) { return make_float2(x, y); }
template <class C> __device__ __forceinline__ C zero();
template <> __device__ __forceinline__ double2 zero<double2>() { return make_double2(0.0, 0.0); }
template <> __device__ __forceinline__ float2 zero<float2>() { return make_float2(0.f, 0.f); }
__device__ __forceinline__ double2 zero2() { return zero<double2>(); }
template <class C> __device__ __forceinline__ C add(C a, C b) { return mk(a.x + b.x, a.y + b.y); }
template <class C> __device__ __forceinline__ C sub(C a, C b) { return mk(a.x - b.x, a.y - b.y); }
template <class C> __device__ __forceinline__ C mul(C a, C b) {
    return mk(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
template <class C> __device__ __forceinline__ C mac(C acc, C a, C b) {
    return mk(fma(a.x, b.x, fma(-a.y, b.y, acc.x)), fma(a.x, b.y, fma(a.y, b.x, acc.y)));
}
template <class C, class S> __device__ __forceinline__ C axpy(S w, C v, C acc) {
    return mk(fma(w, v.x, acc.x), fma(w, v.y, acc.y));
}
template <class C, class S> __device__ __forceinline__ C lerpw(C c0, C c1, S w1) {
    return mk(fma(w1, c1.x - c0.x, c0.x), fma(w1, c1.y - c0.y, c0.y));
}
__device__ __forceinline__ double relw(int r) { return r == 1 ? (1.0 / 3.0) : r == 2 ? (2.0 / 3.0) : (r == 3 ? 1.0 : 0.0); }
// complex128 <-> the kernel's complex type
__device__ __forceinline__ double2 to_c(double2 v, double2) { return v; }
__device__ __forceinline__ float2 to_c(double2 v, float2) { return make_float2(static_cast<float>(v.x), static_cast<float>(v.y)); }
__device__ __forceinline__ double2 to_d(double2 v) { return v; }
__device__ __forceinline__ double2 to_d(float2 v) { return make_double2(v.x, v.y); }

template <class C>
__device__ __forceinline__ C stage_sc(C smooth, C w, bool cp, int bpx, int hb) {
    if (bpx) return cp ? zero<C>() : mul(w, smooth);
    if ((hb && cp) || (w.x == 0 && w.y == 0)) return zero<C>();
    return mul(w, smooth);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}

// 16-byte cp.async; zero-fills the destination when !valid (src-size 0)
__device__ __forceinline__ void cp_async16z(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src), "r"(valid ? 16 : 0)
                 : "memory");
}

constexpr int kRing = 4;  // rows in flight
constexpr int kHaloT = TX >= 64 ? 32 : 0;   // first of the two halo-column threads
constexpr int kCvT = TX >= 128 ? 64 : 0;    // first coarse-row thread
static_assert(kCvT + CXW <= TX, "coarse-row tasks");

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bulk_row(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void rbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "TMG_RW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra TMG_RW_%=;\n"
        "}\n" ::"r"(su32(bar)),
        "r"(parity)
        : "memory");
}

// S = double: complex128; S = float: the finest level stored and computed in
// complex64 (precision = fast-complex64), coarse values / partials / norms in double.
// Bulk copies need 16-byte aligned addresses and sizes: x0 - 1 and every row
// length are even, so complex64 rows of v start aligned; its b rows are copied
// from x0 - 1 as well (BOFF = 1: one leading element the kernel skips).
template <bool BPX, class S>
__global__ void __launch_bounds__(TX) k_fused2(const Args a) {
    using C = typename Cx<S>::T;
    constexpr int BOFF = sizeof(C) == 8 ? 1 : 0;
    constexpr int TXB = TX + 2 * BOFF;
    dev::griddep_wait();
    __shared__ C Pb[2][TX + 2];                // corrected rows (x halo at 0 and TX+1)
    __shared__ C Vb[BPX ? 4 : 2][CXW];         // y-interpolated coarse rows (sc[, si])
    __shared__ C tb[TX];                       // y-restricted columns
    __shared__ unsigned long long rbar[kRing]; // row ring: one mbarrier per slot (bulk copies)
    extern __shared__ __align__(16) unsigned char dynRaw[];
    auto Ru = reinterpret_cast<C(*)[TX + 2]>(dynRaw);                                        // row ring: v (own columns + x halo)
    auto Rb = reinterpret_cast<C(*)[TXB]>(dynRaw + kRing * (TX + 2) * sizeof(C));            // row ring: b
    double2* Cs = reinterpret_cast<double2*>(dynRaw + kRing * (TX + 2 + TXB) * sizeof(C));  // coarse-row ring: sc [4][CXW] (+ si [4][CXW])

    const int tid = threadIdx.x;
    const int m = a.g.m, mc = a.g.mc;
    const int x0 = 1 + blockIdx.x * TX, xe = min(x0 + TX, m);
    const int y0 = 1 + blockIdx.y * a.g.yc, y1 = min(y0 + a.g.yc, m);
    const int nrows = y1 - y0 + 2;
    const long long n1 = a.n1;
    const int cx0 = (x0 - 1) / 3;
    const int x = x0 + tid;
    const bool owned = x < xe;

    // own column: coarse interpolation slot and weight
    const int qxo = min(x / 3, mc - 1);
    const int vo = qxo - cx0;
    const S wxo = static_cast<S>(relw(x - 3 * qxo));
    const bool cpx = x % 3 == 0;
    // halo columns (threads 0 and 1): x0 - 1 and xe
    // per-row side tasks spread over the warps (the row barrier waits for the
    // busiest): halo columns on warp 1, coarse rows on warps 2-3, the bulk-copy
    // issue on thread 0, the restriction flush on the last threads
    const int hx = tid == kHaloT ? x0 - 1 : xe;
    const bool haloThread = tid == kHaloT || tid == kHaloT + 1;
    const bool hin = haloThread && hx >= 1 && hx <= m - 1;
    const int hq = min(max(hx, 0) / 3, mc - 1);
    const int hv = hq - cx0;
    const S hw = static_cast<S>(relw(hx - 3 * hq));
    const bool hcpx = hx % 3 == 0;
    const int hslot = tid == kHaloT ? 0 : (xe - x0) + 1;
    const int ct = tid - kCvT;  // coarse-row task: coarse column cx0 + ct

    // coarse rows feeding the strip (sc[, si]) through a 4-slot ring (slot q % 4):
    // rows q(y0-1) and +1 up front, then coarse row Q + 1 rides with fine row
    // 3Q - 1's ring group, so it has landed when computeV(3Q) runs (one row later)
    const int cxo = min(cx0 + ct, mc);
    auto issueCoarse = [&](int q) {
        if (ct >= 0 && ct < CXW && q <= mc) {
            const long long g = cxo + static_cast<long long>(a.n1c) * q;
            cp_async16(Cs + (q & 3) * CXW + ct, a.scC + g);
            if (BPX) cp_async16(Cs + (4 + (q & 3)) * CXW + ct, a.siC + g);
        }
    };
    {
        const int q0 = min(max(y0 - 1, 0) / 3, mc - 1);
        issueCoarse(q0);
        issueCoarse(q0 + 1);
        asm volatile("cp.async.wait_all;" ::: "memory");
    }
    // coarse rows of fine row yy, for coarse columns cx0 + ct; w1y: the row's weight between
    // its two coarse rows (the caller knows yy % 3)
    auto computeV = [&](int yy, double w1y, int vb) {
        if (ct < 0 || ct >= CXW) return;
        const int qy = min(max(yy, 0) / 3, mc - 1);
        const double2* c0 = Cs + (qy & 3) * CXW + ct;
        const double2* c1 = Cs + ((qy + 1) & 3) * CXW + ct;
        Vb[vb][ct] = to_c(lerpw(c0[0], c1[0], w1y), C{});
        if (BPX) Vb[2 + vb][ct] = to_c(lerpw(c0[4 * CXW], c1[4 * CXW], w1y), C{});
    };

    // restriction slots of this strip
    const int Xa = x0 / 3, Xb = (xe + 1) / 3, nsx = Xb - Xa + 1;
    const long long strip = blockIdx.x;
    double2* part = a.partial + (static_cast<long long>(blockIdx.y) * a.g.sy * a.g.nbx + strip) * SXP;
    const long long zStride = static_cast<long long>(a.g.nbx) * SXP;
    const int zBase = (y0 - 1) / 3;
    int zLow = zBase;
    const int ti = TX - 1 - tid;  // slot tasks run away from the halo / coarse-row threads
    auto flush = [&](int zi) {
        if (ti < nsx) {
            const int X = Xa + ti;
            C acc = zero<C>();
#pragma unroll
            for (int kx = -2; kx <= 2; ++kx) {
                const int fx = 3 * X + kx;
                if (fx < x0 || fx >= xe) continue;
                const S wx = static_cast<S>(kx == 0 ? 1.0 : (kx == 1 || kx == -1) ? (2.0 / 3.0) : (1.0 / 3.0));
                acc = axpy(wx, tb[fx - x0], acc);
            }
            part[zi * zStride + ti] = to_d(acc);
        }
    };
    bool pend = false;
    int ziPend = 0;

    const C k0 = to_c(a.k.c[0], C{}), k1 = to_c(a.k.c[1], C{}), k2 = to_c(a.k.c[2], C{});
    const bool zeroSc = a.level < a.ellMin;
    const bool injectOK = BPX && a.level > a.ellMin && cpx && owned;
    double nmax = 0.0, nsum = 0.0;
    C accLo = zero<C>(), accHi = zero<C>();
    C Aprev = zero<C>(), Acur = zero<C>();

    // Row ring: row yy's state v = u + sc (fused3.cuh "v-form") over the strip
    // and its halo columns [x0 - 1, xe], and its load vector b over [x0, xe),
    // bulk-copied by one thread kRing - 1 rows ahead into slot (yy - y0 + 1) % kRing
    // (mbarrier per slot); coarse row Q + 1 (sc[, si]) rides with fine row 3Q - 1,
    // so it has landed when computeV(3Q) runs (one row later).  Rows off the
    // domain (0, m) are not copied: phase B reads them as zeros.  The row loop is
    // unrolled by three (yy % 3 a compile-time constant, y0 = 1 mod 3).
    if (tid == 0) {
        for (int k = 0; k < kRing; ++k)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&rbar[k])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const unsigned uBytes = static_cast<unsigned>(xe - x0 + 2) * static_cast<unsigned>(sizeof(C)),
                   bBytes = static_cast<unsigned>(xe - x0 + 2 * BOFF) * static_cast<unsigned>(sizeof(C));
    const C* gU = static_cast<const C*>(static_cast<const void*>(a.u));
    const C* gB = static_cast<const C*>(static_cast<const void*>(a.b));
    const int cCount = min(CXW, mc + 1 - cx0);
    auto issueRow = [&](int it2, auto U3) {  // thread 0; U3: (y0 - 1 + it2) % 3
        constexpr int uu = decltype(U3)::value;
        const int yy = y0 - 1 + it2, slot = it2 & (kRing - 1);
        const bool yin = yy >= 1 && yy <= m - 1, bin = yy >= y0 && yy < y1;
        const int q = (yy + 1) / 3 + 1;
        const bool coarse = uu == 2 && yy >= 2 && (yy + 1) / 3 < mc && q <= mc;  // needed from fine row yy + 1
        const unsigned cb = coarse ? static_cast<unsigned>(cCount) * 16u : 0u;
        const unsigned tx = (yin ? uBytes : 0u) + (bin ? bBytes : 0u) + (BPX ? 2u : 1u) * cb;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&rbar[slot])), "r"(tx) : "memory");
        const long long row = n1 * yy;
        if (yin) bulk_row(&Ru[slot][0], gU + (x0 - 1) + row, uBytes, &rbar[slot]);
        if (bin) bulk_row(&Rb[slot][0], gB + (x0 - BOFF) + row, bBytes, &rbar[slot]);
        if (coarse) {
            const long long g = cx0 + static_cast<long long>(a.n1c) * q;
            bulk_row(Cs + (q & 3) * CXW, a.scC + g, cb, &rbar[slot]);
            if (BPX) bulk_row(Cs + (4 + (q & 3)) * CXW, a.siC + g, cb, &rbar[slot]);
        }
    };
    using U0 = std::integral_constant<int, 0>;
    using U1 = std::integral_constant<int, 1>;
    using U2 = std::integral_constant<int, 2>;
    if (tid == 0) {
        issueRow(0, U0{});
        if (nrows > 1) issueRow(1, U1{});
        if (nrows > 2) issueRow(2, U2{});
    }
    C cPrev = zero<C>();
    C bq = zero<C>();
    {
        const int yf = y0 - 1, qf = min(max(yf, 0) / 3, mc - 1);
        computeV(yf, relw(yf - 3 * qf), 0);
    }
    __syncthreads();

    C* uOut = static_cast<C*>(static_cast<void*>(a.uNew)) + x + n1 * y0;  // row yy - 1 of the residual steps (it >= 2), advanced by each
    C* scOut = static_cast<C*>(static_cast<void*>(a.scNew)) + x + n1 * y0;
    const C wRaw = to_c(a.k.wRaw, C{}), invDiag = to_c(a.k.invDiag, C{});
    auto step = [&](int it, auto U3) {
        constexpr int u3 = decltype(U3)::value;  // yy % 3
        constexpr int kz = (u3 + 2) % 3;         // (yy - 1) % 3
        const int yy = y0 - 1 + it;
        const bool yin = yy >= 1 && yy <= m - 1;
        rbar_wait(&rbar[it & (kRing - 1)], static_cast<unsigned>(it / kRing) & 1u);  // row yy landed
        const C uC = Ru[it & (kRing - 1)][tid + 1];
        const C huC = haloThread ? Ru[it & (kRing - 1)][hslot] : zero<C>();
        if (it >= 2) bq = Rb[(it + kRing - 1) & (kRing - 1)][tid + BOFF];  // b of row yy - 1 (the residual row)
        const C* V = Vb[it & 1];
        C* P = Pb[it & 1];
        // ---- phase B: corrected row yy ----
        C cOwn = zero<C>();
        if (yin && owned) {
            C scv = lerpw(V[vo], V[vo + 1], wxo);
            if (BPX && !(cpx && u3 == 0)) scv = sub(scv, lerpw(Vb[2 + (it & 1)][vo], Vb[2 + (it & 1)][vo + 1], wxo));
            cOwn = add(uC, scv);
        }
        if (owned) P[tid + 1] = cOwn;
        if (haloThread) {
            C c = zero<C>();
            if (yin && hin) {
                C scv = lerpw(V[hv], V[hv + 1], hw);
                if (BPX && !(hcpx && u3 == 0)) scv = sub(scv, lerpw(Vb[2 + (it & 1)][hv], Vb[2 + (it & 1)][hv + 1], hw));
                c = add(huC, scv);
            }
            P[hslot] = c;
        }
        // row yy + 1 has residue (u3 + 1) % 3; the top lattice row m = 3 mc takes weight 1
        if (it + 1 < nrows) computeV(yy + 1, yy + 1 == m ? 1.0 : relw((u3 + 1) % 3), (it + 1) & 1);
        __syncthreads();
        // every thread has read row yy - 1's slot: refill it with row yy + 3 (same residue)
        if (tid == 0 && it + kRing - 1 < nrows) issueRow(it + kRing - 1, U3);
        // ---- phase C ----
        if (pend) {
            flush(ziPend);
            pend = false;
        }
        const C E = add(P[tid], P[tid + 2]);
        C T = mul(k1, cOwn);
        T = mac(T, k2, E);
        C U = mul(k0, cOwn);
        U = mac(U, k1, E);
        if (it >= 2) {
            const C hu = add(Aprev, T);
            const C r = owned ? sub(bq, hu) : zero<C>();
            const S m2 = fma(r.x, r.x, r.y * r.y);
            nmax = static_cast<double>(m2) > nmax ? static_cast<double>(m2) : nmax;  // == fmax (a NaN is ignored)
            nsum += static_cast<double>(m2);
            const C smooth = mul(r, invDiag);
            const C scn = zeroSc ? zero<C>() : stage_sc(smooth, wRaw, cpx && kz == 0, BPX ? 1 : 0, a.hb);
            if (owned) {
                if (a.writeSc) *scOut = scn;
                *uOut = add(cPrev, scn);  // next state v of row yy - 1
            }
            if (BPX && kz == 0 && injectOK)
                a.sinextC[x / 3 + static_cast<long long>(a.n1c) * ((yy - 1) / 3)] = to_d(mul(wRaw, smooth));
            if (kz == 0) {
                accLo = add(accLo, r);
            } else if (kz == 1) {
                accLo = axpy(static_cast<S>(2.0 / 3.0), r, accLo);
                accHi = axpy(static_cast<S>(1.0 / 3.0), r, accHi);
            } else {
                accLo = axpy(static_cast<S>(1.0 / 3.0), r, accLo);
                accHi = axpy(static_cast<S>(2.0 / 3.0), r, accHi);
                tb[tid] = accLo;
                accLo = accHi;
                accHi = zero<C>();
                pend = true;  // x-reduction on the next row's barrier
                ziPend = zLow - zBase;
                ++zLow;
            }
            uOut += n1;
            scOut += n1;
        }
        Aprev = add(Acur, U);
        Acur = T;
        cPrev = cOwn;
    };
    // yy = y0 - 1 + it and y0 = 1 (mod 3): yy % 3 == it % 3
    for (int it = 0; it < nrows; it += 3) {
        step(it, U0{});
        if (it + 1 >= nrows) break;
        step(it + 1, U1{});
        if (it + 2 >= nrows) break;
        step(it + 2, U2{});
    }
    __syncthreads();
    if (pend) flush(ziPend);
    __syncthreads();
    tb[tid] = accLo;
    __syncthreads();
    flush(zLow - zBase);
    __syncthreads();
    tb[tid] = accHi;
    __syncthreads();
    flush(zLow + 1 - zBase);
    dev::block_norms(nmax, nsum, a.norms);
}

// derive_u: k_fused2's phase B for one point, from global memory
template <class S>
__global__ void __launch_bounds__(256) k_derive_u2(const typename Cx<S>::T* __restrict__ vOld,
                                                   const double2* __restrict__ scTD, const double2* __restrict__ siTD,
                                                   unsigned n1, unsigned n1c, unsigned fa, unsigned fb,
                                                   double2* __restrict__ uOut) {
    using C = typename Cx<S>::T;
    const int m = static_cast<int>(n1) - 1, mc = static_cast<int>(n1c) - 1;
    for (unsigned f = fa + blockIdx.x * blockDim.x + threadIdx.x; f < fb; f += gridDim.x * blockDim.x) {
        const int y = static_cast<int>(f / n1), x = static_cast<int>(f - static_cast<unsigned>(y) * n1);
        if (x < 1 || x > m - 1 || y < 1 || y > m - 1) {
            uOut[f] = zero2();
            continue;
        }
        const int qx = min(x / 3, mc - 1), qy = min(y / 3, mc - 1);
        const double w1y = relw(y - 3 * qy);
        const S wx = static_cast<S>(relw(x - 3 * qx));
        auto prolong = [&](const double2* src) {  // computeV (y, stored in the kernel's precision), then x
            const double2* c = src + qx + static_cast<long long>(n1c) * qy;
            const C v0 = to_c(lerpw(__ldg(c), __ldg(c + n1c), w1y), C{});
            const C v1 = to_c(lerpw(__ldg(c + 1), __ldg(c + 1 + n1c), w1y), C{});
            return lerpw(v0, v1, wx);
        };
        C scv = prolong(scTD);
        if (siTD && !(x % 3 == 0 && y % 3 == 0)) scv = sub(scv, prolong(siTD));
        uOut[f] = to_d(add(__ldg(vOld + f), scv));
    }
}

template <bool SMOOTH>
__global__ void __launch_bounds__(256) k_combine2(const Args a, double2* rc, const fast::ResArgs sa) {
    dev::griddep_wait();
    const int mc = a.g.mc, m = a.g.m, yc = a.g.yc;
    const unsigned n1c = a.n1c;
    const unsigned total = n1c * n1c;
    for (unsigned f = blockIdx.x * blockDim.x + threadIdx.x; f < total; f += gridDim.x * blockDim.x) {
        const int W1 = static_cast<int>(f / n1c), W0 = static_cast<int>(f - static_cast<unsigned>(W1) * n1c);
        if (W0 < 1 || W0 > mc - 1 || W1 < 1 || W1 > mc - 1) continue;
        const int by0 = (max(1, 3 * W1 - 2) - 1) / yc, by1 = (min(m - 1, 3 * W1 + 2) - 1) / yc;
        const int bx0 = (max(1, 3 * W0 - 2) - 1) / TX, bx1 = (min(m - 1, 3 * W0 + 2) - 1) / TX;
        double2 v[4];  // at most two strips / chunks per axis: loaded up front, added in (by, bx) order
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int by = by0 + (q >> 1), bx = bx0 + (q & 1);
            const int yi = W1 - (by * yc) / 3, xi = W0 - (1 + bx * TX) / 3;
            v[q] = (by <= by1 && bx <= bx1)
                       ? __ldcs(a.partial + ((static_cast<long long>(by) * a.g.sy + yi) * a.g.nbx + bx) * SXP + xi)
                       : zero2();
        }
        double2 acc = zero2();
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (by0 + (q >> 1) <= by1 && bx0 + (q & 1) <= bx1) acc = add(acc, v[q]);
        rc[f] = acc;
        if (SMOOTH) {  // level L-1 smoothing (k_smooth_coarse) on the value just formed (fused3::k_combine<true>)
            const dev::Lvl& cl = sa.lv;
            if (sa.bpx && cl.si) {
                cl.si[f] = cl.sinext[f];
                cl.sinext[f] = zero2();
            }
            if (cl.level < sa.ellMin) {
                cl.sc[f] = zero2();
                continue;
            }
            const bool cp = (W0 % 3 == 0) && (W1 % 3 == 0);
            const double2 smooth = mul(acc, sa.k.invDiag);
            cl.sc[f] = stage_sc(smooth, sa.k.wRaw, cp, sa.bpx, sa.hb);
            if (sa.bpx && cl.level > sa.ellMin && cp)
                sa.par.sinext[(W0 / 3) + sa.par.n1 * (W1 / 3)] = mul(sa.k.wRaw, smooth);
        }
    }
}

}  // namespace

Geometry geometry(int m, int mc, int smCount) {
    Geometry g{};
    g.m = m;
    g.mc = mc;
    const int inner = std::max(1, m - 1);
    g.nbx = (inner + TX - 1) / TX;
    int per = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_fused2<false, double>, TX, 0) != cudaSuccess || per < 1) per = 4;
    const int resident = 2 * per * std::max(1, smCount);  // two waves of strips
    const int want = std::max(1, (resident + g.nbx - 1) / g.nbx);
    g.yc = std::min(kMaxYc, std::max(3, ((inner + want - 1) / want + 2) / 3 * 3));  // cap: staged coarse rows
    g.nby = (inner + g.yc - 1) / g.yc;
    g.sy = g.yc / 3 + 2;
    return g;
}

size_t partial_count(const Geometry& g) { return static_cast<size_t>(g.nby) * g.sy * g.nbx * SXP; }

int blocks(const Geometry& g) { return g.nbx * g.nby; }

size_t smem_bytes(const Geometry& g, bool bpx, bool c64) {
    (void)g;
    const size_t rows = c64 ? static_cast<size_t>(kRing) * (2 * TX + 4) * sizeof(float2)   // v rows + b rows (from x0 - 1)
                            : static_cast<size_t>(kRing) * (2 * TX + 2) * sizeof(double2);
    return rows + static_cast<size_t>(bpx ? 8 : 4) * CXW * sizeof(double2);
}

void derive_u(const double2* vOld, const double2* scTD, const double2* siTD, unsigned n1, unsigned n1c, unsigned fa,
              unsigned fb, double2* uOut, bool c64, cudaStream_t s) {
    if (fb <= fa) return;
    const unsigned blocks = std::min<unsigned>((fb - fa + 255) / 256, 148u * 32u);
    if (c64)
        k_derive_u2<float><<<blocks, 256, 0, s>>>(reinterpret_cast<const float2*>(vOld), scTD, siTD, n1, n1c, fa, fb, uOut);
    else
        k_derive_u2<double><<<blocks, 256, 0, s>>>(vOld, scTD, siTD, n1, n1c, fa, fb, uOut);
}

template <bool BPX, class S>
static void launch_as(const Args& a, dim3 grid, size_t smem, cudaStream_t s) {
    // static + dynamic shared memory may pass 48 KB (BPX, long chunks); a per-device
    // attribute, so set on every launch (host-side call)
    cudaFuncSetAttribute(k_fused2<BPX, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    dev::launch_k(k_fused2<BPX, S>, grid, dim3(TX), smem, s, a);
}

void launch(const Args& a, cudaStream_t s) {
    dim3 grid(a.g.nbx, a.g.nby);
    const size_t smem = smem_bytes(a.g, a.bpx != 0, a.c64 != 0);
    if (a.c64) {
        if (a.bpx) launch_as<true, float>(a, grid, smem, s);
        else launch_as<false, float>(a, grid, smem, s);
    } else {
        if (a.bpx) launch_as<true, double>(a, grid, smem, s);
        else launch_as<false, double>(a, grid, smem, s);
    }
}

void combine(const Args& a, double2* rCoarse, cudaStream_t s, const fast::ResArgs* smooth) {
    const unsigned total = a.n1c * a.n1c;
    const unsigned nb = std::max(1u, std::min((total + 255) / 256, 4096u));
    if (smooth) dev::launch_k(k_combine2<true>, dim3(nb), dim3(256), 0, s, a, rCoarse, *smooth);
    else dev::launch_k(k_combine2<false>, dim3(nb), dim3(256), 0, s, a, rCoarse, fast::ResArgs{});
}

}  // namespace fused2
}  // namespace tmg
