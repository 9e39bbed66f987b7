// Fused fine pass for 3D (see fused3.cuh).

#include "fused3.cuh"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <type_traits>

namespace tmg {
namespace fused3 {

namespace {

// ---- complex arithmetic on double2 (complex128) and float2 (complex64) ----
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
template <class C> __device__ __forceinline__ C ld(const C* p) { return __ldg(p); }
// complex128 <-> the kernel's complex type
__device__ __forceinline__ double2 to_c(double2 v, double2) { return v; }
__device__ __forceinline__ float2 to_c(double2 v, float2) { return make_float2(static_cast<float>(v.x), static_cast<float>(v.y)); }
__device__ __forceinline__ double2 to_d(double2 v) { return v; }
__device__ __forceinline__ double2 to_d(float2 v) { return make_double2(v.x, v.y); }
template <class S> __device__ __forceinline__ S third(int num) {  // num / 3 in the kernel's precision
    return static_cast<S>(num == 1 ? (1.0 / 3.0) : num == 2 ? (2.0 / 3.0) : num == 3 ? 1.0 : 0.0);
}

template <class C>
__device__ __forceinline__ C stage_sc(C smooth, C w, bool cp, int bpx, int hb) {
    if (bpx) return cp ? zero<C>() : mul(w, smooth);
    if ((hb && cp) || (w.x == 0 && w.y == 0)) return zero<C>();
    return mul(w, smooth);
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "TMG_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra TMG_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// Kernel shape: R rows of points per thread (fused3.cuh).
template <int R>
struct Cfg {
    static constexpr int TYT = TY / R;                 // thread rows
    static constexpr int NT = TX * TYT;                // threads per block
    static constexpr int STAGES = R == 2 ? 3 : 4;      // ring depth (R = 2 stages carry a b tile too)
    static constexpr int MINB = R == 2 ? 4 : 3;        // blocks per SM
    static_assert(TY % R == 0, "tile height");
};

// Shared-memory carve-up (bytes; every TMA destination 128-byte aligned).
// C = the kernel's complex type (16 B complex128 or 8 B complex64).
template <class C, int R>
struct Smem {
    static constexpr int STAGES = Cfg<R>::STAGES;
    static constexpr int kPlane = (HX * HY * static_cast<int>(sizeof(C)) + 127) / 128 * 128;  // halo'd fine tile
    static constexpr unsigned kTileBytes = HX * HY * sizeof(C);
    static constexpr int kC = (CX * CY * 2 * 16 + 127) / 128 * 128;  // two complex128 coarse planes
    static constexpr unsigned kCBytes = CX * CY * 2 * sizeof(double2);
    static constexpr int kV = (HY * CX + 7) / 8 * 8;  // z- and y-interpolated coarse rows (elements of C)
    static constexpr int kP = (HX * HY + 7) / 8 * 8;  // corrected plane (elements of C)
    // R = 2: the b tile of the plane the step's residual is for (32 x TY, no halo), TMA'd with the stage
    // complex64: the b tile starts one column early (x0 - 1, even: the TMA box start is then 16-byte
    // aligned as for complex128) and is two columns wider; the kernel skips the leading column
    static constexpr int kBOff = sizeof(C) == 8 ? 1 : 0;
    static constexpr int kBW = TX + 2 * kBOff;  // b tile row length
    static constexpr int kBt = R == 2 ? (kBW * TY * static_cast<int>(sizeof(C)) + 127) / 128 * 128 : 0;
    static constexpr unsigned kBtBytes = R == 2 ? kBW * TY * sizeof(C) : 0;
    template <bool BPX>
    __host__ __device__ static constexpr int stage() { return kPlane + (BPX ? 2 : 1) * kC + kBt; }
    template <bool BPX>
    __host__ __device__ static constexpr size_t bytes() {
        return STAGES * stage<BPX>() + ((BPX ? 4 : 2) * kV + 2 * kP + TX * TY + TY * SX) * sizeof(C) +
               STAGES * sizeof(uint64_t);
    }
};

// One point per thread (the round-1 shape; the complex64 kernel).
template <bool BPX, class S>
__global__ void __launch_bounds__(Cfg<1>::NT, Cfg<1>::MINB)
    k_fused3_r1(const __grid_constant__ CUtensorMap mapU, const __grid_constant__ CUtensorMap mapC,
                const __grid_constant__ CUtensorMap mapI, const __grid_constant__ CUtensorMap mapB, const Args a) {
    using C = typename Cx<S>::T;
    using M = Smem<C, 1>;
    constexpr int NT = Cfg<1>::NT, STAGES = Cfg<1>::STAGES;
    (void)mapB;
    dev::griddep_wait();
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int SB = M::template stage<BPX>();                 // stage stride, bytes
    unsigned char* ring = smem;                                  // STAGES x {v tile, coarse sc[, si]}
    C* Vb = reinterpret_cast<C*>(smem + STAGES * SB);            // [2][kV] (+[2][kV] si)
    C* Pb = Vb + (BPX ? 4 : 2) * M::kV;                          // [2][kP] corrected planes
    C* tb = Pb + 2 * M::kP;                                      // [TY][TX] z-restricted columns
    C* rb = tb + NT;                                             // [TY][SX] x-restricted rows
    uint64_t* bar = reinterpret_cast<uint64_t*>(rb + TY * SX);
    auto tile = [&](int st) { return reinterpret_cast<const C*>(ring + st * SB); };
    auto coarse = [&](int st) { return reinterpret_cast<const double2*>(ring + st * SB + M::kPlane); };

    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
    const int m = a.g.m, mc = a.g.mc;
    const int bzg = blockIdx.z + a.chunkBase;  // global z-chunk (slabs launch a chunk range)
    const int x0 = 1 + blockIdx.x * TX, y0 = 1 + blockIdx.y * TY, z0 = 1 + bzg * a.g.zc;
    const int xe = min(x0 + TX, m), ye = min(y0 + TY, m), z1 = min(z0 + a.g.zc, m);
    const int nplanes = z1 - z0 + 2;
    const long long sy = a.n1, sz = static_cast<long long>(a.n1) * a.n1;
    const int cx0 = (x0 - 1) / 3, cy0 = (y0 - 1) / 3;
    constexpr unsigned stageBytes = M::kTileBytes + (BPX ? 2 : 1) * M::kCBytes;
    constexpr int xScale = sizeof(C) / sizeof(S);  // tensor-map x coordinates count scalars

    auto issue = [&](int stage, int zz) {
        unsigned char* st = ring + stage * SB;
        const int cz = min(zz / 3, mc - 1);
        mbar_expect_tx(&bar[stage], stageBytes);
        tma_load3(st, &mapU, xScale * (x0 - 1), y0 - 1, zz - a.tmaZ0, &bar[stage]);
        tma_load3(st + M::kPlane, &mapC, 2 * cx0, cy0, cz - a.tmaZ0c, &bar[stage]);
        if (BPX) tma_load3(st + M::kPlane + M::kC, &mapI, 2 * cx0, cy0, cz - a.tmaZ0c, &bar[stage]);
    };

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0)
        for (int s = 0; s < STAGES && s < nplanes; ++s) issue(s, z0 - 1 + s);

    // ---- per-thread constants ----
    // Phase B: every thread corrects its own column's point; threads [0, RING)
    // also one halo-ring point, threads [RING, RING + HY*CX) one row of the
    // z/y-interpolated coarse plane of the next fine plane.
    constexpr int RING = 2 * HX + 2 * TY;
    const int x = x0 + tx, y = y0 + ty;
    const bool owned = x < xe && y < ye;  // == own point inside [1, m-1]^2
    const bool cpxy = (x % 3 == 0) && (y % 3 == 0);
    const int po = (ty + 1) * HX + (tx + 1);
    int vo;
    S wxo;
    {
        const int qx = min(x / 3, mc - 1);
        vo = (ty + 1) * CX + (qx - cx0);
        wxo = third<S>(x - 3 * qx);
    }
    // coarse-row tasks take 16 lanes per row from thread VT0 on (bank-conflict-free: see k_fused3_r2)
    constexpr int VT0 = (RING + 31) / 32 * 32;
    static_assert(CX <= 16 && VT0 + HY * 16 <= NT, "phase-B task map");
    const int vs = tid - VT0;
    const int task = tid < RING ? 1 : ((vs >= 0 && (vs & 15) < CX && (vs >> 4) < HY) ? 2 : 0);
    int pr = 0, vr = 0;
    S wxr = 0;
    bool pinr = false, cpr = false;
    int vcOff = 0;
    double w1y = 0.0;
    const int vt = (vs >> 4) * CX + (vs & 15);
    if (task == 1) {
        const int k = tid;
        int lx, ly;
        if (k < HX) { lx = k; ly = 0; }
        else if (k < 2 * HX) { lx = k - HX; ly = HY - 1; }
        else { lx = ((k - 2 * HX) & 1) ? HX - 1 : 0; ly = 1 + ((k - 2 * HX) >> 1); }  // halo columns interleaved
        const int gx = x0 - 1 + lx, gy = y0 - 1 + ly;
        pinr = gx >= 1 && gx <= m - 1 && gy >= 1 && gy <= m - 1;
        const int qx = min(max(gx, 0) / 3, mc - 1);
        pr = ly * HX + lx;
        vr = ly * CX + (qx - cx0);
        wxr = third<S>(gx - 3 * qx);
        cpr = (gx % 3 == 0) && (gy % 3 == 0);
    } else if (task == 2) {
        const int ly = vs >> 4, ci = vs & 15;
        const int gy = y0 - 1 + ly;
        const int qy = min(max(gy, 0) / 3, mc - 1);
        vcOff = (qy - cy0) * CX + ci;
        w1y = third<double>(gy - 3 * qy);
    }
    // the coarse (complex128) correction interpolated in y and z, stored in the kernel's precision
    // w1z: the z weight of plane zz between its two coarse planes (the caller knows zz % 3)
    auto computeV = [&](int stage, double w1z, int vb) {
        const double2* Cc = coarse(stage);
        const double2 a0 = lerpw(Cc[vcOff], Cc[vcOff + CX], w1y);
        const double2 a1 = lerpw(Cc[vcOff + CX * CY], Cc[vcOff + CX * CY + CX], w1y);
        Vb[vb * M::kV + vt] = to_c(lerpw(a0, a1, w1z), C{});
        if (BPX) {
            const double2* I = Cc + M::kC / 16;
            const double2 b0 = lerpw(I[vcOff], I[vcOff + CX], w1y);
            const double2 b1 = lerpw(I[vcOff + CX * CY], I[vcOff + CX * CY + CX], w1y);
            Vb[(2 + vb) * M::kV + vt] = to_c(lerpw(b0, b1, w1z), C{});
        }
    };

    double nmax = 0.0, nsum = 0.0;
    C accLo = zero<C>(), accHi = zero<C>();

    // restriction slots of this tile (xy); z handled by the column accumulators
    const int Xa = x0 / 3, Xb = (xe + 1) / 3, Ya = y0 / 3, Yb = (ye + 1) / 3;
    const int nsx = Xb - Xa + 1, nsy = Yb - Ya + 1;
    // partial layout [bz][zi][by][bx][SY][SX]: one chunk's zi = 0 slots are contiguous
    const long long tileXY = blockIdx.x + static_cast<long long>(a.g.nbx) * blockIdx.y;
    const long long tilesXY = static_cast<long long>(a.g.nbx) * a.g.nby;
    double2* part = a.partial + (static_cast<long long>(bzg) * a.g.sz * tilesXY + tileXY) * (SY * SX);
    const long long zStride = tilesXY * (SY * SX);
    const int zBase = (z0 - 1) / 3;
    int zLow = zBase;
    const bool slotThread = tid < nsx * nsy;
    const int sxi = slotThread ? tid % nsx : 0, syi = slotThread ? tid / nsx : 0;
    auto wk = [](int k) { return static_cast<S>(k == 0 ? 1.0 : (k == 1 || k == -1) ? (2.0 / 3.0) : (1.0 / 3.0)); };
    auto flushSlots = [&](int zi) {
        __syncthreads();
        if (slotThread) {
            const int X = Xa + sxi, Y = Ya + syi;
            C acc = zero<C>();
#pragma unroll
            for (int ky = -2; ky <= 2; ++ky) {
                const int fy = 3 * Y + ky;
                if (fy < y0 || fy >= ye) continue;
                C row = zero<C>();
#pragma unroll
                for (int kx = -2; kx <= 2; ++kx) {
                    const int fx = 3 * X + kx;
                    if (fx < x0 || fx >= xe) continue;
                    row = axpy(wk(kx), tb[(fy - y0) * TX + (fx - x0)], row);
                }
                acc = axpy(wk(ky), row, acc);
            }
            part[zi * zStride + syi * SX + sxi] = to_d(acc);
        }
    };

    // Pipelined xy reduction of a finished coarse plane: the step after tb is
    // written reduces rows (stage 1, into rb), the next one columns (stage 2,
    // into the partials); both ride on the steps' own barriers.  Same
    // arithmetic as flushSlots.  Task i runs on thread NT-1-i, away from the
    // threads that carry phase-B halo / coarse-row work.
    const int ti = NT - 1 - tid;
    const int s1y = nsx > 0 ? ti / nsx : 0, s1x = ti - s1y * nsx;  // stage-1 task (row, slot) / stage-2 (sy, sx)
    auto stage1 = [&]() {
        if (ti < TY * nsx) {
            const int fyl = s1y, sx = s1x;
            if (y0 + fyl < ye) {
                const int X = Xa + sx;
                C row = zero<C>();
#pragma unroll
                for (int kx = -2; kx <= 2; ++kx) {
                    const int fx = 3 * X + kx;
                    if (fx < x0 || fx >= xe) continue;
                    row = axpy(wk(kx), tb[fyl * TX + (fx - x0)], row);
                }
                rb[fyl * SX + sx] = row;
            }
        }
    };
    auto stage2 = [&](int zi) {
        if (ti < nsx * nsy) {
            const int sx = s1x, syy = s1y;
            const int Y = Ya + syy;
            C acc = zero<C>();
#pragma unroll
            for (int ky = -2; ky <= 2; ++ky) {
                const int fy = 3 * Y + ky;
                if (fy < y0 || fy >= ye) continue;
                acc = axpy(wk(ky), rb[(fy - y0) * SX + sx], acc);
            }
            part[zi * zStride + syy * SX + sx] = to_d(acc);
        }
    };
    bool pend1 = false, pend2 = false;
    int zi1 = 0, zi2 = 0;

    const long long colBase = x + y * sy;
    const C* bPtr = static_cast<const C*>(a.b) + colBase + static_cast<long long>(z0) * sz;
    C* uPtr = static_cast<C*>(a.uNew) + colBase + static_cast<long long>(z0) * sz;
    C* sPtr = static_cast<C*>(a.scNew) + colBase + static_cast<long long>(z0) * sz;
    double2* siPtr = a.sinextC + (x / 3) + a.n1c * (static_cast<long long>(y / 3) + static_cast<long long>(a.n1c) * ((z0 + 2) / 3));
    C bq0 = (owned && z0 < z1) ? ld(bPtr) : zero<C>();
    const bool zeroSc = a.level < a.ellMin;
    const bool injectOK = BPX && a.level > a.ellMin && cpxy && owned;
    const C k0 = to_c(a.k.c[0], C{}), k1 = to_c(a.k.c[1], C{}), k2 = to_c(a.k.c[2], C{}), k3 = to_c(a.k.c[3], C{});
    const C invDiag = to_c(a.k.invDiag, C{}), wRaw = to_c(a.k.wRaw, C{});

    mbar_wait(&bar[0], 0);
    if (task == 2) {
        const int zf = z0 - 1, cz = min(zf / 3, mc - 1);
        computeV(0, third<double>(zf - 3 * cz), 0);
    }
    __syncthreads();

    // running stencil accumulators: Aprev = H u at plane p-1 minus its plane-p terms, Acur = plane p's so far
    C Aprev = zero<C>(), Acur = zero<C>();
    int stage = 0;
    unsigned parity = 0;

    auto step = [&](int it, auto U3) {
        constexpr int u = decltype(U3)::value;  // zz % 3 == u
        const int zz = z0 - 1 + it;
        const bool hasNext = it + 1 < nplanes;
        const int nstage = stage + 1 == STAGES ? 0 : stage + 1;
        const unsigned nparity = stage + 1 == STAGES ? parity ^ 1u : parity;
        mbar_wait(&bar[stage], parity);
        if (hasNext) mbar_wait(&bar[nstage], nparity);
        const bool zin = zz >= 1 && zz <= m - 1;
        const C* Ut = tile(stage);  // fine state v = u + sc of plane zz
        const C* V = Vb + (it & 1) * M::kV;
        C* P = Pb + (it & 1) * M::kP;
        // ---- phase B ----
        C cOwn;
        {
            C scv = lerpw(V[vo], V[vo + 1], wxo);
            if (BPX && !(cpxy && u == 0)) {
                const C* Vi = Vb + (2 + (it & 1)) * M::kV;
                scv = sub(scv, lerpw(Vi[vo], Vi[vo + 1], wxo));
            }
            cOwn = (zin && owned) ? add(Ut[po], scv) : zero<C>();
            P[po] = cOwn;
        }
        if (task == 1) {
            C scv = lerpw(V[vr], V[vr + 1], wxr);
            if (BPX && !(cpr && u == 0)) {
                const C* Vi = Vb + (2 + (it & 1)) * M::kV;
                scv = sub(scv, lerpw(Vi[vr], Vi[vr + 1], wxr));
            }
            P[pr] = (zin && pinr) ? add(Ut[pr], scv) : zero<C>();
        } else if (task == 2 && hasNext) {
            // plane zz + 1 has residue (u + 1) % 3; the top lattice plane m = 3 mc takes weight 1
            computeV(nstage, zz + 1 == m ? 1.0 : third<double>((u + 1) % 3), (it + 1) & 1);
        }
        __syncthreads();
        if (tid == 0 && it + STAGES < nplanes) issue(stage, zz + STAGES);
        stage = nstage;
        parity = nparity;
        // ---- phase C ----
        if (u == 1 && pend1) {
            stage1();
            pend1 = false;
            pend2 = true;
            zi2 = zi1;
        } else if (u == 2 && pend2) {
            stage2(zi2);
            pend2 = false;
        }
        const C* c = P + po;
        const C E = add(add(c[-1], c[1]), add(c[-HX], c[HX]));
        const C K = add(add(c[-1 - HX], c[1 - HX]), add(c[-1 + HX], c[1 + HX]));
        C T = mul(k1, cOwn);
        T = mac(T, k2, E);
        T = mac(T, k3, K);
        C Uo = mul(k0, cOwn);
        Uo = mac(Uo, k1, E);
        Uo = mac(Uo, k2, K);
        if (it >= 2) {
            constexpr int kz = (u + 2) % 3;  // plane z = zz - 1
            const C hu = add(Aprev, T);
            const C r = owned ? sub(bq0, hu) : zero<C>();
            bPtr += sz;
            if (owned && zz < z1) bq0 = ld(bPtr);
            const S m2 = fma(r.x, r.x, r.y * r.y);
            nmax = static_cast<double>(m2) > nmax ? static_cast<double>(m2) : nmax;  // == fmax (a NaN is ignored)
            nsum += static_cast<double>(m2);
            const C smooth = mul(r, invDiag);
            const C scn = zeroSc ? zero<C>() : stage_sc(smooth, wRaw, cpxy && kz == 0, BPX ? 1 : 0, a.hb);
            if (owned) {
                if (a.writeSc) *sPtr = scn;
                // next cycle's state v = u + sc of plane zz - 1 (its corrected u is
                // still in the other P buffer: rewritten only in the next phase B)
                *uPtr = add(Pb[((it + 1) & 1) * M::kP + po], scn);
            }
            sPtr += sz;
            uPtr += sz;
            if (BPX && kz == 0 && injectOK) {
                *siPtr = to_d(mul(wRaw, smooth));
                siPtr += static_cast<long long>(a.n1c) * a.n1c;
            }
            if (kz == 0) {
                accLo = add(accLo, r);
            } else if (kz == 1) {
                accLo = axpy(static_cast<S>(2.0 / 3.0), r, accLo);
                accHi = axpy(static_cast<S>(1.0 / 3.0), r, accHi);
            } else {
                accLo = axpy(static_cast<S>(1.0 / 3.0), r, accLo);
                accHi = axpy(static_cast<S>(2.0 / 3.0), r, accHi);
                tb[ty * TX + tx] = accLo;
                accLo = accHi;
                accHi = zero<C>();
                pend1 = true;
                zi1 = zLow - zBase;
                ++zLow;
            }
        }
        Aprev = add(Acur, Uo);
        Acur = T;
    };
    using U0 = std::integral_constant<int, 0>;
    using U1 = std::integral_constant<int, 1>;
    using U2 = std::integral_constant<int, 2>;
    // zz = z0 - 1 + it and z0 = 1 (mod 3): zz % 3 == it % 3
    for (int it = 0; it < nplanes; it += 3) {
        step(it, U0{});
        if (it + 1 >= nplanes) break;
        step(it + 1, U1{});
        if (it + 2 >= nplanes) break;
        step(it + 2, U2{});
    }
    __syncthreads();
    if (pend1) {  // drain the pipelined reduction
        stage1();
        __syncthreads();
        stage2(zi1);
    } else if (pend2) {
        stage2(zi2);
    }
    __syncthreads();
    tb[ty * TX + tx] = accLo;
    flushSlots(zLow - zBase);
    __syncthreads();
    tb[ty * TX + tx] = accHi;
    flushSlots(zLow + 1 - zBase);
    dev::block_norms(nmax, nsum, a.norms);
}

// Two rows per thread (rows y, y + 1 of the 32 x TY tile; the complex128 kernel).
// Same pass as the one-row kernel with twice the points per thread: the
// in-plane sums of the two rows share their x-pair sums s_j = c(x-1) + c(x+1)
// (rows y-1 .. y+2: 10 shared-memory loads for two points instead of 16), the
// halo ring is 100 / 512 points instead of 84 / 256, and every warp carries
// two independent points (more latency hiding per issue slot).
template <bool BPX, class S>
__global__ void __launch_bounds__(Cfg<2>::NT, Cfg<2>::MINB)
    k_fused3_r2(const __grid_constant__ CUtensorMap mapU, const __grid_constant__ CUtensorMap mapC,
                const __grid_constant__ CUtensorMap mapI, const __grid_constant__ CUtensorMap mapB, const Args a) {
    using C = typename Cx<S>::T;
    using M = Smem<C, 2>;
    constexpr int NT = Cfg<2>::NT, STAGES = Cfg<2>::STAGES, ROWS = 2;
    dev::griddep_wait();
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int SB = M::template stage<BPX>();
    unsigned char* ring = smem;
    C* Vb = reinterpret_cast<C*>(smem + STAGES * SB);
    C* Pb = Vb + (BPX ? 4 : 2) * M::kV;
    C* tb = Pb + 2 * M::kP;                                      // [TY][TX] z-restricted columns
    C* rb = tb + TX * TY;                                        // [TY][SX] x-restricted rows
    uint64_t* bar = reinterpret_cast<uint64_t*>(rb + TY * SX);
    auto tile = [&](int st) { return reinterpret_cast<const C*>(ring + st * SB); };
    auto coarse = [&](int st) { return reinterpret_cast<const double2*>(ring + st * SB + M::kPlane); };

    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
    const int m = a.g.m, mc = a.g.mc;
    const int bzg = blockIdx.z + a.chunkBase;
    const int x0 = 1 + blockIdx.x * TX, y0 = 1 + blockIdx.y * TY, z0 = 1 + bzg * a.g.zc;
    const int xe = min(x0 + TX, m), ye = min(y0 + TY, m), z1 = min(z0 + a.g.zc, m);
    const int nplanes = z1 - z0 + 2;
    const long long sy = a.n1, sz = static_cast<long long>(a.n1) * a.n1;
    const int cx0 = (x0 - 1) / 3, cy0 = (y0 - 1) / 3;
    constexpr unsigned stageBytes = M::kTileBytes + (BPX ? 2 : 1) * M::kCBytes + M::kBtBytes;
    constexpr int xScale = sizeof(C) / sizeof(S);
    constexpr int kBtOff = M::kPlane + (BPX ? 2 : 1) * M::kC;

    // stage of plane zz: the halo'd v tile, the coarse planes, and b of plane zz - 1
    // (the plane this step's residual is for; out-of-range planes land as zeros)
    auto issue = [&](int stage, int zz) {
        unsigned char* st = ring + stage * SB;
        const int cz = min(zz / 3, mc - 1);
        mbar_expect_tx(&bar[stage], stageBytes);
        tma_load3(st, &mapU, xScale * (x0 - 1), y0 - 1, zz - a.tmaZ0, &bar[stage]);
        tma_load3(st + M::kPlane, &mapC, 2 * cx0, cy0, cz - a.tmaZ0c, &bar[stage]);
        if (BPX) tma_load3(st + M::kPlane + M::kC, &mapI, 2 * cx0, cy0, cz - a.tmaZ0c, &bar[stage]);
        tma_load3(st + kBtOff, &mapB, xScale * (x0 - M::kBOff), y0, zz - 1 - a.tmaZ0, &bar[stage]);
    };

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0)
        for (int s = 0; s < STAGES && s < nplanes; ++s) issue(s, z0 - 1 + s);

    // ---- per-thread constants ----
    // Phase B tasks besides the own two points: the HY x CX entries of the
    // z/y-interpolated coarse plane and the NRING halo-ring points (map below).
    constexpr int NRING = 2 * HX + 2 * TY;
    const int x = x0 + tx;
    const int yr0 = y0 + ROWS * ty;  // the thread's rows yr0, yr0 + 1
    bool owned[2], cpxy[2];
    // row r's corrected-plane / coarse-row slots: po + r * HX, vo + r * CX
    const int po = (ROWS * ty + 1) * HX + (tx + 1);
    int vo;
    S wxo;
    {
        const int qx = min(x / 3, mc - 1);
        wxo = third<S>(x - 3 * qx);
        vo = (ROWS * ty + 1) * CX + (qx - cx0);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int y = yr0 + r;
            owned[r] = x < xe && y < ye;
            cpxy[r] = (x % 3 == 0) && (y % 3 == 0);
        }
    }
    // Bank-conflict-free task map: coarse-row tasks take 16 lanes per row (a
    // quarter warp never straddles two rows of the same coarse row, whose
    // elements 8 apart share banks), first the rows [0, NT / 16) on every thread,
    // the rest on the last warp; ring points on threads [0, NRING), the two halo
    // columns interleaved (left / right of a row are 33 elements apart: distinct
    // banks, while the rows of one column are 34 apart: 4 rows wrap the banks).
    static_assert(CX <= 16 && HY * 16 <= NT + 32 && NRING <= NT, "phase-B task map");
    const int vly = tid >> 4, vci = tid & 15;
    const int v2 = tid - (NT - 32);                          // second pass: rows NT / 16 .. on the last warp
    const int vly2 = (NT + v2) >> 4, vci2 = v2 & 15;
    const int rk = tid < NRING ? tid : -1;
    const int vk2 = (v2 >= 0 && vly2 < HY && vci2 < CX) ? vly2 * CX + vci2 : -1;
    int pr = 0, vr = 0;
    S wxr = 0;
    bool pinr = false, cpr = false;
    if (rk >= 0) {
        int lx, ly;
        if (rk < HX) { lx = rk; ly = 0; }
        else if (rk < 2 * HX) { lx = rk - HX; ly = HY - 1; }
        else { lx = ((rk - 2 * HX) & 1) ? HX - 1 : 0; ly = 1 + ((rk - 2 * HX) >> 1); }
        const int gx = x0 - 1 + lx, gy = y0 - 1 + ly;
        pinr = gx >= 1 && gx <= m - 1 && gy >= 1 && gy <= m - 1;
        const int qx = min(max(gx, 0) / 3, mc - 1);
        pr = ly * HX + lx;
        vr = ly * CX + (qx - cx0);
        wxr = third<S>(gx - 3 * qx);
        cpr = (gx % 3 == 0) && (gy % 3 == 0);
    }
    const bool vtask = vci < CX && vly < HY;
    // coarse-row task k: offset into the coarse tile and the y weight
    auto vparams = [&](int k, int& off, double& w) {
        const int ly = k / CX, ci = k % CX;
        const int gy = y0 - 1 + ly;
        const int qy = min(max(gy, 0) / 3, mc - 1);
        off = (qy - cy0) * CX + ci;
        w = third<double>(gy - 3 * qy);
    };
    int vcOff = 0;
    double w1y = 0.0;
    const int vslot = vly * CX + vci;
    if (vtask) vparams(vslot, vcOff, w1y);
    // w1z: the z weight of plane zz between its two coarse planes (the caller knows zz % 3)
    auto computeV = [&](int stage, double w1z, int vb) {
        const double2* Cc = coarse(stage);
        auto one = [&](int o, double wy, int slot) {
            const double2 a0 = lerpw(Cc[o], Cc[o + CX], wy);
            const double2 a1 = lerpw(Cc[o + CX * CY], Cc[o + CX * CY + CX], wy);
            Vb[vb * M::kV + slot] = to_c(lerpw(a0, a1, w1z), C{});
            if (BPX) {
                const double2* I = Cc + M::kC / 16;
                const double2 b0 = lerpw(I[o], I[o + CX], wy);
                const double2 b1 = lerpw(I[o + CX * CY], I[o + CX * CY + CX], wy);
                Vb[(2 + vb) * M::kV + slot] = to_c(lerpw(b0, b1, w1z), C{});
            }
        };
        if (vtask) one(vcOff, w1y, vslot);
        if (vk2 >= 0) {  // the few threads with a second coarse-row task: parameters on the fly
            int o2;
            double wy2;
            vparams(vk2, o2, wy2);
            one(o2, wy2, vk2);
        }
    };

    double nmax = 0.0, nsum = 0.0;
    C accLo[2] = {zero<C>(), zero<C>()}, accHi[2] = {zero<C>(), zero<C>()};

    const int Xa = x0 / 3, Xb = (xe + 1) / 3, Ya = y0 / 3, Yb = (ye + 1) / 3;
    const int nsx = Xb - Xa + 1, nsy = Yb - Ya + 1;
    const long long tileXY = blockIdx.x + static_cast<long long>(a.g.nbx) * blockIdx.y;
    const long long tilesXY = static_cast<long long>(a.g.nbx) * a.g.nby;
    double2* part = a.partial + (static_cast<long long>(bzg) * a.g.sz * tilesXY + tileXY) * (SY * SX);
    const long long zStride = tilesXY * (SY * SX);
    const int zBase = (z0 - 1) / 3;
    int zLow = zBase;
    const bool slotThread = tid < nsx * nsy;
    const int sxi = slotThread ? tid % nsx : 0, syi = slotThread ? tid / nsx : 0;
    auto wk = [](int k) { return static_cast<S>(k == 0 ? 1.0 : (k == 1 || k == -1) ? (2.0 / 3.0) : (1.0 / 3.0)); };
    auto flushSlots = [&](int zi) {
        __syncthreads();
        if (slotThread) {
            const int X = Xa + sxi, Y = Ya + syi;
            C acc = zero<C>();
#pragma unroll
            for (int ky = -2; ky <= 2; ++ky) {
                const int fy = 3 * Y + ky;
                if (fy < y0 || fy >= ye) continue;
                C row = zero<C>();
#pragma unroll
                for (int kx = -2; kx <= 2; ++kx) {
                    const int fx = 3 * X + kx;
                    if (fx < x0 || fx >= xe) continue;
                    row = axpy(wk(kx), tb[(fy - y0) * TX + (fx - x0)], row);
                }
                acc = axpy(wk(ky), row, acc);
            }
            part[zi * zStride + syi * SX + sxi] = to_d(acc);
        }
    };
    const int ti = NT - 1 - tid;
    const int s1y = ti / nsx, s1x = ti - s1y * nsx;
    auto stage1 = [&]() {
        if (ti < TY * nsx && y0 + s1y < ye) {
            const int X = Xa + s1x;
            C row = zero<C>();
#pragma unroll
            for (int kx = -2; kx <= 2; ++kx) {
                const int fx = 3 * X + kx;
                if (fx < x0 || fx >= xe) continue;
                row = axpy(wk(kx), tb[s1y * TX + (fx - x0)], row);
            }
            rb[s1y * SX + s1x] = row;
        }
    };
    auto stage2 = [&](int zi) {
        if (ti < nsx * nsy) {
            const int Y = Ya + s1y;
            C acc = zero<C>();
#pragma unroll
            for (int ky = -2; ky <= 2; ++ky) {
                const int fy = 3 * Y + ky;
                if (fy < y0 || fy >= ye) continue;
                acc = axpy(wk(ky), rb[(fy - y0) * SX + s1x], acc);
            }
            part[zi * zStride + s1y * SX + s1x] = to_d(acc);
        }
    };
    bool pend1 = false, pend2 = false;
    int zi1 = 0, zi2 = 0;

    const long long colBase = x + static_cast<long long>(yr0) * sy;  // row 0; row 1 is + sy
    C* uPtr = static_cast<C*>(a.uNew) + colBase + static_cast<long long>(z0) * sz;
    C* sPtr = static_cast<C*>(a.scNew) + colBase + static_cast<long long>(z0) * sz;
    C bq[2];  // b of the step's residual plane, from the stage's b tile
    const bool zeroSc = a.level < a.ellMin;
    const C k0 = to_c(a.k.c[0], C{}), k1 = to_c(a.k.c[1], C{}), k2 = to_c(a.k.c[2], C{}), k3 = to_c(a.k.c[3], C{});
    const C invDiag = to_c(a.k.invDiag, C{}), wRaw = to_c(a.k.wRaw, C{});

    mbar_wait(&bar[0], 0);
    {
        const int zf = z0 - 1, cz = min(zf / 3, mc - 1);
        computeV(0, third<double>(zf - 3 * cz), 0);
    }
    __syncthreads();

    C Aprev[2] = {zero<C>(), zero<C>()}, Acur[2] = {zero<C>(), zero<C>()};
    int stage = 0;
    unsigned parity = 0;

    auto step = [&](int it, auto U3) {
        constexpr int u = decltype(U3)::value;  // zz % 3 == u
        const int zz = z0 - 1 + it;
        const bool hasNext = it + 1 < nplanes;
        const int nstage = stage + 1 == STAGES ? 0 : stage + 1;
        const unsigned nparity = stage + 1 == STAGES ? parity ^ 1u : parity;
        mbar_wait(&bar[stage], parity);
        if (hasNext) mbar_wait(&bar[nstage], nparity);
        const bool zin = zz >= 1 && zz <= m - 1;
        const C* Ut = tile(stage);
        const C* V = Vb + (it & 1) * M::kV;
        C* P = Pb + (it & 1) * M::kP;
        {  // b of plane zz - 1, read before the stage is refilled
            const C* Bt = reinterpret_cast<const C*>(ring + stage * SB + kBtOff);
#pragma unroll
            for (int r = 0; r < 2; ++r) bq[r] = Bt[(ROWS * ty + r) * M::kBW + tx + M::kBOff];
        }
        // ---- phase B ----
        C cOwn[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            C scv = lerpw(V[(vo + r * CX)], V[(vo + r * CX) + 1], wxo);
            if (BPX && !(cpxy[r] && u == 0)) {
                const C* Vi = Vb + (2 + (it & 1)) * M::kV;
                scv = sub(scv, lerpw(Vi[(vo + r * CX)], Vi[(vo + r * CX) + 1], wxo));
            }
            cOwn[r] = (zin && owned[r]) ? add(Ut[(po + r * HX)], scv) : zero<C>();
            P[(po + r * HX)] = cOwn[r];
        }
        if (rk >= 0) {
            C scv = lerpw(V[vr], V[vr + 1], wxr);
            if (BPX && !(cpr && u == 0)) {
                const C* Vi = Vb + (2 + (it & 1)) * M::kV;
                scv = sub(scv, lerpw(Vi[vr], Vi[vr + 1], wxr));
            }
            P[pr] = (zin && pinr) ? add(Ut[pr], scv) : zero<C>();
        }
        // plane zz + 1 has residue (u + 1) % 3; the top lattice plane m = 3 mc sits on the
        // last coarse plane of the clamped pair (weight 1)
        if (hasNext) computeV(nstage, zz + 1 == m ? 1.0 : third<double>((u + 1) % 3), (it + 1) & 1);
        __syncthreads();
        if (tid == 0 && it + STAGES < nplanes) issue(stage, zz + STAGES);
        stage = nstage;
        parity = nparity;
        // keep the ring slot a run-time value: with 3 stages and the 3-way unrolled
        // plane loop the compiler would otherwise specialise every slot address
        // per step (+ 70 B of register spills)
        asm volatile("" : "+r"(stage));
        // ---- phase C ----
        if (u == 1 && pend1) {
            stage1();
            pend1 = false;
            pend2 = true;
            zi2 = zi1;
        } else if (u == 2 && pend2) {
            stage2(zi2);
            pend2 = false;
        }
        // rows y-1 .. y+2 around the thread's two points: x-pair sums s_j, centres
        const C* c = P + ROWS * ty * HX + tx;  // row y-1, column x-1
        C sj[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) sj[j] = add(c[j * HX], c[j * HX + 2]);
        const C mTop = c[1], mBot = c[3 * HX + 1];
        const C E[2] = {add(sj[1], add(mTop, cOwn[1])), add(sj[2], add(cOwn[0], mBot))};
        const C K[2] = {add(sj[0], sj[2]), add(sj[1], sj[3])};
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            C T = mul(k1, cOwn[r]);
            T = mac(T, k2, E[r]);
            T = mac(T, k3, K[r]);
            C Uo = mul(k0, cOwn[r]);
            Uo = mac(Uo, k1, E[r]);
            Uo = mac(Uo, k2, K[r]);
            if (it >= 2) {
                constexpr int kz = (u + 2) % 3;  // plane z = zz - 1
                const C hu = add(Aprev[r], T);
                const C res = owned[r] ? sub(bq[r], hu) : zero<C>();
                const S m2 = fma(res.x, res.x, res.y * res.y);
                nmax = static_cast<double>(m2) > nmax ? static_cast<double>(m2) : nmax;  // == fmax (a NaN is ignored)
                nsum += static_cast<double>(m2);
                const C smooth = mul(res, invDiag);
                const C scn = zeroSc ? zero<C>() : stage_sc(smooth, wRaw, cpxy[r] && kz == 0, BPX ? 1 : 0, a.hb);
                if (owned[r]) {
                    if (a.writeSc) sPtr[r * sy] = scn;
                    uPtr[r * sy] = add(Pb[((it + 1) & 1) * M::kP + (po + r * HX)], scn);
                }
                if (BPX && kz == 0 && a.level > a.ellMin && cpxy[r] && owned[r])
                    a.sinextC[(x / 3) + a.n1c * (static_cast<long long>((yr0 + r) / 3) +
                                                 static_cast<long long>(a.n1c) * ((zz - 1) / 3))] =
                        to_d(mul(wRaw, smooth));
                if (kz == 0) {
                    accLo[r] = add(accLo[r], res);
                } else if (kz == 1) {
                    accLo[r] = axpy(static_cast<S>(2.0 / 3.0), res, accLo[r]);
                    accHi[r] = axpy(static_cast<S>(1.0 / 3.0), res, accHi[r]);
                } else {
                    accLo[r] = axpy(static_cast<S>(1.0 / 3.0), res, accLo[r]);
                    accHi[r] = axpy(static_cast<S>(2.0 / 3.0), res, accHi[r]);
                    tb[(ROWS * ty + r) * TX + tx] = accLo[r];
                    accLo[r] = accHi[r];
                    accHi[r] = zero<C>();
                }
            }
            Aprev[r] = add(Acur[r], Uo);
            Acur[r] = T;
        }
        if (it >= 2) {
            sPtr += sz;
            uPtr += sz;
            if ((u + 2) % 3 == 2) {
                pend1 = true;
                zi1 = zLow - zBase;
                ++zLow;
            }
        }
    };
    using U0 = std::integral_constant<int, 0>;
    using U1 = std::integral_constant<int, 1>;
    using U2 = std::integral_constant<int, 2>;
    for (int it = 0; it < nplanes; it += 3) {
        step(it, U0{});
        if (it + 1 >= nplanes) break;
        step(it + 1, U1{});
        if (it + 2 >= nplanes) break;
        step(it + 2, U2{});
    }
    __syncthreads();
    if (pend1) {
        stage1();
        __syncthreads();
        stage2(zi1);
    } else if (pend2) {
        stage2(zi2);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 2; ++r) tb[(ROWS * ty + r) * TX + tx] = accLo[r];
    flushSlots(zLow - zBase);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 2; ++r) tb[(ROWS * ty + r) * TX + tx] = accHi[r];
    flushSlots(zLow + 1 - zBase);
    dev::block_norms(nmax, nsum, a.norms);
}

// derive_u (fused3.cuh): phase B of k_fused3 for one point, from global memory
template <class S>
__global__ void __launch_bounds__(256) k_derive_u(const typename Cx<S>::T* __restrict__ vOld,
                                                  const double2* __restrict__ scTD, const double2* __restrict__ siTD,
                                                  unsigned n1, unsigned n1c, unsigned fa, unsigned fb,
                                                  double2* __restrict__ uOut) {
    using C = typename Cx<S>::T;
    const int m = static_cast<int>(n1) - 1, mc = static_cast<int>(n1c) - 1;
    for (unsigned f = fa + blockIdx.x * blockDim.x + threadIdx.x; f < fb; f += gridDim.x * blockDim.x) {
        const unsigned fr = f / n1;
        const int x = static_cast<int>(f - fr * n1), y = static_cast<int>(fr % n1), z = static_cast<int>(fr / n1);
        if (x < 1 || x > m - 1 || y < 1 || y > m - 1 || z < 1 || z > m - 1) {
            uOut[f] = zero2();
            continue;
        }
        const int qx = min(x / 3, mc - 1), qy = min(y / 3, mc - 1), qz = min(z / 3, mc - 1);
        const double w1y = third<double>(y - 3 * qy), w1z = third<double>(z - 3 * qz);
        const long long sy = n1c, sz = static_cast<long long>(n1c) * n1c;
        auto prolong = [&](const double2* src) {  // computeV (y, then z, in the kernel's precision), then x
            C V[2];
#pragma unroll
            for (int dx = 0; dx < 2; ++dx) {
                const double2* c = src + (qx + dx) + sy * qy + sz * qz;
                const double2 a0 = lerpw(ld(c), ld(c + sy), w1y);
                const double2 a1 = lerpw(ld(c + sz), ld(c + sz + sy), w1y);
                V[dx] = to_c(lerpw(a0, a1, w1z), C{});
            }
            return lerpw(V[0], V[1], third<S>(x - 3 * qx));
        };
        C scv = prolong(scTD);
        // td-bpx: minus P si off the cPoints (phase B's `BPX && !(cpxy && u == 0)`)
        if (siTD && !(x % 3 == 0 && y % 3 == 0 && z % 3 == 0)) scv = sub(scv, prolong(siTD));
        uOut[f] = to_d(add(ld(vOld + f), scv));
    }
}

template <bool SMOOTH>
__global__ void __launch_bounds__(256) k_combine(const Args a, double2* rc, int za, int zb, const fast::ResArgs sa) {
    dev::griddep_wait();
    const int mc = a.g.mc, m = a.g.m, zc = a.g.zc;
    const unsigned n1c = a.n1c;
    const unsigned first = static_cast<unsigned>(za) * n1c * n1c;  // coarse lattices < 2^32 points
    const unsigned total = static_cast<unsigned>(zb - za) * n1c * n1c;
    const long long tilesXY = static_cast<long long>(a.g.nbx) * a.g.nby;
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const unsigned f = first + t;
        const unsigned fr = f / n1c;
        const int W0 = static_cast<int>(f - fr * n1c), W1 = static_cast<int>(fr % n1c), W2 = static_cast<int>(fr / n1c);
        if (W0 < 1 || W0 > mc - 1 || W1 < 1 || W1 > mc - 1 || W2 < 1 || W2 > mc - 1) continue;
        // the tiles / chunks covering W's stencil: at most two per axis (5 fine
        // points < TX, TY, zc); all candidate partials are loaded up front, then
        // added in the (bz, by, bx) order
        const int bz0 = (max(1, 3 * W2 - 2) - 1) / zc, bz1 = (min(m - 1, 3 * W2 + 2) - 1) / zc;
        const int by0 = (max(1, 3 * W1 - 2) - 1) / TY, by1 = (min(m - 1, 3 * W1 + 2) - 1) / TY;
        const int bx0 = (max(1, 3 * W0 - 2) - 1) / TX, bx1 = (min(m - 1, 3 * W0 + 2) - 1) / TX;
        double2 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int bz = bz0 + (q >> 2), by = by0 + ((q >> 1) & 1), bx = bx0 + (q & 1);
            const bool use = bz <= bz1 && by <= by1 && bx <= bx1;
            const int zi = W2 - (bz * zc) / 3, yi = W1 - (1 + by * TY) / 3, xi = W0 - (1 + bx * TX) / 3;
            const long long tile = bx + static_cast<long long>(a.g.nbx) * by;
            v[q] = use ? __ldcs(a.partial + ((static_cast<long long>(bz) * a.g.sz + zi) * tilesXY + tile) * (SY * SX) +
                                yi * SX + xi)
                       : zero2();
        }
        double2 acc = zero2();
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int bz = bz0 + (q >> 2), by = by0 + ((q >> 1) & 1), bx = bx0 + (q & 1);
            if (bz <= bz1 && by <= by1 && bx <= bx1) acc = add(acc, v[q]);
        }
        rc[f] = acc;
        if (SMOOTH) {  // level L-1 smoothing (k_smooth_coarse) on the value just formed
            const dev::Lvl& cl = sa.lv;
            if (sa.bpx && cl.si) {
                cl.si[f] = cl.sinext[f];
                cl.sinext[f] = zero2();
            }
            if (cl.level < sa.ellMin) {
                cl.sc[f] = zero2();
                continue;
            }
            const bool cp = (W0 % 3 == 0) && (W1 % 3 == 0) && (W2 % 3 == 0);
            const double2 smooth = mul(acc, sa.k.invDiag);
            cl.sc[f] = stage_sc(smooth, sa.k.wRaw, cp, sa.bpx, sa.hb);
            if (sa.bpx && cl.level > sa.ellMin && cp)
                sa.par.sinext[(W0 / 3) + sa.par.n1 * ((W1 / 3) + sa.par.n1 * (W2 / 3))] = mul(sa.k.wRaw, smooth);
        }
    }
}

}  // namespace

Geometry geometry(int m, int mc, int parts, int resident) {
    Geometry g{};
    g.m = m;
    g.mc = mc;
    const int inner = std::max(1, m - 1);
    g.nbx = (inner + TX - 1) / TX;
    g.nby = (inner + TY - 1) / TY;
    const int tiles = g.nbx * g.nby;
    parts = std::max(1, parts);
    // at least 8 chunks and ~2 waves of blocks (measured best at 243^3 and
    // 729^3; a finer wave model did not pay), in multiples of `parts`
    int want = std::max(8, (2 * std::max(1, resident) + tiles - 1) / tiles);
    if (dev::switches().zchunks > 0) want = dev::switches().zchunks;  // developer A/B
    want = (want + parts - 1) / parts * parts;
    for (;; want += parts) {
        g.zc = std::max(3, ((inner + want - 1) / want + 2) / 3 * 3);
        g.nbz = (inner + g.zc - 1) / g.zc;
        if (g.nbz % parts == 0 || g.zc == 3) break;
    }
    g.sz = g.zc / 3 + 2;
    return g;
}

size_t partial_count(const Geometry& g) {
    return static_cast<size_t>(g.nbx) * g.nby * g.nbz * g.sz * SY * SX;
}

int blocks(const Geometry& g) { return g.nbx * g.nby * g.nbz; }

namespace {
template <class S>
constexpr int rows_of() { return sizeof(S) == 4 ? TMG_F3_ROWS_C64 : TMG_F3_ROWS; }
template <class S, bool BPX>
constexpr size_t smem_of() {
    using C = typename Cx<S>::T;
    return rows_of<S>() == 2 ? Smem<C, 2>::template bytes<BPX>() : Smem<C, 1>::template bytes<BPX>();
}
template <bool BPX, class S>
constexpr auto kernel_of() { return rows_of<S>() == 2 ? k_fused3_r2<BPX, S> : k_fused3_r1<BPX, S>; }
}  // namespace

size_t smem_bytes(bool bpx, bool c64) {
    if (c64) return bpx ? smem_of<float, true>() : smem_of<float, false>();
    return bpx ? smem_of<double, true>() : smem_of<double, false>();
}

bool encode_map(CUtensorMap* map, const void* base, unsigned n1, int kind, bool c64, int nz) {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !ptr)
            return false;
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    const bool f32 = c64 && kind != 2;  // coarse planes stay complex128
    const cuuint64_t es = f32 ? 4 : 8;
    const cuuint64_t dims[3] = {2ull * n1, n1, nz > 0 ? static_cast<cuuint64_t>(nz) : n1};
    const cuuint64_t strides[2] = {2 * es * n1, 2 * es * n1 * n1};
    // kind 1 (b tiles): complex64 boxes are two columns wider (Smem::kBW)
    const cuuint32_t box[3] = {kind == 0 ? 2u * HX : kind == 1 ? 2u * (TX + (f32 ? 2u : 0u)) : 2u * CX,
                               static_cast<cuuint32_t>(kind == 0 ? HY : kind == 1 ? TY : CY), kind == 2 ? 2u : 1u};
    const cuuint32_t estr[3] = {1u, 1u, 1u};
    const CUresult r = fn(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                          const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

int resident_blocks(int smCount) {
    // blocks per SM of the non-BPX complex128 kernel at its dynamic shared memory size
    const size_t smem = smem_bytes(false);
    constexpr auto k = kernel_of<false, double>();
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int per = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, Cfg<rows_of<double>()>::NT, smem) != cudaSuccess ||
        per < 1)
        per = Cfg<rows_of<double>()>::MINB;
    return per * smCount;
}

namespace {
template <bool BPX, class S>
void launch_one(const Args& a, const CUtensorMap& mapU, const CUtensorMap& mapC, const CUtensorMap& mapI,
                const CUtensorMap& mapB, cudaStream_t s, dim3 grid) {
    // the shared-memory limit is a per-device function attribute: set it on every
    // launch (a host-side call, no device work) so a second device is configured too
    const size_t smem = smem_of<S, BPX>();
    constexpr auto k = kernel_of<BPX, S>();
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    dev::launch_k(k, grid, dim3(TX, Cfg<rows_of<S>()>::TYT), smem, s, mapU, mapC, mapI, mapB, a);
}
}  // namespace

void launch(const Args& a, const CUtensorMap& mapU, const CUtensorMap& mapC, const CUtensorMap& mapI,
            const CUtensorMap& mapB, cudaStream_t s, int nchunks) {
    const dim3 grid(a.g.nbx, a.g.nby, nchunks > 0 ? nchunks : a.g.nbz);
    if (a.c64) {
        if (a.bpx) launch_one<true, float>(a, mapU, mapC, mapI, mapB, s, grid);
        else launch_one<false, float>(a, mapU, mapC, mapI, mapB, s, grid);
    } else {
        if (a.bpx) launch_one<true, double>(a, mapU, mapC, mapI, mapB, s, grid);
        else launch_one<false, double>(a, mapU, mapC, mapI, mapB, s, grid);
    }
}

void derive_u(const void* vOld, const double2* scTD, const double2* siTD, unsigned n1, unsigned n1c, unsigned fa,
              unsigned fb, double2* uOut, bool c64, cudaStream_t s) {
    if (fb <= fa) return;
    const unsigned blocks = std::min<unsigned>((fb - fa + 255) / 256, 148u * 32u);
    if (c64)
        k_derive_u<float><<<blocks, 256, 0, s>>>(static_cast<const float2*>(vOld), scTD, siTD, n1, n1c, fa, fb, uOut);
    else
        k_derive_u<double><<<blocks, 256, 0, s>>>(static_cast<const double2*>(vOld), scTD, siTD, n1, n1c, fa, fb,
                                                  uOut);
}

void combine(const Args& a, double2* rCoarse, int nblocks, cudaStream_t s, int za, int zb,
             const fast::ResArgs* smooth) {
    if (za < 0) {
        za = 0;
        zb = a.g.mc + 1;
    }
    if (zb <= za) return;
    if (smooth) dev::launch_k(k_combine<true>, dim3(nblocks), dim3(256), 0, s, a, rCoarse, za, zb, *smooth);
    else dev::launch_k(k_combine<false>, dim3(nblocks), dim3(256), 0, s, a, rCoarse, za, zb, fast::ResArgs{});
}

}  // namespace fused3
}  // namespace tmg
