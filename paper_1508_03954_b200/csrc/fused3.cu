// Fused fine pass for 3D (see fused3.cuh).

#include "fused3.cuh"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>

namespace tmg {
namespace fused3 {

namespace {

__device__ __forceinline__ double2 zero2() { return make_double2(0.0, 0.0); }
__device__ __forceinline__ double2 add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 mul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 mac(double2 acc, double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, acc.x)), fma(a.x, b.y, fma(a.y, b.x, acc.y)));
}
__device__ __forceinline__ double2 axpy(double w, double2 v, double2 acc) {
    return make_double2(fma(w, v.x, acc.x), fma(w, v.y, acc.y));
}
__device__ __forceinline__ double2 ld(const double2* p) { return __ldg(p); }

__device__ __forceinline__ double2 lerp(double2 c0, double2 c1, int rel) {
    if (rel == 0) return c0;
    if (rel == 3) return c1;
    const double w1 = rel == 1 ? (1.0 / 3.0) : (2.0 / 3.0);
    return make_double2(fma(w1, c1.x - c0.x, c0.x), fma(w1, c1.y - c0.y, c0.y));
}

// trilinear prolongation from the coarse lattice (transfer.cpp:20-40 order)
__device__ __forceinline__ double2 prolong3(const double2* __restrict__ src, unsigned n1c, int mc, int x, int y,
                                            int z) {
    const int qx = min(x / 3, mc - 1), qy = min(y / 3, mc - 1), qz = min(z / 3, mc - 1);
    const int rx = x - 3 * qx, ry = y - 3 * qy, rz = z - 3 * qz;
    const double2* p = src + qx + static_cast<long long>(n1c) * (qy + static_cast<long long>(n1c) * qz);
    const long long sy = n1c, sz = static_cast<long long>(n1c) * n1c;
    const double2 a = lerp(ld(p), ld(p + 1), rx);
    const double2 b = lerp(ld(p + sy), ld(p + sy + 1), rx);
    const double2 c = lerp(ld(p + sz), ld(p + sz + 1), rx);
    const double2 d = lerp(ld(p + sz + sy), ld(p + sz + sy + 1), rx);
    return lerp(lerp(a, b, ry), lerp(c, d, ry), rz);
}

__device__ __forceinline__ double2 stage_sc(double2 smooth, double2 w, bool cp, int bpx, int hb) {
    if (bpx) return cp ? zero2() : mul(w, smooth);
    if ((hb && cp) || (w.x == 0.0 && w.y == 0.0)) return zero2();
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

constexpr int kPlane = (HX * HY + 7) / 8 * 8;  // stage strides: TMA destinations are 128-byte aligned
constexpr unsigned kTileBytes = HX * HY * sizeof(double2);
constexpr int kB = TX * TY;                      // b tile (no halo)
constexpr unsigned kBBytes = kB * sizeof(double2);
constexpr int kC = (CX * CY * 2 + 7) / 8 * 8;     // two coarse planes
constexpr unsigned kCBytes = CX * CY * 2 * sizeof(double2);

__device__ __forceinline__ double2 shfl2(double2 v, int src) {
    return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

__global__ void __launch_bounds__(TX* TY, 2)
    k_fused3(const __grid_constant__ CUtensorMap mapU, const __grid_constant__ CUtensorMap mapS,
             const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapC,
             const __grid_constant__ CUtensorMap mapI, const Args a) {
    extern __shared__ __align__(128) unsigned char smem[];
    double2* bufU = reinterpret_cast<double2*>(smem);
    double2* bufS = bufU + STAGES * kPlane;
    double2* bufB = bufS + STAGES * kPlane;
    double2* bufC = bufB + STAGES * kB;
    double2* bufI = bufC + STAGES * kC;             // BPX si planes (only when a.bpx)
    double2* plane = bufI + STAGES * kC;
    double2* xs = plane + 2 * kPlane;               // [TY][SX] x-restricted rows
    uint64_t* bar = reinterpret_cast<uint64_t*>(xs + TY * SX);

    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
    const int m = a.g.m, mc = a.g.mc;
    const int x0 = 1 + blockIdx.x * TX, y0 = 1 + blockIdx.y * TY, z0 = 1 + blockIdx.z * a.g.zc;
    const int xe = min(x0 + TX, m), ye = min(y0 + TY, m), z1 = min(z0 + a.g.zc, m);
    const int nplanes = z1 - z0 + 2;
    const long long sy = a.n1, sz = static_cast<long long>(a.n1) * a.n1;
    const int cx0 = (x0 - 1) / 3, cy0 = (y0 - 1) / 3;
    const unsigned stageBytes = 2 * kTileBytes + kBBytes + kCBytes * (a.bpx ? 2u : 1u);

    auto issue = [&](int stage, int zz) {
        const int cz = min(zz / 3, mc - 1);
        mbar_expect_tx(&bar[stage], stageBytes);
        tma_load3(bufU + stage * kPlane, &mapU, 2 * (x0 - 1), y0 - 1, zz, &bar[stage]);
        tma_load3(bufS + stage * kPlane, &mapS, 2 * (x0 - 1), y0 - 1, zz, &bar[stage]);
        tma_load3(bufB + stage * kB, &mapB, 2 * x0, y0, zz, &bar[stage]);
        tma_load3(bufC + stage * kC, &mapC, 2 * cx0, cy0, cz, &bar[stage]);
        if (a.bpx) tma_load3(bufI + stage * kC, &mapI, 2 * cx0, cy0, cz, &bar[stage]);
    };

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0)
        for (int s = 0; s < STAGES && s < nplanes; ++s) issue(s, z0 - 1 + s);

    const int x = x0 + tx, y = y0 + ty;
    const bool owned = x < xe && y < ye;
    const bool cpxy = (x % 3 == 0) && (y % 3 == 0);
    double2 Cm = zero2(), Em = zero2(), Km = zero2(), C0 = zero2(), E0 = zero2(), K0 = zero2();
    double nmax = 0.0, nsum = 0.0;

    // restriction slots of this tile
    const int Xa = x0 / 3, Xb = (xe + 1) / 3, Ya = y0 / 3, Yb = (ye + 1) / 3;
    const int nsx = Xb - Xa + 1, nsy = Yb - Ya + 1;
    const long long blockLin =
        blockIdx.x + static_cast<long long>(gridDim.x) * (blockIdx.y + static_cast<long long>(gridDim.y) * blockIdx.z);
    double2* part = a.partial + blockLin * static_cast<long long>(a.g.sz * SY * SX);
    const int zBase = (z0 - 1) / 3;
    int zLow = zBase;
    double2 accLo = zero2(), accHi = zero2();
    const bool slotThread = tid < nsx * nsy;
    const int sxi = slotThread ? tid % nsx : 0, syi = slotThread ? tid / nsx : 0;

    for (int it = 0; it < nplanes; ++it) {
        const int zz = z0 - 1 + it;
        const int s = it % STAGES;
        mbar_wait(&bar[s], static_cast<unsigned>((it / STAGES) & 1));
        double2* P = plane + (it & 1) * kPlane;
        {
            const double2* U = bufU + s * kPlane;
            const double2* Sc = bufS + s * kPlane;
            const double2* Cc = bufC + s * kC;
            const double2* Ci = bufI + s * kC;
            const bool zin = zz >= 1 && zz <= m - 1;
            const int cz = min(zz / 3, mc - 1), rz = zz - 3 * cz;
            for (int p = tid; p < HX * HY; p += TX * TY) {
                const int lx = p % HX, ly = p / HX;
                const int gx = x0 - 1 + lx, gy = y0 - 1 + ly;
                double2 v = zero2();
                if (zin && gx >= 1 && gx <= m - 1 && gy >= 1 && gy <= m - 1) {
                    const int qx = min(gx / 3, mc - 1), qy = min(gy / 3, mc - 1);
                    const int rx = gx - 3 * qx, ry = gy - 3 * qy;
                    const int o = (qx - cx0) + CX * (qy - cy0);
                    auto tri = [&](const double2* C) {
                        const double2 a0 = lerp(C[o], C[o + 1], rx), a1 = lerp(C[o + CX], C[o + CX + 1], rx);
                        const double2 b0 = lerp(C[o + CX * CY], C[o + CX * CY + 1], rx);
                        const double2 b1 = lerp(C[o + CX * CY + CX], C[o + CX * CY + CX + 1], rx);
                        return lerp(lerp(a0, a1, ry), lerp(b0, b1, ry), rz);
                    };
                    double2 scv = add(Sc[p], tri(Cc));
                    if (a.bpx && !((gx % 3 == 0) && (gy % 3 == 0) && (zz % 3 == 0))) scv = sub(scv, tri(Ci));
                    v = add(U[p], scv);
                }
                P[p] = v;
            }
        }
        __syncthreads();
        double2 Cp = zero2(), Ep = zero2(), Kp = zero2();
        if (owned) {
            const double2* c = P + (ty + 1) * HX + (tx + 1);
            Cp = c[0];
            Ep = add(add(c[-1], c[1]), add(c[-HX], c[HX]));
            Kp = add(add(c[-1 - HX], c[1 - HX]), add(c[-1 + HX], c[1 + HX]));
            if (zz >= z0 && zz < z1) a.uNew[x + y * sy + zz * sz] = Cp;
        }
        if (it >= 2) {
            const int z = zz - 1;
            const int sb = (it - 1) % STAGES;
            double2 r = zero2();
            if (owned) {
                const double2 faces = add(E0, add(Cm, Cp));
                const double2 edges = add(K0, add(Em, Ep));
                const double2 corners = add(Km, Kp);
                double2 hu = mul(a.k.c[0], C0);
                hu = mac(hu, a.k.c[1], faces);
                hu = mac(hu, a.k.c[2], edges);
                hu = mac(hu, a.k.c[3], corners);
                r = sub(bufB[sb * kB + ty * TX + tx], hu);
                const double m2 = fma(r.x, r.x, r.y * r.y);
                nmax = fmax(nmax, m2);
                nsum += m2;
                const bool cp = cpxy && (z % 3 == 0);
                const double2 smooth = mul(r, a.k.invDiag);
                const long long f = x + y * sy + z * sz;
                a.scNew[f] = a.level < a.ellMin ? zero2() : stage_sc(smooth, a.k.wRaw, cp, a.bpx, a.hb);
                if (a.bpx && cp && a.level > a.ellMin)
                    a.sinextC[(x / 3) + a.n1c * (static_cast<long long>(y / 3) + static_cast<long long>(a.n1c) * (z / 3))] =
                        mul(a.k.wRaw, smooth);
            }
            // restriction, x direction, inside the row's warp (lane j -> slot X = Xa + j)
            {
                const int X = Xa + tx;
                double2 acc = zero2();
#pragma unroll
                for (int k = -2; k <= 2; ++k) {
                    const int lane = 3 * X + k - x0;
                    const double2 v = shfl2(r, lane & 31);
                    const double w = (k == 0) ? 1.0 : ((k == -1 || k == 1) ? 2.0 / 3.0 : 1.0 / 3.0);
                    if (lane >= 0 && lane < 32 && tx < nsx) acc = axpy(w, v, acc);
                }
                if (tx < nsx) xs[ty * SX + tx] = acc;
            }
            __syncthreads();
            if (tid == 0 && it - 1 + STAGES < nplanes) issue(sb, zz - 1 + STAGES);
            if (slotThread) {
                const int Y = Ya + syi;
                double2 val = zero2();
#pragma unroll
                for (int k = -2; k <= 2; ++k) {
                    const int fy = 3 * Y + k;
                    const double w = (k == 0) ? 1.0 : ((k == -1 || k == 1) ? 2.0 / 3.0 : 1.0 / 3.0);
                    if (fy >= y0 && fy < ye) val = axpy(w, xs[(fy - y0) * SX + sxi], val);
                }
                const int kz = z % 3;
                if (kz == 0) {
                    accLo = add(accLo, val);
                } else if (kz == 1) {
                    accLo = axpy(2.0 / 3.0, val, accLo);
                    accHi = axpy(1.0 / 3.0, val, accHi);
                } else {
                    accLo = axpy(1.0 / 3.0, val, accLo);
                    accHi = axpy(2.0 / 3.0, val, accHi);
                    part[((zLow - zBase) * SY + syi) * SX + sxi] = accLo;
                    ++zLow;
                    accLo = accHi;
                    accHi = zero2();
                }
            }
        } else if (it == 1 && tid == 0 && STAGES < nplanes) {
            issue(0, z0 - 1 + STAGES);  // plane z0-1 is halo only: its stage is free after the sync
        }
        Cm = C0;
        Em = E0;
        Km = K0;
        C0 = Cp;
        E0 = Ep;
        K0 = Kp;
    }
    if (slotThread) {
        part[((zLow - zBase) * SY + syi) * SX + sxi] = accLo;
        part[((zLow + 1 - zBase) * SY + syi) * SX + sxi] = accHi;
    }
    dev::block_norms(nmax, nsum, a.norms);
}

__global__ void __launch_bounds__(256) k_combine(const Args a, double2* rc) {
    const int mc = a.g.mc, m = a.g.m, zc = a.g.zc;
    const unsigned n1c = a.n1c;
    const unsigned total = n1c * n1c * n1c;
    for (unsigned f = blockIdx.x * blockDim.x + threadIdx.x; f < total; f += gridDim.x * blockDim.x) {
        const int W0 = static_cast<int>(f % n1c), W1 = static_cast<int>((f / n1c) % n1c),
                  W2 = static_cast<int>(f / (n1c * n1c));
        if (W0 < 1 || W0 > mc - 1 || W1 < 1 || W1 > mc - 1 || W2 < 1 || W2 > mc - 1) continue;
        double2 acc = zero2();
        const int bz0 = (max(1, 3 * W2 - 2) - 1) / zc, bz1 = (min(m - 1, 3 * W2 + 2) - 1) / zc;
        const int by0 = (max(1, 3 * W1 - 2) - 1) / TY, by1 = (min(m - 1, 3 * W1 + 2) - 1) / TY;
        const int bx0 = (max(1, 3 * W0 - 2) - 1) / TX, bx1 = (min(m - 1, 3 * W0 + 2) - 1) / TX;
        for (int bz = bz0; bz <= bz1; ++bz) {
            const int zi = W2 - (bz * zc) / 3;
            for (int by = by0; by <= by1; ++by) {
                const int yi = W1 - (1 + by * TY) / 3;
                for (int bx = bx0; bx <= bx1; ++bx) {
                    const int xi = W0 - (1 + bx * TX) / 3;
                    const long long bl = bx + static_cast<long long>(a.g.nbx) * (by + static_cast<long long>(a.g.nby) * bz);
                    acc = add(acc, a.partial[((bl * a.g.sz + zi) * SY + yi) * SX + xi]);
                }
            }
        }
        rc[f] = acc;
    }
}

}  // namespace

Geometry geometry(int m, int mc) {
    Geometry g{};
    g.m = m;
    g.mc = mc;
    const int inner = std::max(1, m - 1);
    g.nbx = (inner + TX - 1) / TX;
    g.nby = (inner + TY - 1) / TY;
    const int tiles = g.nbx * g.nby;
    const int want = std::max(1, (4 * 2 * 148 + tiles - 1) / tiles);
    g.zc = std::max(3, ((inner + want - 1) / want + 2) / 3 * 3);
    g.nbz = (inner + g.zc - 1) / g.zc;
    g.sz = g.zc / 3 + 2;
    return g;
}

size_t partial_count(const Geometry& g) {
    return static_cast<size_t>(g.nbx) * g.nby * g.nbz * g.sz * SY * SX;
}

int blocks(const Geometry& g) { return g.nbx * g.nby * g.nbz; }

size_t smem_bytes() {
    return (2 * STAGES * kPlane + STAGES * kB + 2 * STAGES * kC + 2 * kPlane + TY * SX) * sizeof(double2) +
           STAGES * sizeof(uint64_t);
}

bool encode_map(CUtensorMap* map, const double2* base, unsigned n1, int kind) {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !ptr)
            return false;
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    const cuuint64_t dims[3] = {2ull * n1, n1, n1};
    const cuuint64_t strides[2] = {16ull * n1, 16ull * n1 * n1};
    const cuuint32_t box[3] = {kind == 0 ? 2u * HX : kind == 1 ? 2u * TX : 2u * CX,
                               static_cast<cuuint32_t>(kind == 0 ? HY : kind == 1 ? TY : CY), kind == 2 ? 2u : 1u};
    const cuuint32_t estr[3] = {1u, 1u, 1u};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double2*>(base), dims, strides, box,
                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

void launch(const Args& a, const CUtensorMap& mapU, const CUtensorMap& mapS, const CUtensorMap& mapB,
            const CUtensorMap& mapC, const CUtensorMap& mapI, cudaStream_t s) {
    static bool configured = false;
    const size_t smem = smem_bytes();
    if (!configured) {
        cudaFuncSetAttribute(k_fused3, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        configured = true;
    }
    dim3 grid(a.g.nbx, a.g.nby, a.g.nbz);
    k_fused3<<<grid, dim3(TX, TY), smem, s>>>(mapU, mapS, mapB, mapC, mapI, a);
}

void combine(const Args& a, double2* rCoarse, int nblocks, cudaStream_t s) {
    k_combine<<<nblocks, 256, 0, s>>>(a, rCoarse);
}

}  // namespace fused3
}  // namespace tmg
