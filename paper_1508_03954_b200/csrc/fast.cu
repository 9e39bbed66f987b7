// Fast-precision cycle kernels; see fast.cuh for the formulation and
// DESIGN.md §3 for the roofline of each kernel.

#include "fast.cuh"

#include <algorithm>
#include <cstdlib>

namespace tmg {
namespace fast {

using dev::Lvl;

namespace {

__device__ __forceinline__ double2 add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 mul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// acc + a * b
__device__ __forceinline__ double2 mac(double2 acc, double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, acc.x)), fma(a.x, b.y, fma(a.y, b.x, acc.y)));
}
__device__ __forceinline__ double2 ld(const double2* p) { return __ldg(p); }

__device__ __forceinline__ double2 lerp(double2 c0, double2 c1, int rel) {
    if (rel == 0) return c0;
    if (rel == 3) return c1;
    const double w1 = rel == 1 ? (1.0 / 3.0) : (2.0 / 3.0);
    return make_double2(fma(w1, c1.x - c0.x, c0.x), fma(w1, c1.y - c0.y, c0.y));
}

template <int P>
__device__ __forceinline__ double2 prolong_at(const double2* __restrict__ src, unsigned n1, const int* q,
                                              const int* rel) {
    double2 v[1 << P];
#pragma unroll
    for (int e = 0; e < (1 << P); ++e) {
        unsigned f = 0, s = 1;
#pragma unroll
        for (int d = 0; d < P; ++d) {
            f += static_cast<unsigned>(q[d] + ((e >> d) & 1)) * s;
            s *= n1;
        }
        v[e] = ld(src + f);
    }
#pragma unroll
    for (int d = 0; d < P; ++d)
#pragma unroll
        for (int i = 0; i < (1 << (P - 1 - d)); ++i) v[i] = lerp(v[2 * i], v[2 * i + 1], rel[d]);
    return v[0];
}

// sc staging shared by fine and coarse smoothing (cycles.cpp:264-278)
__device__ __forceinline__ double2 stage(double2 smooth, double2 w, bool cp, int bpx, int hb) {
    if (bpx) return cp ? make_double2(0.0, 0.0) : mul(w, smooth);
    if ((hb && cp) || (w.x == 0.0 && w.y == 0.0)) return make_double2(0.0, 0.0);
    return mul(w, smooth);
}

// ---- K1f / K1c: top-down correction ----------------------------------------
template <int P, bool FINE>
__global__ void __launch_bounds__(256) k_topdown(Lvl c, Lvl pr, int bpx, unsigned fa, unsigned fb) {
    dev::griddep_wait();
    for (unsigned f = fa + blockIdx.x * blockDim.x + threadIdx.x; f < fb; f += gridDim.x * blockDim.x) {
        int idx[P];
        dev::unflat<P>(f, c.n1, idx);
        if (dev::on_boundary<P>(idx, static_cast<int>(c.m))) continue;  // u = sc = 0 stay pinned
        int q[P], rel[P];
#pragma unroll
        for (int d = 0; d < P; ++d) {
            q[d] = min(idx[d] / 3, static_cast<int>(pr.m) - 1);
            rel[d] = idx[d] - 3 * q[d];
        }
        double2 sc = add(c.sc[f], prolong_at<P>(pr.sc, pr.n1, q, rel));
        if (bpx && !dev::is_cpoint<P>(idx)) sc = sub(sc, prolong_at<P>(pr.si, pr.n1, q, rel));
        if (FINE) {
            c.u[f] = add(c.u[f], sc);  // sf is identically zero on the finest level
        } else {
            (c.scOut ? c.scOut : c.sc)[f] = sc;
        }
    }
}

// Same update, one thread per parent cell column in x: the three fine points
// x = 3qx + {0,1,2} share their 2^P parent values, loaded once (P = 2, 3).
template <int P, bool FINE>
__global__ void __launch_bounds__(256) k_topdown_tri(Lvl c, Lvl pr, int bpx, unsigned ra, unsigned rb) {
    dev::griddep_wait();
    const unsigned mcp = pr.m, n1 = c.n1;
    const int m = static_cast<int>(c.m);
    const unsigned total = (rb - ra) * mcp;  // rows [ra, rb) of the (P-1)-dim row index
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const unsigned row = ra + t / mcp;
        const int qx = static_cast<int>(t - (t / mcp) * mcp);
        int idx[P];
        unsigned rr = row;
#pragma unroll
        for (int d = 1; d < P; ++d) {
            idx[d] = static_cast<int>(rr % n1);
            rr /= n1;
        }
        bool bnd = false;
#pragma unroll
        for (int d = 1; d < P; ++d) bnd |= (idx[d] == 0) | (idx[d] == m);
        if (bnd) continue;
        int q[P], rel[P];
        q[0] = qx;
#pragma unroll
        for (int d = 1; d < P; ++d) {
            q[d] = min(idx[d] / 3, static_cast<int>(mcp) - 1);
            rel[d] = idx[d] - 3 * q[d];
        }
        double2 vs[1 << P], vi[1 << P];
#pragma unroll
        for (int e = 0; e < (1 << P); ++e) {
            unsigned f = 0, s = 1;
#pragma unroll
            for (int d = 0; d < P; ++d) {
                f += static_cast<unsigned>(q[d] + ((e >> d) & 1)) * s;
                s *= pr.n1;
            }
            vs[e] = ld(pr.sc + f);
            vi[e] = bpx ? ld(pr.si + f) : make_double2(0.0, 0.0);
        }
        bool cpr = true;
#pragma unroll
        for (int d = 1; d < P; ++d) cpr &= idx[d] % 3 == 0;
        const unsigned fb = row * n1;
        double2 own[3];  // the three points' current values, loaded before any store
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int x = 3 * qx + k;
            own[k] = (x >= 1 && x <= m - 1) ? ld((FINE ? c.u : c.sc) + fb + static_cast<unsigned>(x)) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int x = 3 * qx + k;
            if (x < 1 || x > m - 1) continue;
            rel[0] = k;
            double2 w[1 << P];
#pragma unroll
            for (int e = 0; e < (1 << P); ++e) w[e] = vs[e];
#pragma unroll
            for (int d = 0; d < P; ++d)
#pragma unroll
                for (int i = 0; i < (1 << (P - 1 - d)); ++i) w[i] = lerp(w[2 * i], w[2 * i + 1], rel[d]);
            const unsigned f = fb + static_cast<unsigned>(x);
            double2 sc = add(FINE ? c.sc[f] : own[k], w[0]);  // k_topdown order: (sc + P sc) - P si
            if (bpx && !(cpr && k == 0)) {
#pragma unroll
                for (int e = 0; e < (1 << P); ++e) w[e] = vi[e];
#pragma unroll
                for (int d = 0; d < P; ++d)
#pragma unroll
                    for (int i = 0; i < (1 << (P - 1 - d)); ++i) w[i] = lerp(w[2 * i], w[2 * i + 1], rel[d]);
                sc = sub(sc, w[0]);
            }
            if (FINE) c.u[f] = add(own[k], sc);
            else (c.scOut ? c.scOut : c.sc)[f] = sc;
        }
    }
}

// ---- K2f (3D): r = b - H u by z-marching planes -----------------------------
// Block = 32 x 4 columns (x, y); each thread walks ZCH planes in z, forming per
// plane the centre / 4-edge / 4-corner sums of its 3x3 neighbourhood so every
// u value is loaded 9x per vertex from L1 (not 27x) and once from HBM.
constexpr int TX = 32, TY = 4;

__global__ void __launch_bounds__(TX* TY) k_residual3(ResArgs a, int zch) {
    const Lvl& F = a.lv;
    const int m = static_cast<int>(F.m);
    const long long sy = F.n1, sz = static_cast<long long>(F.n1) * F.n1;
    const int x = blockIdx.x * TX + threadIdx.x + 1;
    const int y = blockIdx.y * TY + threadIdx.y + 1;
    const int z0 = blockIdx.z * zch + 1;
    const int z1 = min(z0 + zch, m);
    double nmax = 0.0, nsum = 0.0;
    if (x <= m - 1 && y <= m - 1 && z0 < z1) {
        const double2 c0 = a.k.c[0], c1 = a.k.c[1], c2 = a.k.c[2], c3 = a.k.c[3];
        const double2* __restrict__ u = F.u;
        const long long base = x + y * sy;
        auto plane = [&](int z, double2& C, double2& E, double2& K) {
            const double2* p = u + base + z * sz;
            C = ld(p);
            E = add(add(ld(p - 1), ld(p + 1)), add(ld(p - sy), ld(p + sy)));
            K = add(add(ld(p - 1 - sy), ld(p + 1 - sy)), add(ld(p - 1 + sy), ld(p + 1 + sy)));
        };
        double2 Cm, Em, Km, C0, E0, K0, Cp, Ep, Kp;
        plane(z0 - 1, Cm, Em, Km);
        plane(z0, C0, E0, K0);
        const bool cpxy = (x % 3 == 0) && (y % 3 == 0);
        const bool inject = a.bpx && F.level > a.ellMin;
        for (int z = z0; z < z1; ++z) {
            plane(z + 1, Cp, Ep, Kp);
            const double2 faces = add(E0, add(Cm, Cp));
            const double2 edges = add(K0, add(Em, Ep));
            const double2 corners = add(Km, Kp);
            double2 hu = mul(c0, C0);
            hu = mac(hu, c1, faces);
            hu = mac(hu, c2, edges);
            hu = mac(hu, c3, corners);
            const long long f = base + z * sz;
            const double2 r = sub(ld(F.chi + f), hu);
            const double m2 = fma(r.x, r.x, r.y * r.y);
            nmax = fmax(nmax, m2);
            nsum += m2;
            const bool cp = cpxy && (z % 3 == 0);
            const double2 smooth = mul(r, a.k.invDiag);
            F.sc[f] = F.level < a.ellMin ? make_double2(0.0, 0.0) : stage(smooth, a.k.wRaw, cp, a.bpx, a.hb);
            F.rhat[f] = r;
            if (inject && cp) {
                const unsigned wf = static_cast<unsigned>(x / 3) +
                                    a.par.n1 * (static_cast<unsigned>(y / 3) + a.par.n1 * static_cast<unsigned>(z / 3));
                a.par.sinext[wf] = mul(a.k.wRaw, smooth);
            }
            Cm = C0; Em = E0; Km = K0;
            C0 = Cp; E0 = Ep; K0 = Kp;
        }
    }
    dev::block_norms(nmax, nsum, a.partials);
}

// ---- fast load vector: b = ms (M x M x M) f, the assembled consistent mass
// matrix as a separable 1/6 2/3 1/6 stencil per axis (kernels.cpp:69-87 summed
// over the cells around each vertex; interior vertices only, the boundary ones
// are pinned).  z-marching like k_residual3: 32 B of HBM per vertex.
__global__ void __launch_bounds__(TX* TY) k_load3(Lvl F, const double2* __restrict__ f, double2 ms, int zlo,
                                                  int zhi, int zch) {
    const int m = static_cast<int>(F.m);
    const long long sy = F.n1, sz = static_cast<long long>(F.n1) * F.n1;
    const int x = blockIdx.x * TX + threadIdx.x + 1;
    const int y = blockIdx.y * TY + threadIdx.y + 1;
    const int z0 = zlo + blockIdx.z * zch;
    const int z1 = min(z0 + zch, zhi);
    if (x > m - 1 || y > m - 1 || z0 >= z1) return;
    const long long base = x + y * sy;
    const double wc = 4.0 / 9.0, we = 1.0 / 9.0, wk = 1.0 / 36.0;  // (2/3)^2, (2/3)(1/6), (1/6)^2
    auto plane = [&](int z) {
        const double2* p = f + base + z * sz;
        const double2 C = ld(p);
        const double2 E = add(add(ld(p - 1), ld(p + 1)), add(ld(p - sy), ld(p + sy)));
        const double2 K = add(add(ld(p - 1 - sy), ld(p + 1 - sy)), add(ld(p - 1 + sy), ld(p + 1 + sy)));
        return make_double2(fma(wc, C.x, fma(we, E.x, wk * K.x)), fma(wc, C.y, fma(we, E.y, wk * K.y)));
    };
    double2 Sm = plane(z0 - 1), S0 = plane(z0);
    for (int z = z0; z < z1; ++z) {
        const double2 Sp = plane(z + 1);
        const double2 S = make_double2(fma(2.0 / 3.0, S0.x, (Sm.x + Sp.x) / 6.0), fma(2.0 / 3.0, S0.y, (Sm.y + Sp.y) / 6.0));
        F.chi[base + z * sz] = mul(ms, S);
        Sm = S0;
        S0 = Sp;
    }
}

template <int P>
__global__ void __launch_bounds__(256) k_load_lowdim(Lvl F, const double2* __restrict__ f, double2 ms) {
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < F.n; i += gridDim.x * blockDim.x) {
        int idx[P];
        dev::unflat<P>(i, F.n1, idx);
        if (dev::on_boundary<P>(idx, static_cast<int>(F.m))) continue;
        double2 S;
        if (P == 1) {
            S = make_double2(fma(2.0 / 3.0, f[i].x, (f[i - 1].x + f[i + 1].x) / 6.0),
                             fma(2.0 / 3.0, f[i].y, (f[i - 1].y + f[i + 1].y) / 6.0));
        } else {
            const long long sy = F.n1;
            const double2* p = f + i;
            const double2 C = ld(p);
            const double2 E = add(add(ld(p - 1), ld(p + 1)), add(ld(p - sy), ld(p + sy)));
            const double2 K = add(add(ld(p - 1 - sy), ld(p + 1 - sy)), add(ld(p - 1 + sy), ld(p + 1 + sy)));
            const double wc = 4.0 / 9.0, we = 1.0 / 9.0, wk = 1.0 / 36.0;
            S = make_double2(fma(wc, C.x, fma(we, E.x, wk * K.x)), fma(wc, C.y, fma(we, E.y, wk * K.y)));
        }
        F.chi[i] = mul(ms, S);
    }
}

// ---- K2f (1D / 2D): thread per vertex ---------------------------------------
template <int P>
__global__ void __launch_bounds__(256) k_residual_lowdim(ResArgs a) {
    const Lvl& F = a.lv;
    double nmax = 0.0, nsum = 0.0;
    for (unsigned f = blockIdx.x * blockDim.x + threadIdx.x; f < F.n; f += gridDim.x * blockDim.x) {
        int idx[P];
        dev::unflat<P>(f, F.n1, idx);
        if (dev::on_boundary<P>(idx, static_cast<int>(F.m))) continue;
        double2 hu;
        if (P == 1) {
            hu = mul(a.k.c[0], ld(F.u + f));
            hu = mac(hu, a.k.c[1], add(ld(F.u + f - 1), ld(F.u + f + 1)));
        } else {
            const long long sy = F.n1;
            const double2* p = F.u + f;
            hu = mul(a.k.c[0], ld(p));
            hu = mac(hu, a.k.c[1], add(add(ld(p - 1), ld(p + 1)), add(ld(p - sy), ld(p + sy))));
            hu = mac(hu, a.k.c[2], add(add(ld(p - 1 - sy), ld(p + 1 - sy)), add(ld(p - 1 + sy), ld(p + 1 + sy))));
        }
        const double2 r = sub(ld(F.chi + f), hu);
        const double m2 = fma(r.x, r.x, r.y * r.y);
        nmax = fmax(nmax, m2);
        nsum += m2;
        const bool cp = dev::is_cpoint<P>(idx);
        const double2 smooth = mul(r, a.k.invDiag);
        F.sc[f] = F.level < a.ellMin ? make_double2(0.0, 0.0) : stage(smooth, a.k.wRaw, cp, a.bpx, a.hb);
        F.rhat[f] = r;
        if (a.bpx && F.level > a.ellMin && cp) {
            int wi[P];
#pragma unroll
            for (int d = 0; d < P; ++d) wi[d] = idx[d] / 3;
            a.par.sinext[dev::flat<P>(wi, a.par.n1)] = mul(a.k.wRaw, smooth);
        }
    }
    dev::block_norms(nmax, nsum, a.partials);
}

// k_smooth_coarse's update of one interior point on its just-restricted residual
// (the restriction kernels' fold; boundary sc / si stay zero)
template <int P>
__device__ __forceinline__ void smooth_interior(const ResArgs& a, unsigned f, const int* idx, double2 r) {
    const Lvl& c = a.lv;
    if (a.bpx && c.si) {
        c.si[f] = c.sinext[f];
        c.sinext[f] = make_double2(0.0, 0.0);
    }
    if (c.level < a.ellMin) {
        c.sc[f] = make_double2(0.0, 0.0);
        return;
    }
    const bool cp = dev::is_cpoint<P>(idx);
    const double2 smooth = mul(r, a.k.invDiag);
    c.sc[f] = stage(smooth, a.k.wRaw, cp, a.bpx, a.hb);
    if (a.bpx && c.level > a.ellMin && cp) {
        int wi[P];
#pragma unroll
        for (int d = 0; d < P; ++d) wi[d] = idx[d] / 3;
        a.par.sinext[dev::flat<P>(wi, a.par.n1)] = mul(a.k.wRaw, smooth);
    }
}

// ---- K3r: r_{l-1} = R r_l (separable 1D weights 1/3 2/3 1 2/3 1/3) -----------
// SMOOTH: also the coarse level's smoothing on the value just formed.
template <int P, bool SMOOTH = false>
__global__ void __launch_bounds__(256) k_restrict(Lvl fine, Lvl coarse, unsigned fa, unsigned fb, const ResArgs sa) {
    dev::griddep_wait();
    const double w[5] = {1.0 / 3.0, 2.0 / 3.0, 1.0, 2.0 / 3.0, 1.0 / 3.0};
    const long long sy = fine.n1, sz = static_cast<long long>(fine.n1) * fine.n1;
    for (unsigned f = fa + blockIdx.x * blockDim.x + threadIdx.x; f < fb; f += gridDim.x * blockDim.x) {
        int W[P];
        dev::unflat<P>(f, coarse.n1, W);
        if (dev::on_boundary<P>(W, static_cast<int>(coarse.m))) continue;
        long long centre = 0, s = 1;
#pragma unroll
        for (int d = 0; d < P; ++d) {
            centre += 3LL * W[d] * s;
            s *= fine.n1;
        }
        const double2* __restrict__ r = fine.rhat + centre;
        double2 acc = make_double2(0.0, 0.0);
        if (P == 1) {
#pragma unroll
            for (int i = 0; i < 5; ++i) {
                const double2 v = ld(r + (i - 2));
                acc.x = fma(w[i], v.x, acc.x);
                acc.y = fma(w[i], v.y, acc.y);
            }
        } else if (P == 2) {
#pragma unroll
            for (int j = 0; j < 5; ++j) {
                double2 row = make_double2(0.0, 0.0);
#pragma unroll
                for (int i = 0; i < 5; ++i) {
                    const double2 v = ld(r + (j - 2) * sy + (i - 2));
                    row.x = fma(w[i], v.x, row.x);
                    row.y = fma(w[i], v.y, row.y);
                }
                acc.x = fma(w[j], row.x, acc.x);
                acc.y = fma(w[j], row.y, acc.y);
            }
        } else {
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                double2 pl = make_double2(0.0, 0.0);
#pragma unroll
                for (int j = 0; j < 5; ++j) {
                    double2 row = make_double2(0.0, 0.0);
#pragma unroll
                    for (int i = 0; i < 5; ++i) {
                        const double2 v = ld(r + (k - 2) * sz + (j - 2) * sy + (i - 2));
                        row.x = fma(w[i], v.x, row.x);
                        row.y = fma(w[i], v.y, row.y);
                    }
                    pl.x = fma(w[j], row.x, pl.x);
                    pl.y = fma(w[j], row.y, pl.y);
                }
                acc.x = fma(w[k], pl.x, acc.x);
                acc.y = fma(w[k], pl.y, acc.y);
            }
        }
        coarse.rhat[f] = acc;
        if (SMOOTH) smooth_interior<P>(sa, f, W, acc);
    }
}

// ---- 3D row kernels for the big coarse levels ----------------------------------
// One block per (y, z) row: the four parent rows a row interpolates from (and
// for the restriction the 25 fine rows a coarse row gathers) are staged in
// shared memory once, so the per-point work is a handful of lerps instead of
// eight scattered loads with full index arithmetic.  Same arithmetic order as
// prolong_at / k_restrict (bitwise equal results).
constexpr int kRowThreads = 256;

__global__ void __launch_bounds__(kRowThreads) k_topdown3_rows(Lvl c, Lvl pr, int bpx, int zlo) {
    dev::griddep_wait();
    extern __shared__ double2 rs[];  // [4 (+4 BPX)][pr.n1]
    const int m = static_cast<int>(c.m), mcp = static_cast<int>(pr.m);
    const int y = 1 + blockIdx.x, z = zlo + blockIdx.y;
    const int qy = min(y / 3, mcp - 1), qz = min(z / 3, mcp - 1);
    const int ry = y - 3 * qy, rz = z - 3 * qz;
    const unsigned pn1 = pr.n1;
    const int nsrc = bpx ? 8 : 4;
    for (int t = threadIdx.x; t < nsrc * static_cast<int>(pn1); t += blockDim.x) {
        const int r = t / static_cast<int>(pn1), qx = t % static_cast<int>(pn1);
        const int e = r & 3;
        const double2* src = r < 4 ? pr.sc : pr.si;
        rs[t] = ld(src + qx + pn1 * (static_cast<unsigned>(qy + (e & 1)) + pn1 * static_cast<unsigned>(qz + (e >> 1))));
    }
    __syncthreads();
    const bool cpyz = (y % 3 == 0) && (z % 3 == 0);
    const size_t rowOff = c.n1 * (static_cast<unsigned>(y) + c.n1 * static_cast<unsigned>(z));
    const double2* row = c.sc + rowOff;
    double2* out = (c.scOut ? c.scOut : c.sc) + rowOff;
    for (int x = 1 + threadIdx.x; x <= m - 1; x += blockDim.x) {
        const int qx = min(x / 3, mcp - 1), rx = x - 3 * qx;
        auto pro = [&](const double2* R) {
            const double2 a0 = lerp(R[qx], R[qx + 1], rx);
            const double2 a1 = lerp(R[pn1 + qx], R[pn1 + qx + 1], rx);
            const double2 a2 = lerp(R[2 * pn1 + qx], R[2 * pn1 + qx + 1], rx);
            const double2 a3 = lerp(R[3 * pn1 + qx], R[3 * pn1 + qx + 1], rx);
            return lerp(lerp(a0, a1, ry), lerp(a2, a3, ry), rz);
        };
        double2 sc = add(row[x], pro(rs));
        if (bpx && !(cpyz && x % 3 == 0)) sc = sub(sc, pro(rs + 4 * pn1));
        out[x] = sc;
    }
}

template <bool SMOOTH = false>
__global__ void __launch_bounds__(kRowThreads) k_restrict3_rows(Lvl fine, Lvl coarse, int zlo, const ResArgs sa) {
    dev::griddep_wait();
    extern __shared__ double2 rw[];  // [25][coarse.n1] x-restricted fine rows
    const double w[5] = {1.0 / 3.0, 2.0 / 3.0, 1.0, 2.0 / 3.0, 1.0 / 3.0};
    const int mc = static_cast<int>(coarse.m);
    const int W1 = 1 + blockIdx.x, W2 = zlo + blockIdx.y;
    const unsigned fn1 = fine.n1, cn1 = coarse.n1;
    const int nW = mc - 1;
    for (int t = threadIdx.x; t < 25 * nW; t += blockDim.x) {
        const int jk = t / nW, W0 = 1 + t % nW;
        const int j = jk % 5, k = jk / 5;
        const double2* r = fine.rhat + static_cast<long long>(3 * W0) +
                           fn1 * (static_cast<long long>(3 * W1 + j - 2) + static_cast<long long>(fn1) * (3 * W2 + k - 2));
        double2 rowv = make_double2(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            const double2 v = ld(r + (i - 2));
            rowv.x = fma(w[i], v.x, rowv.x);
            rowv.y = fma(w[i], v.y, rowv.y);
        }
        rw[jk * nW + (W0 - 1)] = rowv;
    }
    __syncthreads();
    double2* out = coarse.rhat + cn1 * (static_cast<unsigned>(W1) + cn1 * static_cast<unsigned>(W2));
    for (int W0 = 1 + threadIdx.x; W0 <= mc - 1; W0 += blockDim.x) {
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            double2 pl = make_double2(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < 5; ++j) {
                const double2 rowv = rw[(k * 5 + j) * nW + (W0 - 1)];
                pl.x = fma(w[j], rowv.x, pl.x);
                pl.y = fma(w[j], rowv.y, pl.y);
            }
            acc.x = fma(w[k], pl.x, acc.x);
            acc.y = fma(w[k], pl.y, acc.y);
        }
        out[W0] = acc;
        if (SMOOTH) {
            const int W[3] = {W0, W1, W2};
            smooth_interior<3>(sa, static_cast<unsigned>(W0) + cn1 * (static_cast<unsigned>(W1) + cn1 * static_cast<unsigned>(W2)), W, acc);
        }
    }
}

// ---- K3c: coarse smoothing on the restricted residual ------------------------
template <int P>
__global__ void __launch_bounds__(256) k_smooth_coarse(ResArgs a, unsigned fa, unsigned fb) {
    dev::griddep_wait();
    const Lvl& c = a.lv;
    for (unsigned f = fa + blockIdx.x * blockDim.x + threadIdx.x; f < fb; f += gridDim.x * blockDim.x) {
        int idx[P];
        dev::unflat<P>(f, c.n1, idx);
        if (a.bpx && c.si) {  // si = siNext (cycles.cpp:247); identically zero unless BPX
            c.si[f] = c.sinext[f];
            c.sinext[f] = make_double2(0.0, 0.0);
        }
        if (dev::on_boundary<P>(idx, static_cast<int>(c.m)) || c.level < a.ellMin) {
            c.sc[f] = make_double2(0.0, 0.0);
            continue;
        }
        const bool cp = dev::is_cpoint<P>(idx);
        const double2 smooth = mul(c.rhat[f], a.k.invDiag);
        c.sc[f] = stage(smooth, a.k.wRaw, cp, a.bpx, a.hb);
        if (a.bpx && c.level > a.ellMin && cp) {
            int wi[P];
#pragma unroll
            for (int d = 0; d < P; ++d) wi[d] = idx[d] / 3;
            a.par.sinext[dev::flat<P>(wi, a.par.n1)] = mul(a.k.wRaw, smooth);
        }
    }
}

constexpr int kZch = 48;

// ---- pyramid top-down (see fast.cuh) ---------------------------------------
// Threads (32, 8); the tile of level T is 32 x 8 x bz points (P = 3) or
// 32 x 8 bz (P = 2).  Box of level l-1 feeding box [lo, hi] of level l:
// [min(lo/3, m-1), min(hi/3, m-1) + 1] per axis (q = min(idx/3, m-1), q + 1).
constexpr int kPyrTX = 32, kPyrTY = 8;
// level-T points per thread (3D: 8 planes -- fewer CTAs share the ancestor work; measured 18.4 -> 16.5 us at 243^3)
template <int P>
__host__ __device__ constexpr int pyr_k() { return P == 3 ? 8 : 4; }

// lerp for rel in {0, 1, 2} (interior points; rel = 3 only on the top boundary),
// branch-free, bit-identical to lerp()
__device__ __forceinline__ double2 lerp012(double2 c0, double2 c1, int rel) {
    const double w1 = rel == 1 ? (1.0 / 3.0) : (2.0 / 3.0);
    const double2 v = make_double2(fma(w1, c1.x - c0.x, c0.x), fma(w1, c1.y - c0.y, c0.y));
    return rel == 0 ? c0 : v;
}

// P-linear prolongation from a box in shared memory (strides s1 = sz0, s2 = sz0 * sz1)
template <int P>
__device__ __forceinline__ double2 prolong_box(const double2* box, int s1, int s2, const int* q, const int* rel) {
    const double2* b = box + q[0] + s1 * q[1] + (P == 3 ? s2 * q[2] : 0);
    double2 v[1 << P];
#pragma unroll
    for (int e = 0; e < (1 << P); ++e) v[e] = b[(e & 1) + ((e >> 1) & 1) * s1 + (P == 3 ? ((e >> 2) & 1) * s2 : 0)];
#pragma unroll
    for (int d = 0; d < P; ++d)
#pragma unroll
        for (int i = 0; i < (1 << (P - 1 - d)); ++i) v[i] = lerp012(v[2 * i], v[2 * i + 1], rel[d]);
    return v[0];
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}

// Box loops: thread (tx, ty) walks x = tx (boxes are at most 32 wide), y = ty,
// ty + 8, ..., and (P = 3) every z.
template <int P>
__global__ void __launch_bounds__(kPyrTX* kPyrTY) k_topdown_pyr(const PyrArgs a) {
    dev::griddep_wait();
    extern __shared__ __align__(16) double2 pyr[];
    __shared__ int blo[kPyrMaxLevels][3], bsz[kPyrMaxLevels][3];
    __shared__ PyrLevel slv[kPyrMaxLevels];
    __shared__ int soff[kPyrMaxLevels], scap[kPyrMaxLevels];
    const int tid = threadIdx.x, tx = tid & (kPyrTX - 1), ty = tid / kPyrTX;
    const int T = a.T;
    // per-level parameters into shared memory in one parallel round: a
    // dynamically indexed kernel parameter is a serialised constant-cache miss
    if (tid <= T) {
        slv[tid] = a.lv[tid];
        soff[tid] = a.off[tid];
        scap[tid] = a.cap[tid];
    }
    __syncthreads();
    if (tid == 0) {
        int lo[3], hi[3];
        const int t0 = blockIdx.x % a.nbx, t1 = (blockIdx.x / a.nbx) % a.nby, t2 = blockIdx.x / (a.nbx * a.nby);
        const int ext[3] = {kPyrTX, P == 3 ? kPyrTY : kPyrTY * pyr_k<P>(), pyr_k<P>()};
        const int tl[3] = {t0, t1, t2};
        for (int d = 0; d < P; ++d) {
            lo[d] = tl[d] * ext[d];
            hi[d] = min(lo[d] + ext[d] - 1, slv[T].m);
            blo[T][d] = lo[d];
            bsz[T][d] = hi[d] - lo[d] + 1;
        }
        for (int l = T - 1; l >= 0; --l) {
            const int mp = slv[l].m;
            for (int d = 0; d < P; ++d) {
                lo[d] = min(lo[d] / 3, mp - 1);
                hi[d] = min(hi[d] / 3, mp - 1) + 1;
                blo[l][d] = lo[d];
                bsz[l][d] = hi[d] - lo[d] + 1;
            }
            if (P == 2) blo[l][2] = 0, bsz[l][2] = 1;
        }
        if (P == 2) blo[T][2] = 0, bsz[T][2] = 1;
    }
    __syncthreads();
    // (1) this thread's level-T points into registers (in flight during the pyramid)
    const PyrLevel LT = slv[T];
    double2 own[pyr_k<P>()];
    unsigned fo[pyr_k<P>()];
    const int gx = blo[T][0] + tx;
    const bool xin = tx < bsz[T][0] && gx > 0 && gx < LT.m;
#pragma unroll
    for (int k = 0; k < pyr_k<P>(); ++k) {
        const int gy = blo[T][1] + ty + (P == 2 ? kPyrTY * k : 0), gz = P == 3 ? blo[T][2] + k : 0;
        const bool in = xin && gy - blo[T][1] < bsz[T][1] && gy > 0 && gy < LT.m &&
                        (P == 2 || (k < bsz[T][2] && gz > 0 && gz < LT.m));
        fo[k] = in ? static_cast<unsigned>(gx) + static_cast<unsigned>(LT.n1) *
                         (static_cast<unsigned>(gy) + static_cast<unsigned>(LT.n1) * static_cast<unsigned>(gz))
                   : 0xffffffffu;
        own[k] = in ? ld(a.scTin + fo[k]) : make_double2(0.0, 0.0);
    }
    // (2) every ancestor box's sc (and si) into shared memory, all copies in flight at once
    for (int l = 0; l < T; ++l) {
        const PyrLevel L = slv[l];
        const int s0 = bsz[l][0], s1 = bsz[l][1], s2 = bsz[l][2];
        if (tx >= s0) continue;
        double2* td = pyr + soff[l];
        for (int z = 0; z < s2; ++z)
            for (int y = ty; y < s1; y += kPyrTY) {
                const unsigned f = static_cast<unsigned>(blo[l][0] + tx) +
                                   static_cast<unsigned>(L.n1) * (static_cast<unsigned>(blo[l][1] + y) +
                                                                  static_cast<unsigned>(L.n1) * static_cast<unsigned>(blo[l][2] + z));
                const int i = tx + s0 * (y + s1 * z);
                cp_async16(td + i, L.sc + f);
                if (a.bpx) cp_async16(td + scap[l] + i, L.si + f);
            }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    // (3) td_l = sc_l + P td_{l-1} (- P si_{l-1}) off the boundary, coarsest first, in place
    for (int l = 1; l < T; ++l) {
        const int m = slv[l].m, mp = slv[l - 1].m;
        const int s0 = bsz[l][0], s1 = bsz[l][1], s2 = bsz[l][2];
        const int p0 = bsz[l - 1][0], p1 = bsz[l - 1][1];
        double2* td = pyr + soff[l];
        const double2* ptd = pyr + soff[l - 1];
        const int g0 = blo[l][0] + tx;
        if (tx < s0 && g0 > 0 && g0 < m) {
            int q[3], rel[3];
            q[0] = min(g0 / 3, mp - 1);
            rel[0] = g0 - 3 * q[0];
            q[0] -= blo[l - 1][0];
            for (int z = 0; z < s2; ++z) {
                const int g2 = blo[l][2] + z;
                if (P == 3) {
                    if (g2 <= 0 || g2 >= m) continue;
                    q[2] = min(g2 / 3, mp - 1);
                    rel[2] = g2 - 3 * q[2];
                    q[2] -= blo[l - 1][2];
                }
                for (int y = ty; y < s1; y += kPyrTY) {
                    const int g1 = blo[l][1] + y;
                    if (g1 <= 0 || g1 >= m) continue;
                    q[1] = min(g1 / 3, mp - 1);
                    rel[1] = g1 - 3 * q[1];
                    q[1] -= blo[l - 1][1];
                    const int i = tx + s0 * (y + s1 * z);
                    double2 v = add(td[i], prolong_box<P>(ptd, p0, p0 * p1, q, rel));
                    const bool cp = rel[0] == 0 && rel[1] == 0 && (P == 2 || rel[2] == 0);
                    if (a.bpx && !cp) v = sub(v, prolong_box<P>(ptd + scap[l - 1], p0, p0 * p1, q, rel));
                    td[i] = v;
                }
            }
        }
        __syncthreads();
    }
    // (4) level T: the CTA's tile, in place
    const int mp = slv[T - 1].m;
    const double2* ptd = pyr + soff[T - 1];
    const int p0 = bsz[T - 1][0], p1 = bsz[T - 1][1];
    int q[3], rel[3];
    q[0] = min(gx / 3, mp - 1);
    rel[0] = gx - 3 * q[0];
    q[0] -= blo[T - 1][0];
#pragma unroll
    for (int k = 0; k < pyr_k<P>(); ++k) {
        if (fo[k] == 0xffffffffu) continue;
        const int gy = blo[T][1] + ty + (P == 2 ? kPyrTY * k : 0), gz = P == 3 ? blo[T][2] + k : 0;
        q[1] = min(gy / 3, mp - 1);
        rel[1] = gy - 3 * q[1];
        q[1] -= blo[T - 1][1];
        if (P == 3) {
            q[2] = min(gz / 3, mp - 1);
            rel[2] = gz - 3 * q[2];
            q[2] -= blo[T - 1][2];
        }
        double2 v = add(own[k], prolong_box<P>(ptd, p0, p0 * p1, q, rel));
        const bool cp = rel[0] == 0 && rel[1] == 0 && (P == 2 || rel[2] == 0);
        if (a.bpx && !cp) v = sub(v, prolong_box<P>(ptd + scap[T - 1], p0, p0 * p1, q, rel));
        a.scT[fo[k]] = v;
    }
}


// ---- coarse chains: every coarse level of one cycle phase in one launch -----
//
// The coarse levels of a cycle are a dependency chain of small passes
// (top-down l = 1..top, then smoothing + restriction top..1); as separate
// launches each costs a launch / drain of a few microseconds and dominated
// the cycle below 243^3.  One cooperative launch runs the whole chain with a
// grid barrier between levels.  Data produced inside the launch is read with
// ld.global.cg (L2), never through the non-coherent L1 / read-only path.
__device__ __forceinline__ double2 ldcg(const double2* p) { return __ldcg(p); }

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& gen, int cluster) {
    if (cluster) {  // the whole chain is one thread-block cluster: hardware cluster barrier
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        return;
    }
    if (gridDim.x == 1) {  // single-CTA chain: a block barrier suffices
        __threadfence_block();
        __syncthreads();
        return;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned target = gen + 1;
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicExch(bar + 1, target);
        } else {
            while (*reinterpret_cast<volatile unsigned*>(bar + 1) != target) __nanosleep(32);
        }
        __threadfence();
    }
    ++gen;
    __syncthreads();
}

template <int P>
__device__ __forceinline__ double2 prolong_cg(const double2* __restrict__ src, unsigned n1, const int* q,
                                              const int* rel) {
    double2 v[1 << P];
#pragma unroll
    for (int e = 0; e < (1 << P); ++e) {
        unsigned f = 0, s = 1;
#pragma unroll
        for (int d = 0; d < P; ++d) {
            f += static_cast<unsigned>(q[d] + ((e >> d) & 1)) * s;
            s *= n1;
        }
        v[e] = ldcg(src + f);
    }
#pragma unroll
    for (int d = 0; d < P; ++d)
#pragma unroll
        for (int i = 0; i < (1 << (P - 1 - d)); ++i) v[i] = lerp(v[2 * i], v[2 * i + 1], rel[d]);
    return v[0];
}

template <int P>
__global__ void __launch_bounds__(kChainThreads) k_chain_down(ChainArgs a) {
    unsigned gen = *reinterpret_cast<volatile unsigned*>(a.bar + 1);
    const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    for (int l = 1; l <= a.top; ++l) {
        const Lvl& c = a.lv[l];
        const Lvl& pr = a.lv[l - 1];
        for (unsigned f = tid; f < c.n; f += stride) {
            int idx[P];
            dev::unflat<P>(f, c.n1, idx);
            if (dev::on_boundary<P>(idx, static_cast<int>(c.m))) continue;
            int q[P], rel[P];
#pragma unroll
            for (int d = 0; d < P; ++d) {
                q[d] = min(idx[d] / 3, static_cast<int>(pr.m) - 1);
                rel[d] = idx[d] - 3 * q[d];
            }
            double2 sc = add(c.sc[f], prolong_cg<P>(pr.sc, pr.n1, q, rel));
            if (a.bpx && !dev::is_cpoint<P>(idx)) sc = sub(sc, prolong_at<P>(pr.si, pr.n1, q, rel));
            c.sc[f] = sc;
        }
        if (l < a.top) grid_barrier(a.bar, gen, a.cluster);
    }
}

// 3D: eight lanes per coarse vertex, lanes 0..4 each form one plane's 25-point
// partial, lane 0 combines them in plane order (the arithmetic of k_restrict),
// so the latency chain is 25 loads instead of 125 on the small levels.
__device__ __forceinline__ void chain_restrict3(const Lvl& fine, const Lvl& coarse, unsigned tid, unsigned stride) {
    const double w[5] = {1.0 / 3.0, 2.0 / 3.0, 1.0, 2.0 / 3.0, 1.0 / 3.0};
    const long long sy = fine.n1, sz = static_cast<long long>(fine.n1) * fine.n1;
    const unsigned lane = threadIdx.x & 31u, grp = lane >> 3, k = lane & 7u;
    const unsigned warp = tid >> 5, warps = stride >> 5;
    for (unsigned base = warp * 4u; base < coarse.n; base += warps * 4u) {
        const unsigned f = base + grp;
        int W[3] = {0, 0, 0};
        bool act = f < coarse.n;
        if (act) {
            dev::unflat<3>(f, coarse.n1, W);
            act = !dev::on_boundary<3>(W, static_cast<int>(coarse.m));
        }
        double2 pl = make_double2(0.0, 0.0);
        if (act && k < 5) {
            const double2* __restrict__ r =
                fine.rhat + (3LL * W[0] + sy * (3LL * W[1]) + sz * (3LL * W[2])) + (static_cast<int>(k) - 2) * sz;
#pragma unroll
            for (int j = 0; j < 5; ++j) {
                double2 row = make_double2(0.0, 0.0);
#pragma unroll
                for (int i = 0; i < 5; ++i) {
                    const double2 v = ldcg(r + (j - 2) * sy + (i - 2));
                    row.x = fma(w[i], v.x, row.x);
                    row.y = fma(w[i], v.y, row.y);
                }
                pl.x = fma(w[j], row.x, pl.x);
                pl.y = fma(w[j], row.y, pl.y);
            }
        }
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int kk = 0; kk < 5; ++kk) {
            const double px = __shfl_sync(0xffffffffu, pl.x, (grp << 3) + kk);
            const double py = __shfl_sync(0xffffffffu, pl.y, (grp << 3) + kk);
            acc.x = fma(w[kk], px, acc.x);
            acc.y = fma(w[kk], py, acc.y);
        }
        if (act && k == 0) coarse.rhat[f] = acc;
    }
}

template <int P>
__device__ __forceinline__ void chain_restrict(const Lvl& fine, const Lvl& coarse, unsigned tid, unsigned stride) {
    if (P == 3) {
        chain_restrict3(fine, coarse, tid, stride);
        return;
    }
    const double w[5] = {1.0 / 3.0, 2.0 / 3.0, 1.0, 2.0 / 3.0, 1.0 / 3.0};
    const long long sy = fine.n1, sz = static_cast<long long>(fine.n1) * fine.n1;
    for (unsigned f = tid; f < coarse.n; f += stride) {
        int W[P];
        dev::unflat<P>(f, coarse.n1, W);
        if (dev::on_boundary<P>(W, static_cast<int>(coarse.m))) continue;
        long long centre = 0, s = 1;
#pragma unroll
        for (int d = 0; d < P; ++d) {
            centre += 3LL * W[d] * s;
            s *= fine.n1;
        }
        const double2* __restrict__ r = fine.rhat + centre;
        double2 acc = make_double2(0.0, 0.0);
        if (P == 1) {
#pragma unroll
            for (int i = 0; i < 5; ++i) {
                const double2 v = ldcg(r + (i - 2));
                acc.x = fma(w[i], v.x, acc.x);
                acc.y = fma(w[i], v.y, acc.y);
            }
        } else if (P == 2) {
#pragma unroll
            for (int j = 0; j < 5; ++j) {
                double2 row = make_double2(0.0, 0.0);
#pragma unroll
                for (int i = 0; i < 5; ++i) {
                    const double2 v = ldcg(r + (j - 2) * sy + (i - 2));
                    row.x = fma(w[i], v.x, row.x);
                    row.y = fma(w[i], v.y, row.y);
                }
                acc.x = fma(w[j], row.x, acc.x);
                acc.y = fma(w[j], row.y, acc.y);
            }
        } else {
            double2 pl[5];
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                pl[k] = make_double2(0.0, 0.0);
#pragma unroll
                for (int j = 0; j < 5; ++j) {
                    double2 row = make_double2(0.0, 0.0);
#pragma unroll
                    for (int i = 0; i < 5; ++i) {
                        const double2 v = ldcg(r + (k - 2) * sz + (j - 2) * sy + (i - 2));
                        row.x = fma(w[i], v.x, row.x);
                        row.y = fma(w[i], v.y, row.y);
                    }
                    pl[k].x = fma(w[j], row.x, pl[k].x);
                    pl[k].y = fma(w[j], row.y, pl[k].y);
                }
            }
#pragma unroll
            for (int k = 0; k < 5; ++k) {
                acc.x = fma(w[k], pl[k].x, acc.x);
                acc.y = fma(w[k], pl[k].y, acc.y);
            }
        }
        coarse.rhat[f] = acc;
    }
}

template <int P>
__global__ void __launch_bounds__(kChainThreads) k_chain_up(ChainArgs a) {
    unsigned gen = *reinterpret_cast<volatile unsigned*>(a.bar + 1);
    const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    if (a.firstRestrict && a.top >= a.ellMin) {
        chain_restrict<P>(a.fine, a.lv[a.top], tid, stride);
        grid_barrier(a.bar, gen, a.cluster);
    }
    for (int l = a.top; l >= 1; --l) {
        const Lvl& c = a.lv[l];
        const Lvl& par = a.lv[l - 1];
        const LevelCoef& k = a.k[l];
        for (unsigned f = tid; f < c.n; f += stride) {  // smoothing (k_smooth_coarse)
            int idx[P];
            dev::unflat<P>(f, c.n1, idx);
            if (a.bpx && c.si) {
                c.si[f] = ldcg(c.sinext + f);
                c.sinext[f] = make_double2(0.0, 0.0);
            }
            if (dev::on_boundary<P>(idx, static_cast<int>(c.m)) || c.level < a.ellMin) {
                c.sc[f] = make_double2(0.0, 0.0);
                continue;
            }
            const bool cp = dev::is_cpoint<P>(idx);
            const double2 smooth = mul(ldcg(c.rhat + f), k.invDiag);
            c.sc[f] = stage(smooth, k.wRaw, cp, a.bpx, a.hb);
            if (a.bpx && c.level > a.ellMin && cp) {
                int wi[P];
#pragma unroll
                for (int d = 0; d < P; ++d) wi[d] = idx[d] / 3;
                par.sinext[dev::flat<P>(wi, par.n1)] = mul(k.wRaw, smooth);
            }
        }
        if (l - 1 >= 1 && l - 1 >= a.ellMin) chain_restrict<P>(c, par, tid, stride);  // into l-1, same step
        if (l > 1) grid_barrier(a.bar, gen, a.cluster);
    }
    if (a.normOut && blockIdx.x == 0) {  // K5: fixed-order reduction of the fine pass's block partials
        __shared__ double smax[kChainThreads], ssum[kChainThreads];
        double mx = 0.0, sm = 0.0;
        for (int i = threadIdx.x; i < a.normBlocks; i += blockDim.x) {
            mx = fmax(mx, a.normPartials[2 * i]);
            sm += a.normPartials[2 * i + 1];
        }
        smax[threadIdx.x] = mx;
        ssum[threadIdx.x] = sm;
        __syncthreads();
        for (int s = blockDim.x / 2; s > 0; s >>= 1) {
            if (threadIdx.x < s) {
                smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + s]);
                ssum[threadIdx.x] += ssum[threadIdx.x + s];
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            a.normOut[0] = smax[0];
            a.normOut[1] = ssum[0];
        }
    }
}


// ---- bottom-up helpers -------------------------------------------------------
template <int P>
__device__ __forceinline__ void smooth_point(const ChainArgs& a, const Lvl& c, const Lvl& par, const LevelCoef& k,
                                             unsigned f, double2 rh) {
    int idx[P];
    dev::unflat<P>(f, c.n1, idx);
    if (a.bpx && c.si) {
        c.si[f] = ldcg(c.sinext + f);
        c.sinext[f] = make_double2(0.0, 0.0);
    }
    if (dev::on_boundary<P>(idx, static_cast<int>(c.m)) || c.level < a.ellMin) {
        c.sc[f] = make_double2(0.0, 0.0);
        return;
    }
    const bool cp = dev::is_cpoint<P>(idx);
    const double2 smooth = mul(rh, k.invDiag);
    c.sc[f] = stage(smooth, k.wRaw, cp, a.bpx, a.hb);
    if (a.bpx && c.level > a.ellMin && cp) {
        int wi[P];
#pragma unroll
        for (int d = 0; d < P; ++d) wi[d] = idx[d] / 3;
        par.sinext[dev::flat<P>(wi, par.n1)] = mul(k.wRaw, smooth);
    }
}

// R r from a full level lattice in shared memory (chain_restrict's arithmetic)
template <int P>
__device__ __forceinline__ double2 restrict_from(const double2* r, unsigned n1) {
    const double w[5] = {1.0 / 3.0, 2.0 / 3.0, 1.0, 2.0 / 3.0, 1.0 / 3.0};
    const int sy = static_cast<int>(n1), sz = static_cast<int>(n1 * n1);
    double2 acc = make_double2(0.0, 0.0);
    if (P == 2) {
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            double2 row = make_double2(0.0, 0.0);
#pragma unroll
            for (int i = 0; i < 5; ++i) {
                const double2 v = r[(j - 2) * sy + (i - 2)];
                row.x = fma(w[i], v.x, row.x);
                row.y = fma(w[i], v.y, row.y);
            }
            acc.x = fma(w[j], row.x, acc.x);
            acc.y = fma(w[j], row.y, acc.y);
        }
    } else {
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            double2 pl = make_double2(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < 5; ++j) {
                double2 row = make_double2(0.0, 0.0);
#pragma unroll
                for (int i = 0; i < 5; ++i) {
                    const double2 v = r[(k - 2) * sz + (j - 2) * sy + (i - 2)];
                    row.x = fma(w[i], v.x, row.x);
                    row.y = fma(w[i], v.y, row.y);
                }
                pl.x = fma(w[j], row.x, pl.x);
                pl.y = fma(w[j], row.y, pl.y);
            }
            acc.x = fma(w[k], pl.x, acc.x);
            acc.y = fma(w[k], pl.y, acc.y);
        }
    }
    return acc;
}


// ---- bottom-up chain, cooperative form (see fast.cuh) ------------------------
// Step l (l = top .. 1): r_l = R r_{l+1} (source a.fine for l = top) and the
// smoothing of l on the value just formed, one grid barrier per step while
// the source level is big; once it has at most up_single<P>() points the CTA that
// arrives last at a counter runs the remaining steps alone in shared memory.
// Same arithmetic as restrict + k_chain_up, bit for bit.
#ifndef TMG_UP_SINGLE2
#define TMG_UP_SINGLE2 8000
#endif
template <int P>
__host__ __device__ constexpr unsigned up_single() { return P == 2 ? TMG_UP_SINGLE2 : 1200; }  // last-CTA source size (shared memory)

template <int P>
__device__ __forceinline__ void up_step_multi(const ChainArgs& a, const Lvl& src, const Lvl& c, const Lvl& par,
                                              const LevelCoef& k, bool restrictIt, unsigned tid, unsigned stride) {
    if (P == 3) {  // lane groups of 8 per coarse vertex (chain_restrict3), lane 0 smooths
        const double w[5] = {1.0 / 3.0, 2.0 / 3.0, 1.0, 2.0 / 3.0, 1.0 / 3.0};
        const long long sy = src.n1, sz = static_cast<long long>(src.n1) * src.n1;
        const unsigned lane = threadIdx.x & 31u, grp = lane >> 3, kk = lane & 7u;
        const unsigned warp = tid >> 5, warps = stride >> 5;
        for (unsigned base = warp * 4u; base < c.n; base += warps * 4u) {
            const unsigned f = base + grp;
            int W[3] = {0, 0, 0};
            bool act = f < c.n, interior = false;
            if (act) {
                dev::unflat<3>(f, c.n1, W);
                interior = !dev::on_boundary<3>(W, static_cast<int>(c.m));
            }
            double2 pl = make_double2(0.0, 0.0);
            if (restrictIt && act && interior && kk < 5) {
                const double2* __restrict__ r =
                    src.rhat + (3LL * W[0] + sy * (3LL * W[1]) + sz * (3LL * W[2])) + (static_cast<int>(kk) - 2) * sz;
#pragma unroll
                for (int j = 0; j < 5; ++j) {
                    double2 row = make_double2(0.0, 0.0);
#pragma unroll
                    for (int i = 0; i < 5; ++i) {
                        const double2 v = ldcg(r + (j - 2) * sy + (i - 2));
                        row.x = fma(w[i], v.x, row.x);
                        row.y = fma(w[i], v.y, row.y);
                    }
                    pl.x = fma(w[j], row.x, pl.x);
                    pl.y = fma(w[j], row.y, pl.y);
                }
            }
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                const double px = __shfl_sync(0xffffffffu, pl.x, (grp << 3) + q);
                const double py = __shfl_sync(0xffffffffu, pl.y, (grp << 3) + q);
                acc.x = fma(w[q], px, acc.x);
                acc.y = fma(w[q], py, acc.y);
            }
            if (act && kk == 0) {
                if (restrictIt && interior) c.rhat[f] = acc;
                smooth_point<3>(a, c, par, k, f, restrictIt ? acc : make_double2(0.0, 0.0));
            }
        }
    } else {
        for (unsigned f = tid; f < c.n; f += stride) {
            int W[P];
            dev::unflat<P>(f, c.n1, W);
            double2 acc = make_double2(0.0, 0.0);
            if (restrictIt && !dev::on_boundary<P>(W, static_cast<int>(c.m))) {
                unsigned centre = 0, s = 1;
#pragma unroll
                for (int d = 0; d < P; ++d) {
                    centre += 3u * static_cast<unsigned>(W[d]) * s;
                    s *= src.n1;
                }
                const double w[5] = {1.0 / 3.0, 2.0 / 3.0, 1.0, 2.0 / 3.0, 1.0 / 3.0};
                const double2* __restrict__ r = src.rhat + centre;
                const long long sy = src.n1;
                if (P == 1) {
#pragma unroll
                    for (int i = 0; i < 5; ++i) {
                        const double2 v = ldcg(r + (i - 2));
                        acc.x = fma(w[i], v.x, acc.x);
                        acc.y = fma(w[i], v.y, acc.y);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 5; ++j) {
                        double2 row = make_double2(0.0, 0.0);
#pragma unroll
                        for (int i = 0; i < 5; ++i) {
                            const double2 v = ldcg(r + (j - 2) * sy + (i - 2));
                            row.x = fma(w[i], v.x, row.x);
                            row.y = fma(w[i], v.y, row.y);
                        }
                        acc.x = fma(w[j], row.x, acc.x);
                        acc.y = fma(w[j], row.y, acc.y);
                    }
                }
                c.rhat[f] = acc;
            }
            smooth_point<P>(a, c, par, k, f, acc);
        }
    }
}

template <int NT>
__device__ __forceinline__ void chain_norms(const ChainArgs& a) {  // K5 (k_chain_up's tree and order)
    __shared__ double smax[NT], ssum[NT];
    double mx = 0.0, sm = 0.0;
    for (int i = threadIdx.x; i < a.normBlocks; i += NT) {
        mx = fmax(mx, a.normPartials[2 * i]);
        sm += a.normPartials[2 * i + 1];
    }
    smax[threadIdx.x] = mx;
    ssum[threadIdx.x] = sm;
    __syncthreads();
    for (int s = NT / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + s]);
            ssum[threadIdx.x] += ssum[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        a.normOut[0] = smax[0];
        a.normOut[1] = ssum[0];
    }
}

template <int P>
__global__ void __launch_bounds__(kChainThreads) k_up_coop(const ChainArgs a, unsigned* count) {
    dev::griddep_wait();
    extern __shared__ __align__(16) double2 us[];  // last CTA: r (and BPX si_next) of the small levels
    __shared__ unsigned lastFlag;
    unsigned gen = *reinterpret_cast<volatile unsigned*>(a.bar + 1);
    const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    const int top = a.top;
    // multi-CTA steps
    int l = top;
    for (; l >= 1; --l) {
        const Lvl src = l == top ? a.fine : a.lv[l + 1];
        if (src.n <= up_single<P>()) break;
        const bool restrictIt = l >= a.ellMin;
        up_step_multi<P>(a, src, a.lv[l], a.lv[l - 1], a.k[l], restrictIt, tid, stride);
        if (l > 1) {
            const Lvl nsrc = a.lv[l];
            if (nsrc.n > up_single<P>()) grid_barrier(a.bar, gen, 0);
        }
    }
    // the remaining steps: the CTA arriving last; norms: the one arriving first.
    // bar.sync orders the CTA's writes before thread 0's (cumulative) fence + arrival
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned arr = atomicAdd(count, 1u);
        lastFlag = arr == gridDim.x - 1 ? 1u : arr == 0 ? 2u : 0u;
        __threadfence();
    }
    __syncthreads();
    if (lastFlag == 2u || (lastFlag == 1u && gridDim.x == 1)) {
        if (a.normOut) chain_norms<kChainThreads>(a);
        if (gridDim.x > 1) return;
    }
    if (!lastFlag) return;
    if (l < 1) {
        if (threadIdx.x == 0) *count = 0u;
        return;
    }
    // shared memory: r of levels l+1 .. 1 (level l+1 = the source of the first step), si_next of l .. 1 (BPX)
    int offR[kMaxChainLevels + 1], offS[kMaxChainLevels + 1];
    {
        int o = 0;
        for (int j = l + 1; j >= 1; --j) {
            const unsigned n = j == top + 1 ? a.fine.n : a.lv[j].n;
            offR[j] = o;
            o += static_cast<int>(n);
            if (a.bpx && j <= l) {
                offS[j] = o;
                o += static_cast<int>(n);
            }
        }
    }
    {
        const Lvl src = l == top ? a.fine : a.lv[l + 1];
        for (unsigned f = threadIdx.x; f < src.n; f += blockDim.x) cp_async16(us + offR[l + 1] + f, src.rhat + f);
        if (a.bpx)
            for (int j = l; j >= 1; --j) {
                const Lvl c = a.lv[j];
                if (!c.si) continue;
                for (unsigned f = threadIdx.x; f < c.n; f += blockDim.x) cp_async16(us + offS[j] + f, c.sinext + f);
            }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
    }
    for (; l >= 1; --l) {
        const Lvl c = a.lv[l], par = a.lv[l - 1];
        const unsigned srcN1 = l == top ? a.fine.n1 : a.lv[l + 1].n1;
        const LevelCoef k = a.k[l];
        const double2* rsrc = us + offR[l + 1];
        double2* r = us + offR[l];
        const bool restrictIt = l >= a.ellMin;
        for (unsigned f = threadIdx.x; f < c.n; f += blockDim.x) {
            int idx[P];
            dev::unflat<P>(f, c.n1, idx);
            const bool bnd = dev::on_boundary<P>(idx, static_cast<int>(c.m));
            double2 acc = make_double2(0.0, 0.0);
            if (restrictIt && !bnd) {
                unsigned centre = 0, s = 1;
#pragma unroll
                for (int d = 0; d < P; ++d) {
                    centre += 3u * static_cast<unsigned>(idx[d]) * s;
                    s *= srcN1;
                }
                acc = restrict_from<P>(rsrc + centre, srcN1);
                c.rhat[f] = acc;
            }
            r[f] = acc;
            if (a.bpx && c.si) {
                c.si[f] = us[offS[l] + f];
                c.sinext[f] = make_double2(0.0, 0.0);
            }
            if (bnd || c.level < a.ellMin) {
                c.sc[f] = make_double2(0.0, 0.0);
                continue;
            }
            const bool cp = dev::is_cpoint<P>(idx);
            const double2 smooth = mul(acc, k.invDiag);
            c.sc[f] = stage(smooth, k.wRaw, cp, a.bpx, a.hb);
            if (a.bpx && c.level > a.ellMin && cp) {
                int wi[P];
#pragma unroll
                for (int d = 0; d < P; ++d) wi[d] = idx[d] / 3;
                const unsigned g = dev::flat<P>(wi, par.n1);
                const double2 v = mul(k.wRaw, smooth);
                par.sinext[g] = v;
                if (l - 1 >= 1 && par.si) us[offS[l - 1] + g] = v;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *count = 0u;  // re-arm for the next launch
}
}  // namespace

template <int P>
static int chain_grid_for(int smCount) {
    int perSm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&perSm, k_chain_up<P>, kChainThreads, 0);
    int perSm2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&perSm2, k_chain_down<P>, kChainThreads, 0);
    return std::max(1, std::min(std::min(perSm, perSm2), 2)) * smCount;
}

int chain_grid(int P, int smCount) {
    if (P == 1) return chain_grid_for<1>(smCount);
    if (P == 2) return chain_grid_for<2>(smCount);
    return chain_grid_for<3>(smCount);
}

namespace {
template <class K>
void launch_chain(K kernel, const ChainArgs& a, int grid, cudaStream_t s) {
    if (a.cluster) {  // one cluster of `grid` CTAs (<= 16), hardware barriers
        cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);  // per kernel
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kChainThreads);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = grid;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kernel, a);
        return;
    }
    void* args[] = {const_cast<ChainArgs*>(&a)};
    cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kernel), dim3(grid), dim3(kChainThreads), args, 0, s);
}
}  // namespace

void chain_down(int P, const ChainArgs& a, int grid, cudaStream_t s) {
    if (a.top < 1) return;
    if (P == 1) launch_chain(k_chain_down<1>, a, grid, s);
    else if (P == 2) launch_chain(k_chain_down<2>, a, grid, s);
    else launch_chain(k_chain_down<3>, a, grid, s);
}

void chain_up(int P, const ChainArgs& a, int grid, cudaStream_t s) {
    if (P == 1) launch_chain(k_chain_up<1>, a, grid, s);
    else if (P == 2) launch_chain(k_chain_up<2>, a, grid, s);
    else launch_chain(k_chain_up<3>, a, grid, s);
}


size_t up_coop_smem(int P, const ChainArgs& a) {
    const unsigned single = P == 2 ? up_single<2>() : up_single<3>();
    int l = a.top;
    for (; l >= 1; --l) {
        const unsigned n = l == a.top ? a.fine.n : a.lv[l + 1].n;
        if (n <= single) break;
    }
    if (l < 1) return 0;
    size_t pts = 0;
    for (int j = l + 1; j >= 1; --j) {
        const unsigned n = j == a.top + 1 ? a.fine.n : a.lv[j].n;
        pts += n * ((a.bpx && j <= l) ? 2u : 1u);
    }
    (void)P;
    return pts * sizeof(double2);
}

void up_coop(int P, const ChainArgs& a, unsigned* count, int smCount, cudaStream_t s) {
    const size_t smem = up_coop_smem(P, a);
    void* args[] = {const_cast<ChainArgs*>(&a), &count};
    const void* k = P == 1 ? reinterpret_cast<const void*>(k_up_coop<1>)
                    : P == 2 ? reinterpret_cast<const void*>(k_up_coop<2>)
                             : reinterpret_cast<const void*>(k_up_coop<3>);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int per = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, kChainThreads, smem) != cudaSuccess || per < 1) per = 1;
    // as many CTAs as the first (biggest) multi-CTA step has work for: fewer CTAs
    // contend less for the level parameters and arrive sooner at the counter
    const long long work = static_cast<long long>(a.lv[a.top].n) * (P == 3 ? 8 : 1);
    const int grid = static_cast<int>(std::max<long long>(
        1, std::min<long long>(std::min(per, 2) * smCount, (work + kChainThreads - 1) / kChainThreads)));
    cudaLaunchCooperativeKernel(k, dim3(grid), dim3(kChainThreads), args, smem, s);
}

int chain_cluster_size() {
    // the largest cluster the chain kernels can run as (16 needs the non-portable opt-in)
    cudaFuncSetAttribute(k_chain_up<3>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(kChainThreads);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_chain_up<3>, &cfg) == cudaSuccess && n >= 1) return 16;
    cudaGetLastError();
    return 8;
}

namespace {
// plane range [za, zb) of the last axis -> flat index range
void span(int P, const Lvl& v, int za, int zb, unsigned& fa, unsigned& fb) {
    if (za < 0) {
        fa = 0;
        fb = v.n;
        return;
    }
    unsigned plane = 1;
    for (int d = 0; d < P - 1; ++d) plane *= v.n1;
    fa = static_cast<unsigned>(za) * plane;
    fb = static_cast<unsigned>(std::min<long long>(zb, v.n1)) * plane;
    if (fb < fa) fb = fa;
}
}  // namespace

void correct_fine(int P, const Lvl& f, const Lvl& pr, int bpx, int blocks, cudaStream_t s) {
    if (P >= 2 && f.m >= 27) {  // parent-cell triples: 2^P parent loads shared by three points
        const unsigned rows = f.n / f.n1;
        if (P == 2) k_topdown_tri<2, true><<<blocks, 256, 0, s>>>(f, pr, bpx, 0u, rows);
        else k_topdown_tri<3, true><<<blocks, 256, 0, s>>>(f, pr, bpx, 0u, rows);
        return;
    }
    if (P == 1) k_topdown<1, true><<<blocks, 256, 0, s>>>(f, pr, bpx, 0u, f.n);
    else if (P == 2) k_topdown<2, true><<<blocks, 256, 0, s>>>(f, pr, bpx, 0u, f.n);
    else k_topdown<3, true><<<blocks, 256, 0, s>>>(f, pr, bpx, 0u, f.n);
}

size_t pyramid_setup(int P, PyrArgs& a, int T) {
    const int bz = P == 3 ? pyr_k<3>() : pyr_k<2>();
    a.T = T;
    a.bz = bz;
    const int n1 = a.lv[T].n1;
    const int ext[3] = {kPyrTX, P == 3 ? kPyrTY : kPyrTY * bz, bz};
    a.nbx = (n1 + ext[0] - 1) / ext[0];
    a.nby = (n1 + ext[1] - 1) / ext[1];
    // box extents: s_{l-1} <= ceil((s_l - 1) / 3) + 2, at most the level's n1
    int sz[3] = {ext[0], ext[1], ext[2]};
    int off = 0;
    for (int l = T - 1; l >= 0; --l) {
        int cap = 1;
        for (int d = 0; d < P; ++d) {
            sz[d] = std::min((sz[d] - 1 + 2) / 3 + 2, a.lv[l].n1);
            cap *= sz[d];
        }
        a.cap[l] = cap;
        a.off[l] = off;
        off += 2 * cap;  // td, si
    }
    return static_cast<size_t>(off) * sizeof(double2);
}

void topdown_pyramid(int P, const PyrArgs& a, size_t smem, cudaStream_t s) {
    const int n1 = a.lv[a.T].n1;
    const int nbz = P == 3 ? (n1 + a.bz - 1) / a.bz : 1;
    const unsigned blocks = static_cast<unsigned>(a.nbx) * a.nby * nbz;
    if (P == 2) {
        if (smem > 48 * 1024) cudaFuncSetAttribute(k_topdown_pyr<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        dev::launch_k(k_topdown_pyr<2>, dim3(blocks), dim3(kPyrTX * kPyrTY), smem, s, a);
    } else {
        if (smem > 48 * 1024) cudaFuncSetAttribute(k_topdown_pyr<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        dev::launch_k(k_topdown_pyr<3>, dim3(blocks), dim3(kPyrTX * kPyrTY), smem, s, a);
    }
}

void topdown_coarse(int P, const Lvl& c, const Lvl& pr, int bpx, int blocks, cudaStream_t s, int za, int zb) {
    if (P == 3 && c.m == 27) {  // row kernel: small levels, where per-thread latency dominated: interior planes of [za, zb)
        const int zlo = std::max(1, za < 0 ? 1 : za), zhi = std::min(static_cast<int>(c.m), za < 0 ? static_cast<int>(c.m) : zb);
        if (zhi <= zlo) return;
        const size_t smem = (bpx ? 8 : 4) * pr.n1 * sizeof(double2);
        dev::launch_k(k_topdown3_rows, dim3(c.m - 1, zhi - zlo), dim3(kRowThreads), smem, s, c, pr, bpx, zlo);
        return;
    }
    if (P >= 2 && c.m >= 243 && dev::switches().triCoarse) {  // big levels: parent-cell triples (k_topdown_tri)
        const unsigned plane = P == 3 ? c.n1 : 1u;  // rows per plane of the last axis
        const unsigned ra = za < 0 ? 0u : static_cast<unsigned>(za) * plane;
        const unsigned rb = za < 0 ? c.n / c.n1 : std::min<unsigned>(static_cast<unsigned>(zb) * plane, c.n / c.n1);
        if (rb <= ra) return;
        if (P == 2) dev::launch_k(k_topdown_tri<2, false>, dim3(blocks), dim3(256), 0, s, c, pr, bpx, ra, rb);
        else dev::launch_k(k_topdown_tri<3, false>, dim3(blocks), dim3(256), 0, s, c, pr, bpx, ra, rb);
        return;
    }
    unsigned fa, fb;
    span(P, c, za, zb, fa, fb);
    if (fb <= fa) return;
    if (P == 1) k_topdown<1, false><<<blocks, 256, 0, s>>>(c, pr, bpx, fa, fb);
    else if (P == 2) dev::launch_k(k_topdown<2, false>, dim3(blocks), dim3(256), 0, s, c, pr, bpx, fa, fb);
    else dev::launch_k(k_topdown<3, false>, dim3(blocks), dim3(256), 0, s, c, pr, bpx, fa, fb);
}

void load_vector(int P, const Lvl& F, const double2* f, double2 ms, int blocks, cudaStream_t s, int za, int zb) {
    if (P == 3) {
        const int m = static_cast<int>(F.m);
        const int zlo = std::max(1, za < 0 ? 1 : za), zhi = std::min(m, za < 0 ? m : zb);
        if (zhi <= zlo) return;
        dim3 grid((m - 1 + TX - 1) / TX, (m - 1 + TY - 1) / TY, (zhi - zlo + kZch - 1) / kZch);
        k_load3<<<grid, dim3(TX, TY), 0, s>>>(F, f, ms, zlo, zhi, kZch);
    } else if (P == 2) {
        k_load_lowdim<2><<<blocks, 256, 0, s>>>(F, f, ms);
    } else {
        k_load_lowdim<1><<<blocks, 256, 0, s>>>(F, f, ms);
    }
}

int residual_fine_blocks(int P, const Lvl& f, int smCount) {
    if (P == 3) {
        const int m = static_cast<int>(f.m);
        const int bx = (m - 1 + TX - 1) / TX, by = (m - 1 + TY - 1) / TY, bz = (m - 1 + kZch - 1) / kZch;
        return bx * by * bz;
    }
    const long long need = (static_cast<long long>(f.n) + 255) / 256;
    return static_cast<int>(std::max<long long>(1, std::min<long long>(need, 8LL * smCount)));
}

int residual_fine(int P, const ResArgs& a, int smCount, cudaStream_t s) {
    const int nb = residual_fine_blocks(P, a.lv, smCount);
    if (P == 3) {
        const int m = static_cast<int>(a.lv.m);
        dim3 grid((m - 1 + TX - 1) / TX, (m - 1 + TY - 1) / TY, (m - 1 + kZch - 1) / kZch);
        k_residual3<<<grid, dim3(TX, TY), 0, s>>>(a, kZch);
    } else if (P == 2) {
        k_residual_lowdim<2><<<nb, 256, 0, s>>>(a);
    } else {
        k_residual_lowdim<1><<<nb, 256, 0, s>>>(a);
    }
    return nb;
}

void restrict_level(int P, const Lvl& fine, const Lvl& coarse, const double*, int blocks, cudaStream_t s, int za,
                    int zb, const ResArgs* smooth) {
    const ResArgs sa = smooth ? *smooth : ResArgs{};
    if (P == 3 && coarse.m == 27) {  // small levels only (big ones are faster grid-stride)
        const int zlo = std::max(1, za < 0 ? 1 : za);
        const int zhi = std::min(static_cast<int>(coarse.m), za < 0 ? static_cast<int>(coarse.m) : zb);
        if (zhi <= zlo) return;
        const size_t smem = 25 * (coarse.m - 1) * sizeof(double2);
        if (smooth) dev::launch_k(k_restrict3_rows<true>, dim3(coarse.m - 1, zhi - zlo), dim3(kRowThreads), smem, s, fine, coarse, zlo, sa);
        else dev::launch_k(k_restrict3_rows<false>, dim3(coarse.m - 1, zhi - zlo), dim3(kRowThreads), smem, s, fine, coarse, zlo, sa);
        return;
    }
    unsigned fa, fb;
    span(P, coarse, za, zb, fa, fb);
    if (fb <= fa) return;
    if (smooth) {
        if (P == 1) dev::launch_k(k_restrict<1, true>, dim3(blocks), dim3(256), 0, s, fine, coarse, fa, fb, sa);
        else if (P == 2) dev::launch_k(k_restrict<2, true>, dim3(blocks), dim3(256), 0, s, fine, coarse, fa, fb, sa);
        else dev::launch_k(k_restrict<3, true>, dim3(blocks), dim3(256), 0, s, fine, coarse, fa, fb, sa);
        return;
    }
    if (P == 1) dev::launch_k(k_restrict<1>, dim3(blocks), dim3(256), 0, s, fine, coarse, fa, fb, sa);
    else if (P == 2) dev::launch_k(k_restrict<2>, dim3(blocks), dim3(256), 0, s, fine, coarse, fa, fb, sa);
    else dev::launch_k(k_restrict<3>, dim3(blocks), dim3(256), 0, s, fine, coarse, fa, fb, sa);
}

void smooth_coarse(int P, const ResArgs& a, int blocks, cudaStream_t s, int za, int zb) {
    unsigned fa, fb;
    span(P, a.lv, za, zb, fa, fb);
    if (fb <= fa) return;
    if (P == 1) dev::launch_k(k_smooth_coarse<1>, dim3(blocks), dim3(256), 0, s, a, fa, fb);
    else if (P == 2) dev::launch_k(k_smooth_coarse<2>, dim3(blocks), dim3(256), 0, s, a, fa, fb);
    else dev::launch_k(k_smooth_coarse<3>, dim3(blocks), dim3(256), 0, s, a, fa, fb);
}

}  // namespace fast
}  // namespace tmg
