// Verification cycles on regular trees: the bottom-up FAS
// V-cycle `bu_fas` (proj/src/cycles.cpp:374-603), the textbook additive
// correction cycle `textbook_add` (cycles.cpp:605-714) and the leaf-level
// residual evaluation `evaluate_residual_norms` (cycles.cpp:716-786), as
// level passes on the device hierarchy's exact storage (u, sc, sf, si, chi,
// u-hat at every level).
//
// The reference sums these cycles' cell contributions and restrictions in
// hash-map iteration order (for_each_cell_at / for_each_vertex_at), which is
// not a traversal order, so they are evaluated here with the assembled class
// stencil and FMA like the fast precision: parity is the tolerance gate of
// the fast path (tests/test_gpu_vcycles.py), not bit-identity.

#include "vcycles.cuh"

#include <algorithm>

namespace tmg {
namespace vc {

using dev::Lvl;

namespace {

__device__ __forceinline__ double2 z2() { return make_double2(0.0, 0.0); }
__device__ __forceinline__ double2 add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 mul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 mac(double2 acc, double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, acc.x)), fma(a.x, b.y, fma(a.y, b.x, acc.y)));
}
__device__ __forceinline__ double2 lerp(double2 c0, double2 c1, int rel) {
    if (rel == 0) return c0;
    if (rel == 3) return c1;
    const double w1 = rel == 1 ? (1.0 / 3.0) : (2.0 / 3.0);
    return make_double2(fma(w1, c1.x - c0.x, c0.x), fma(w1, c1.y - c0.y, c0.y));
}

// H x at an interior vertex: assembled stencil, one coefficient per class
template <int P>
__device__ __forceinline__ double2 apply_h(const double2* __restrict__ x, unsigned f, unsigned n1,
                                           const fast::LevelCoef& k) {
    double2 acc[4] = {z2(), z2(), z2(), z2()};
    const int NB = P == 1 ? 3 : P == 2 ? 9 : 27;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
        int off = 0, cls = 0, stride = 1;
#pragma unroll
        for (int d = 0; d < P; ++d) {
            const int del = (j / (d == 0 ? 1 : d == 1 ? 3 : 9)) % 3 - 1;
            off += del * stride;
            cls += del != 0 ? 1 : 0;
            stride *= static_cast<int>(n1);
        }
        acc[cls] = add(acc[cls], __ldg(x + (static_cast<int>(f) + off)));
    }
    double2 h = mul(k.c[0], acc[0]);
#pragma unroll
    for (int c = 1; c <= P; ++c) h = mac(h, k.c[c], acc[c]);
    return h;
}

// parent-stencil prolongation of `src` (level l-1) at fine index idx
template <int P>
__device__ __forceinline__ double2 prolong_from(const double2* __restrict__ src, const Lvl& pr, const int* idx) {
    int q[P], rel[P];
#pragma unroll
    for (int d = 0; d < P; ++d) {
        q[d] = min(idx[d] / 3, static_cast<int>(pr.m) - 1);
        rel[d] = idx[d] - 3 * q[d];
    }
    double2 v[1 << P];
#pragma unroll
    for (int e = 0; e < (1 << P); ++e) {
        int pi[P];
#pragma unroll
        for (int d = 0; d < P; ++d) pi[d] = q[d] + ((e >> d) & 1);
        v[e] = src[dev::flat<P>(pi, pr.n1)];
    }
#pragma unroll
    for (int d = 0; d < P; ++d)
#pragma unroll
        for (int i = 0; i < (1 << (P - 1 - d)); ++i) v[i] = lerp(v[2 * i], v[2 * i + 1], rel[d]);
    return v[0];
}

#define VC_LOOP(c)                                                                                    \
    for (unsigned f = blockIdx.x * blockDim.x + threadIdx.x; f < (c).n; f += gridDim.x * blockDim.x)

// out = b - H x on interior vertices (b may be null: - H x), 0 on the boundary
template <int P>
__global__ void k_residual(Lvl c, const double2* x, const double2* b, double2* out, fast::LevelCoef k) {
    VC_LOOP(c) {
        int idx[P];
        dev::unflat<P>(f, c.n1, idx);
        if (dev::on_boundary<P>(idx, static_cast<int>(c.m))) {
            out[f] = z2();
            continue;
        }
        const double2 hx = apply_h<P>(x, f, c.n1, k);
        out[f] = b ? sub(b[f], hx) : make_double2(-hx.x, -hx.y);
    }
}

// textbook: u += omega r / diag on interior vertices
template <int P>
__global__ void k_jacobi(Lvl c, const double2* r, double2 w, fast::LevelCoef k) {
    VC_LOOP(c) {
        int idx[P];
        dev::unflat<P>(f, c.n1, idx);
        if (dev::on_boundary<P>(idx, static_cast<int>(c.m))) continue;
        c.u[f] = add(c.u[f], mul(w, mul(r[f], k.invDiag)));
    }
}

// bu_fas smoother staging: sc = omega_of(succ, cPoint) r / diag (0 on the boundary)
template <int P>
__global__ void k_stage(Lvl c, const double2* r, double2 wNonCp, double2 wCp, fast::LevelCoef k) {
    VC_LOOP(c) {
        int idx[P];
        dev::unflat<P>(f, c.n1, idx);
        const double2 w = dev::is_cpoint<P>(idx) && c.level > 0 ? wCp : wNonCp;
        if (dev::on_boundary<P>(idx, static_cast<int>(c.m)) || (w.x == 0.0 && w.y == 0.0)) {
            c.sc[f] = z2();
            continue;
        }
        c.sc[f] = mul(w, mul(r[f], k.invDiag));
    }
}

// bu_fas injection refresh of level l-1 (cycles.cpp:440-456)
template <int P>
__global__ void k_inject(Lvl c, Lvl fine) {
    VC_LOOP(c) {
        int idx[P];
        dev::unflat<P>(f, c.n1, idx);
        int fi[P];
#pragma unroll
        for (int d = 0; d < P; ++d) fi[d] = 3 * idx[d];
        const unsigned ff = dev::flat<P>(fi, fine.n1);
        const double2 u = fine.u[ff];
        c.u[f] = u;
        c.sf[f] = u;
        c.si[f] = fine.sc[ff];
    }
}

// u-hat = u - P u_{l-1} (0 on the boundary)
template <int P>
__global__ void k_uhat(Lvl c, Lvl pr) {
    VC_LOOP(c) {
        int idx[P];
        dev::unflat<P>(f, c.n1, idx);
        c.uhat[f] = dev::on_boundary<P>(idx, static_cast<int>(c.m)) ? z2() : sub(c.u[f], prolong_from<P>(pr.u, pr, idx));
    }
}

// chi_{l-1} = R vals_l (interior coarse vertices; 5^P gather, separable weights)
template <int P>
__global__ void k_restrict(Lvl fine, const double2* vals, Lvl c) {
    const double w[5] = {1.0 / 3.0, 2.0 / 3.0, 1.0, 2.0 / 3.0, 1.0 / 3.0};
    VC_LOOP(c) {
        int W[P];
        dev::unflat<P>(f, c.n1, W);
        if (dev::on_boundary<P>(W, static_cast<int>(c.m))) {
            c.chi[f] = z2();
            continue;
        }
        double2 acc = z2();
        const int NB = P == 1 ? 5 : P == 2 ? 25 : 125;
        for (int j = 0; j < NB; ++j) {
            int v[P];
            double wt = 1.0;
            int jj = j;
#pragma unroll
            for (int d = 0; d < P; ++d) {
                const int o = jj % 5;
                jj /= 5;
                v[d] = 3 * W[d] + o - 2;
                wt *= w[o];
            }
            const double2 x = vals[dev::flat<P>(v, fine.n1)];
            acc = make_double2(fma(wt, x.x, acc.x), fma(wt, x.y, acc.y));
        }
        c.chi[f] = acc;
    }
}

// textbook upward: u_l += omegaCG P u_{l-1} (interior)
template <int P>
__global__ void k_prolong_add(Lvl c, Lvl pr, double2 w) {
    VC_LOOP(c) {
        int idx[P];
        dev::unflat<P>(f, c.n1, idx);
        if (dev::on_boundary<P>(idx, static_cast<int>(c.m))) continue;
        c.u[f] = add(c.u[f], mul(w, prolong_from<P>(pr.u, pr, idx)));
    }
}

// bu_fas upward: upd = sc + P(u - sf - [bpx] si)_{l-1}; u += upd; si_next = upd
template <int P>
__global__ void k_bu_up(Lvl c, Lvl pr, int coarse, int bpx) {
    VC_LOOP(c) {
        int idx[P];
        dev::unflat<P>(f, c.n1, idx);
        if (dev::on_boundary<P>(idx, static_cast<int>(c.m))) {
            if (c.sinext) c.sinext[f] = z2();
            continue;
        }
        double2 upd = c.sc[f];
        if (coarse) {
            int q[P], rel[P];
#pragma unroll
            for (int d = 0; d < P; ++d) {
                q[d] = min(idx[d] / 3, static_cast<int>(pr.m) - 1);
                rel[d] = idx[d] - 3 * q[d];
            }
            double2 v[1 << P];
#pragma unroll
            for (int e = 0; e < (1 << P); ++e) {
                int pi[P];
#pragma unroll
                for (int d = 0; d < P; ++d) pi[d] = q[d] + ((e >> d) & 1);
                const unsigned pf = dev::flat<P>(pi, pr.n1);
                double2 t = sub(pr.u[pf], pr.sf[pf]);
                if (bpx) t = sub(t, pr.si[pf]);
                v[e] = t;
            }
#pragma unroll
            for (int d = 0; d < P; ++d)
#pragma unroll
                for (int i = 0; i < (1 << (P - 1 - d)); ++i) v[i] = lerp(v[2 * i], v[2 * i + 1], rel[d]);
            upd = add(upd, v[0]);
        }
        c.u[f] = add(c.u[f], upd);
        if (c.sinext) c.sinext[f] = upd;  // si_next: the cycle's correction (hanging interpolation only)
    }
}

// norms of r over the interior of the level
template <int P>
__global__ void __launch_bounds__(256) k_norms(Lvl c, const double2* r, double* partials) {
    double mx = 0.0, sm = 0.0;
    VC_LOOP(c) {
        int idx[P];
        dev::unflat<P>(f, c.n1, idx);
        if (dev::on_boundary<P>(idx, static_cast<int>(c.m))) continue;
        const double m2 = fma(r[f].x, r[f].x, r[f].y * r[f].y);
        mx = fmax(mx, m2);
        sm += m2;
    }
    dev::block_norms(mx, sm, partials);
}

__global__ void k_norm_sum(const double* __restrict__ partials, int nb, double* out) {
    __shared__ double smax[256], ssum[256];
    double mx = 0.0, sm = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        mx = fmax(mx, partials[2 * i]);
        sm += partials[2 * i + 1];
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
        out[0] = smax[0];
        out[1] = ssum[0];
    }
}

int nblocks(unsigned n, int smCount) {
    const long long need = (static_cast<long long>(n) + 255) / 256;
    return static_cast<int>(std::max<long long>(1, std::min<long long>(need, 32LL * smCount)));
}

template <int P>
void residual_norms(const Ctx& x, double* out2) {
    const Lvl& F = x.lv[x.L];
    const int nb = nblocks(F.n, x.smCount);
    k_residual<P><<<nb, 256, 0, x.stream>>>(F, F.u, F.chi, x.r[x.L], x.fc[x.L]);
    k_norms<P><<<nb, 256, 0, x.stream>>>(F, x.r[x.L], x.partials);
    k_norm_sum<<<1, 256, 0, x.stream>>>(x.partials, nb, x.dNorm);
    cudaMemcpyAsync(out2, x.dNorm, 2 * sizeof(double), cudaMemcpyDeviceToHost, x.stream);
    cudaStreamSynchronize(x.stream);
}

template <int P>
void textbook(const Ctx& x, double2 wS, double2 wCG) {
    for (int l = x.L; l >= x.ellMin; --l) {
        const Lvl& c = x.lv[l];
        const int nb = nblocks(c.n, x.smCount);
        k_residual<P><<<nb, 256, 0, x.stream>>>(c, c.u, c.chi, x.r[l], x.fc[l]);
        k_jacobi<P><<<nb, 256, 0, x.stream>>>(c, x.r[l], wS, x.fc[l]);
        if (l > x.ellMin) {
            const Lvl& cc = x.lv[l - 1];
            cudaMemsetAsync(cc.u, 0, static_cast<size_t>(cc.n) * sizeof(double2), x.stream);
            k_restrict<P><<<nblocks(cc.n, x.smCount), 256, 0, x.stream>>>(c, x.r[l], cc);
        }
    }
    for (int l = x.ellMin + 1; l <= x.L; ++l)
        k_prolong_add<P><<<nblocks(x.lv[l].n, x.smCount), 256, 0, x.stream>>>(x.lv[l], x.lv[l - 1], wCG);
}

template <int P>
void bufas(const Ctx& x, const double2* wNonCp, const double2* wCp, int bpx) {
    for (int l = x.L; l >= x.ellMin; --l) {
        const Lvl& c = x.lv[l];
        const int nb = nblocks(c.n, x.smCount);
        k_residual<P><<<nb, 256, 0, x.stream>>>(c, c.u, c.chi, x.r[l], x.fc[l]);
        k_stage<P><<<nb, 256, 0, x.stream>>>(c, x.r[l], wNonCp[l], wCp[l], x.fc[l]);
        if (l == x.ellMin) break;
        const Lvl& cc = x.lv[l - 1];
        k_inject<P><<<nblocks(cc.n, x.smCount), 256, 0, x.stream>>>(cc, c);
        k_uhat<P><<<nb, 256, 0, x.stream>>>(c, cc);
        k_residual<P><<<nb, 256, 0, x.stream>>>(c, c.uhat, c.chi, x.r[l], x.fc[l]);  // r-hat
        k_restrict<P><<<nblocks(cc.n, x.smCount), 256, 0, x.stream>>>(c, x.r[l], cc);
    }
    for (int l = x.ellMin; l <= x.L; ++l)
        k_bu_up<P><<<nblocks(x.lv[l].n, x.smCount), 256, 0, x.stream>>>(x.lv[l], x.lv[l - 1], l > x.ellMin ? 1 : 0,
                                                                            bpx);
}

}  // namespace

void textbook_add(int P, const Ctx& x, double2 wS, double2 wCG) {
    if (P == 1) textbook<1>(x, wS, wCG);
    else if (P == 2) textbook<2>(x, wS, wCG);
    else textbook<3>(x, wS, wCG);
}

void bu_fas(int P, const Ctx& x, const double2* wNonCp, const double2* wCp, int bpx) {
    if (P == 1) bufas<1>(x, wNonCp, wCp, bpx);
    else if (P == 2) bufas<2>(x, wNonCp, wCp, bpx);
    else bufas<3>(x, wNonCp, wCp, bpx);
}

void residual_norms(int P, const Ctx& x, double* out2) {
    if (P == 1) residual_norms<1>(x, out2);
    else if (P == 2) residual_norms<2>(x, out2);
    else residual_norms<3>(x, out2);
}

}  // namespace vc
}  // namespace tmg
