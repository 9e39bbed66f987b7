// Device hierarchy + cycle kernels (sm_100a).  See hierarchy.hpp and
// DESIGN.md §3 for the data layout and the kernel/roofline table.
//
// Cycle = two level passes (reference
// proj/src/oracle.cpp:465-509 with the per-vertex semantics of
// proj/src/cycles.cpp:102-303):
//   top-down  l = 1..L   K1 k_topdown           touch_first  (cycles.cpp:102-141)
//   bottom-up l = L..1   K2/K3 k_residual_exact enterCell + touchLast (cycles.cpp:173-303)
//                        K3r k_restrict_exact   restriction into chi_{l-1} (cycles.cpp:292-301)
//   norms                K5 k_norm_final        (cycles.cpp:248-258, 94-97)
// The fast-precision fine pass (K2f) lives in fast.cuh.

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "amr.hpp"
#include "exact_ops.cuh"
#include "fast.cuh"
#include "fused2.cuh"
#include "fused3.cuh"
#include "hierarchy.hpp"
#include "vcycles.cuh"
#include "lattice.cuh"

namespace tmg {

#define TMG_CUDA(call)                                                                          \
    do {                                                                                        \
        cudaError_t err_ = (call);                                                              \
        if (err_ != cudaSuccess) {                                                              \
            if (err_ == cudaErrorMemoryAllocation)                                              \
                throw CapacityError(std::string("device memory exhausted: ") + #call);          \
            throw CudaError(std::string("CUDA error ") + cudaGetErrorString(err_) + " at " + #call); \
        }                                                                                       \
    } while (0)

namespace dev {

struct ResArgs {
    Lvl lv;
    Lvl par;  // level l-1 (injection targets); unused when l <= ellMin
    LevelConst k;
    int ellMin;
    int isFine;
    int bpx;
    int hb;
    double* partials;  // 2 doubles per block: max |r|^2, sum |r|^2
};

// ---- K1: top-down update (touch_first, cycles.cpp:102-141) ----------------
template <int P>
__global__ void __launch_bounds__(256) k_topdown(Lvl c, Lvl pr, int bpx) {
    // The parent cell is taken as q = idx / 3 with rel = idx % 3 in {0, 1, 2}: at the upper
    // boundary parent_stencil's (q - 1, rel 3) names the same corner q as (q, rel 0).  An
    // axis with rel 0 reads its lower corner twice (stride 0) and copies it exactly
    // (transfer.cpp:20-40), so the interpolation needs one exact-copy select, not two.
    // The lattice index is split by multiply-high with M = ceil(2^64 / n1) (exact for
    // 32-bit operands) instead of divisions.  Values and operation order are unchanged.
    const unsigned n1 = c.n1, pn1 = pr.n1;
    const unsigned long long M = ~0ull / n1 + 1ull;
    for (unsigned f = blockIdx.x * blockDim.x + threadIdx.x; f < c.n; f += gridDim.x * blockDim.x) {
        int idx[P];
        {
            unsigned r = f;
#pragma unroll
            for (int d = 0; d + 1 < P; ++d) {
                const unsigned qd = static_cast<unsigned>(__umul64hi(M, r));
                idx[d] = static_cast<int>(r - qd * n1);
                r = qd;
            }
            idx[P - 1] = static_cast<int>(r);
        }
        int rel[P];
        unsigned p0 = 0, ps = 1, str[P];
#pragma unroll
        for (int d = 0; d < P; ++d) {
            const int q = idx[d] / 3;
            rel[d] = idx[d] - 3 * q;
            p0 += static_cast<unsigned>(q) * ps;
            str[d] = rel[d] ? ps : 0u;
            ps *= pn1;
        }
        // one field at a time (register footprint): P sc, P si (BPX), P u
        auto parent_prolong = [&](const double2* __restrict__ src) {
            double2 v[1 << P];
#pragma unroll
            for (int e = 0; e < (1 << P); ++e) {
                unsigned o = p0;
#pragma unroll
                for (int d = 0; d < P; ++d) o += ((e >> d) & 1) ? str[d] : 0u;
                v[e] = src[o];
            }
#pragma unroll
            for (int d = 0; d < P; ++d) {
                const double w0 = rel[d] == 1 ? (2.0 / 3.0) : (1.0 / 3.0);
                const double w1 = rel[d] == 1 ? (1.0 / 3.0) : (2.0 / 3.0);
#pragma unroll
                for (int k = 0; k < (1 << (P - 1 - d)); ++k) {
                    const double2 r = xadd(xscale(w0, v[2 * k]), xscale(w1, v[2 * k + 1]));  // lerp_rel
                    v[k] = rel[d] == 0 ? v[2 * k] : r;
                }
            }
            return v[0];
        };
        double2 sc = xadd(c.sc[f], parent_prolong(pr.sc));
        if (bpx && !is_cpoint<P>(idx)) sc = xsub(sc, parent_prolong(pr.si));
        const double2 sf = c.sf ? c.sf[f] : cz();
        double2 u = xadd(c.u[f], xadd(sc, sf));
        double2 uh = xsub(u, parent_prolong(pr.u));
        if (on_boundary<P>(idx, static_cast<int>(c.m))) {
            u = cz();
            uh = cz();
        }
        c.u[f] = u;
        c.sc[f] = sc;
        c.uhat[f] = uh;
        if (c.sf) c.sf[f] = cz();
    }
}

// Element-by-element residual -(A x) gathered at one interior vertex, with the
// cell contributions summed in traversal order (see exact_ops.cuh rule (1)).
// Products A_s x_{v+delta} are formed once and shared by the cells using them
// (A depends only on the XOR pattern of the corner pair); iterating delta in
// lexicographic order visits every cell's corners b in ascending order, the
// order of proj/src/kernels.cpp:42-47.
template <int P, int ID>
__device__ __forceinline__ double2 ordered_sum(const double2 (&S)[1 << P]) {
    double2 r = xneg(S[perm_cell(P, ID, 0)]);
#pragma unroll
    for (int i = 1; i < (1 << P); ++i) r = xsub(r, S[perm_cell(P, ID, i)]);
    return r;
}

template <int P>
__device__ __forceinline__ double2 element_residual(const double2* __restrict__ x, unsigned f, unsigned n1,
                                                    const double2 (&A)[8], int pid) {
    constexpr int NC = 1 << P;
    int pw[P];
    pw[0] = 1;
#pragma unroll
    for (int d = 1; d < P; ++d) pw[d] = pw[d - 1] * 3;
    double2 S[NC];
#pragma unroll
    for (int j = 0; j < (P == 1 ? 3 : P == 2 ? 9 : 27); ++j) {
        int del[P];
        int off = 0, s = 0, stride = 1;
#pragma unroll
        for (int d = 0; d < P; ++d) {
            del[d] = (j / (d == 0 ? 1 : d == 1 ? 3 : 9)) % 3 - 1;
            off += del[d] * stride;
            stride *= static_cast<int>(n1);
            s |= (del[d] != 0 ? 1 : 0) << d;
        }
        const double2 prod = xmul(A[s], __ldg(x + (static_cast<int>(f) + off)));
#pragma unroll
        for (int e = 0; e < NC; ++e) {
            bool use = true;
            int b = 0;
#pragma unroll
            for (int d = 0; d < P; ++d) {
                const int bd = del[d] - ((e >> d) & 1) + 1;
                use &= (bd == 0 || bd == 1);
                b |= (bd & 1) << d;
            }
            if (use) S[e] = (b == 0) ? prod : xadd(S[e], prod);
        }
    }
    (void)pw;
    if (P == 1) return ordered_sum<P, 0>(S);
    if (P == 2) return pid == 0 ? ordered_sum<P, 0>(S) : ordered_sum<P, (P >= 2 ? 1 : 0)>(S);
    switch (pid) {
        case 0: return ordered_sum<P, 0>(S);
        case 1: return ordered_sum<P, (P >= 3 ? 1 : 0)>(S);
        case 2: return ordered_sum<P, (P >= 3 ? 2 : 0)>(S);
        case 3: return ordered_sum<P, (P >= 3 ? 3 : 0)>(S);
        case 4: return ordered_sum<P, (P >= 3 ? 4 : 0)>(S);
        default: return ordered_sum<P, (P >= 3 ? 5 : 0)>(S);
    }
}

// Multichannel element residual (kernels.cpp:39-59): per cell, the own
// channel's products over b, then for every other channel j (ascending) the
// coupling products (A_ij massScale mas(a,b)) x_j,b, all in the cell's corner
// order; the cells are combined in traversal order as above.
template <int P>
__device__ __forceinline__ double2 element_residual_mc(const double2* const* __restrict__ xs, int nch, int own,
                                                       unsigned f, unsigned n1, const double2 (&A)[8],
                                                       const double2 (&Mc)[8], int pid) {
    constexpr int NC = 1 << P;
    constexpr int NB = P == 1 ? 3 : P == 2 ? 9 : 27;
    double2 S[NC];
    for (int pass = -1; pass < nch; ++pass) {  // pass -1: own channel; then j = 0..nch-1, j != own
        if (pass == own) continue;
        const double2* __restrict__ x = xs[pass < 0 ? own : pass];
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            int del[P];
            int off = 0, s = 0, stride = 1;
#pragma unroll
            for (int d = 0; d < P; ++d) {
                del[d] = (j / (d == 0 ? 1 : d == 1 ? 3 : 9)) % 3 - 1;
                off += del[d] * stride;
                stride *= static_cast<int>(n1);
                s |= (del[d] != 0 ? 1 : 0) << d;
            }
            const double2 prod = xmul(pass < 0 ? A[s] : Mc[s], __ldg(x + (static_cast<int>(f) + off)));
#pragma unroll
            for (int e = 0; e < NC; ++e) {
                bool use = true;
                int b = 0;
#pragma unroll
                for (int d = 0; d < P; ++d) {
                    const int bd = del[d] - ((e >> d) & 1) + 1;
                    use &= (bd == 0 || bd == 1);
                    b |= (bd & 1) << d;
                }
                if (use) S[e] = (pass < 0 && b == 0) ? prod : xadd(S[e], prod);
            }
        }
    }
    if (P == 1) return ordered_sum<P, 0>(S);
    if (P == 2) return pid == 0 ? ordered_sum<P, 0>(S) : ordered_sum<P, (P >= 2 ? 1 : 0)>(S);
    switch (pid) {
        case 0: return ordered_sum<P, 0>(S);
        case 1: return ordered_sum<P, (P >= 3 ? 1 : 0)>(S);
        case 2: return ordered_sum<P, (P >= 3 ? 2 : 0)>(S);
        case 3: return ordered_sum<P, (P >= 3 ? 3 : 0)>(S);
        case 4: return ordered_sum<P, (P >= 3 ? 4 : 0)>(S);
        default: return ordered_sum<P, (P >= 3 ? 5 : 0)>(S);
    }
}

// ---- K2/K3: residual + Jacobi staging + injections (enterCell/touchLast) --
#ifndef TMG_EXACT_RES_MINB
#define TMG_EXACT_RES_MINB 3
#endif
// Coupled channels (ResArgs::mc): the other channels' u / u-hat of this level.
struct McArgs {
    const double2* const* u;
    const double2* const* uhat;
    int nch, own;
    double2 Mc[8];  // A_ij massScale mas(pattern)
};

template <int P, bool MC>
__global__ void __launch_bounds__(256, TMG_EXACT_RES_MINB) k_residual_exact(ResArgs a, McArgs mc) {
    const Lvl& c = a.lv;
    double nmax = 0.0, nsum = 0.0;
    for (unsigned f = blockIdx.x * blockDim.x + threadIdx.x; f < c.n; f += gridDim.x * blockDim.x) {
        int idx[P];
        unflat<P>(f, c.n1, idx);
        const bool bnd = on_boundary<P>(idx, static_cast<int>(c.m));
        const bool cp = is_cpoint<P>(idx);
        double2 r = cz(), rh = cz();
        if (!bnd) {
            const int pid = perm_id<P>(idx);
            if (MC) {
                r = element_residual_mc<P>(mc.u, mc.nch, mc.own, f, c.n1, a.k.A, mc.Mc, pid);
                rh = element_residual_mc<P>(mc.uhat, mc.nch, mc.own, f, c.n1, a.k.A, mc.Mc, pid);
            } else {
                r = element_residual<P>(c.u, f, c.n1, a.k.A, pid);
                rh = element_residual<P>(c.uhat, f, c.n1, a.k.A, pid);
            }
            const double2 chi = c.chi[f];
            r = xadd(chi, r);    // finish_vertex, kernels.cpp:96-97
            rh = xadd(chi, rh);
        }
        if (c.si) {  // si = siNext (cycles.cpp:247); siNext re-zeroed for the next sweep
            c.si[f] = c.sinext[f];
            c.sinext[f] = cz();
        }
        if (a.isFine && !bnd) {
            const double m2 = r.x * r.x + r.y * r.y;
            nmax = fmax(nmax, m2);
            nsum += m2;
        }
        if (c.r) c.r[f] = r;
        c.rhat[f] = rh;
        if (c.level < a.ellMin) {
            c.sc[f] = cz();
            continue;
        }
        const double2 smooth = bnd ? cz() : divdc3(r.x, r.y, a.k.div);
        double2 sc;
        if (a.bpx) {
            sc = cp ? cz() : xmul(a.k.wRaw, smooth);
        } else {
            const bool wz = (a.hb && cp) || xzero(a.k.wRaw);
            sc = wz ? cz() : xmul(a.k.wRaw, smooth);
        }
        c.sc[f] = sc;
        if (c.level > a.ellMin && cp) {  // injections, cycles.cpp:279-291
            int wi[P];
#pragma unroll
            for (int d = 0; d < P; ++d) wi[d] = idx[d] / 3;
            const unsigned wf = flat<P>(wi, a.par.n1);
            const double2 sf = c.sf ? c.sf[f] : cz();
            a.par.sf[wf] = xadd(sf, sc);
            if (a.bpx) a.par.sinext[wf] = xmul(a.k.wRaw, smooth);
        }
    }
    if (a.isFine) block_norms(nmax, nsum, a.partials);
}

// ---- K2/K3 for cell-varying operators (gaussian scenario, problems.cpp:20-24,
// 78-90): the cell matrix A_c (per XOR pattern) and the per-vertex diagonal are
// taken cell by cell in traversal order, the Jacobi division with the
// diagonal's own __divdc3 constants.
template <int P>
__global__ void __launch_bounds__(256) k_residual_cells(ResArgs a, const double2* __restrict__ cellA) {
    constexpr int NC = 1 << P;
    const Lvl& c = a.lv;
    const int m = static_cast<int>(c.m);
    double nmax = 0.0, nsum = 0.0;
    for (unsigned f = blockIdx.x * blockDim.x + threadIdx.x; f < c.n; f += gridDim.x * blockDim.x) {
        int idx[P];
        unflat<P>(f, c.n1, idx);
        const bool bnd = on_boundary<P>(idx, m);
        const bool cp = is_cpoint<P>(idx);
        const int pid = perm_id<P>(idx);
        double2 r = cz(), rh = cz(), dg = cz();
        bool first = true;
        for (int i = 0; i < NC; ++i) {
            const int e = perm_cell(P, pid, i);
            int cell[P];
            bool ok = true;
#pragma unroll
            for (int d = 0; d < P; ++d) {
                cell[d] = idx[d] - 1 + ((e >> d) & 1);
                ok &= (cell[d] >= 0) & (cell[d] <= m - 1);
            }
            if (!ok) continue;
            unsigned cf = 0, s = 1;
#pragma unroll
            for (int d = 0; d < P; ++d) {
                cf += static_cast<unsigned>(cell[d]) * s;
                s *= static_cast<unsigned>(m);
            }
            const double2* A = cellA + static_cast<size_t>(cf) * NC;
            const int ca = (~e) & (NC - 1);
            double2 sr = cz(), sh = cz();
#pragma unroll
            for (int bb = 0; bb < NC; ++bb) {
                int vb[P];
#pragma unroll
                for (int d = 0; d < P; ++d) vb[d] = cell[d] + ((bb >> d) & 1);
                const unsigned vf = flat<P>(vb, c.n1);
                const double2 pu = xmul(A[ca ^ bb], c.u[vf]);
                const double2 ph = xmul(A[ca ^ bb], c.uhat[vf]);
                sr = bb == 0 ? pu : xadd(sr, pu);
                sh = bb == 0 ? ph : xadd(sh, ph);
            }
            if (first) {
                r = xneg(sr);
                rh = xneg(sh);
                dg = A[0];
                first = false;
            } else {
                r = xsub(r, sr);
                rh = xsub(rh, sh);
                dg = xadd(dg, A[0]);
            }
        }
        if (bnd) {
            r = cz();
            rh = cz();
        } else {
            const double2 chi = c.chi[f];
            r = xadd(chi, r);
            rh = xadd(chi, rh);
        }
        if (c.si) {
            c.si[f] = c.sinext[f];
            c.sinext[f] = cz();
        }
        if (a.isFine && !bnd) {
            const double m2 = r.x * r.x + r.y * r.y;
            nmax = fmax(nmax, m2);
            nsum += m2;
        }
        if (c.r) c.r[f] = r;
        c.rhat[f] = rh;
        if (c.level < a.ellMin) {
            c.sc[f] = cz();
            continue;
        }
        const double2 smooth = bnd ? cz() : divdc3(r.x, r.y, div_const_dev(dg.x, dg.y));
        double2 sc;
        if (a.bpx) {
            sc = cp ? cz() : xmul(a.k.wRaw, smooth);
        } else {
            const bool wz = (a.hb && cp) || xzero(a.k.wRaw);
            sc = wz ? cz() : xmul(a.k.wRaw, smooth);
        }
        c.sc[f] = sc;
        if (c.level > a.ellMin && cp) {
            int wi[P];
#pragma unroll
            for (int d = 0; d < P; ++d) wi[d] = idx[d] / 3;
            const unsigned wf = flat<P>(wi, a.par.n1);
            const double2 sf = c.sf ? c.sf[f] : cz();
            a.par.sf[wf] = xadd(sf, sc);
            if (a.bpx) a.par.sinext[wf] = xmul(a.k.wRaw, smooth);
        }
    }
    if (a.isFine) block_norms(nmax, nsum, a.partials);
}

// ---- K3r: restriction chi_{l-1} = R rhat_l in touch-last order -------------
// table: for each permutation id, 5^P offsets (packed base 5) in order.
template <int P>
__global__ void __launch_bounds__(256) k_restrict_exact(Lvl fine, Lvl coarse, const unsigned char* __restrict__ table,
                                                        const double* __restrict__ weights, int zero) {
    constexpr int NT = P == 1 ? 5 : P == 2 ? 25 : 125;
    constexpr int NP = P == 1 ? 1 : P == 2 ? 2 : 6;
    __shared__ unsigned char st[NP * NT];
    __shared__ double sw[NT];
    for (int i = threadIdx.x; i < NP * NT; i += blockDim.x) st[i] = table[i];
    for (int i = threadIdx.x; i < NT; i += blockDim.x) sw[i] = weights[i];
    __syncthreads();
    for (unsigned f = blockIdx.x * blockDim.x + threadIdx.x; f < coarse.n; f += gridDim.x * blockDim.x) {
        if (zero) {
            coarse.chi[f] = cz();
            continue;
        }
        int W[P];
        unflat<P>(f, coarse.n1, W);
        const int pid = perm_id<P>(W);
        double2 acc = cz();
        const int mf = static_cast<int>(fine.m);
        // loads in batches of (up to) 25 independent addresses, then the ordered
        // sum: the touch-last order stays sequential, the latency chain does not
        constexpr int NB = NT < 25 ? NT : 25;
        for (int i0 = 0; i0 < NT; i0 += NB) {
            double2 vals[NB];
            double wts[NB];
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                const int c0 = st[pid * NT + i0 + b];
                int code = c0;
                int v[P];
                bool in = true;
#pragma unroll
                for (int d = 0; d < P; ++d) {
                    v[d] = 3 * W[d] + (code % 5) - 2;
                    code /= 5;
                    in &= (v[d] >= 1) & (v[d] <= mf - 1);
                }
                wts[b] = in ? sw[c0] : 0.0;
                vals[b] = in ? fine.rhat[flat<P>(v, fine.n1)] : cz();
            }
#pragma unroll
            for (int b = 0; b < NB; ++b)
                if (wts[b] != 0.0) acc = xadd(acc, xscale(wts[b], vals[b]));
        }
        coarse.chi[f] = acc;
    }
}

// ---- K5: deterministic final norm reduction --------------------------------
__global__ void k_norm_final(const double* __restrict__ partials, int nblocks, double* out) {
    __shared__ double smax[1024], ssum[1024];
    double mx = 0.0, sm = 0.0;
    for (int i = threadIdx.x; i < nblocks; i += blockDim.x) {
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

// ---- K6: setup kernels -------------------------------------------------------
// Consistent-mass load of the leaf cells (kernels.cpp:69-87), accumulated per
// vertex in traversal cell order; constant across sweeps on a static grid.
template <int P>
__global__ void k_load_vector(Lvl c, const double2* __restrict__ chiNodal, LevelConst k, unsigned fa, unsigned fb,
                              const double2* __restrict__ cellMs) {
    for (unsigned f = fa + blockIdx.x * blockDim.x + threadIdx.x; f < fb; f += gridDim.x * blockDim.x) {
        int idx[P];
        unflat<P>(f, c.n1, idx);
        // permutation: boundary axes carry a single cell, any priority works
        const int pid = perm_id<P>(idx);
        double2 b = cz();
#pragma unroll
        for (int i = 0; i < (1 << P); ++i) {
            int e = 0;
            if (P == 1) e = perm_cell(1, 0, i);
            else if (P == 2) e = pid == 0 ? perm_cell(2, 0, i) : perm_cell(2, 1, i);
            else {
#pragma unroll
                for (int id = 0; id < 6; ++id)
                    if (id == pid) e = perm_cell(3, id, i);
            }
            int cell[P];
            bool ok = true;
#pragma unroll
            for (int d = 0; d < P; ++d) {
                cell[d] = idx[d] - 1 + ((e >> d) & 1);
                ok &= (cell[d] >= 0) & (cell[d] <= static_cast<int>(c.m) - 1);
            }
            if (!ok) continue;
            const int a = (~e) & ((1 << P) - 1);  // corner of the vertex in the cell
            double2 acc = cz();
#pragma unroll
            for (int bb = 0; bb < (1 << P); ++bb) {
                int vb[P];
#pragma unroll
                for (int d = 0; d < P; ++d) vb[d] = cell[d] + ((bb >> d) & 1);
                acc = xadd(acc, xscale(k.M[a ^ bb], chiNodal[flat<P>(vb, c.n1)]));
            }
            double2 ms = k.massScale;
            if (cellMs) {  // per-cell massScale (cell-varying theta)
                unsigned cf = 0, st = 1;
#pragma unroll
                for (int d = 0; d < P; ++d) {
                    cf += static_cast<unsigned>(cell[d]) * st;
                    st *= c.m;
                }
                ms = cellMs[cf];
            }
            b = xadd(b, xmul(ms, acc));
        }
        c.chi[f] = b;
    }
}

// Seeded nodal rhs f(x) keyed on the finest-lattice position,
// optionally masked to the ball |x - 1/2|^2 < 0.04.
template <int P>
__global__ void k_seeded_chi(double2* out, unsigned fa, unsigned n, unsigned n1, unsigned long long seed, int scale,
                             long long mkey, int sphere, int channel) {  // flat indices [fa, n)
    for (unsigned f = fa + blockIdx.x * blockDim.x + threadIdx.x; f < n; f += gridDim.x * blockDim.x) {
        int idx[P];
        unflat<P>(f, n1, idx);
        unsigned long long key = 0;
        long long s2 = 0;
#pragma unroll
        for (int d = 0; d < P; ++d) {
            const long long fi = static_cast<long long>(idx[d]) * scale;
            key |= static_cast<unsigned long long>(static_cast<unsigned short>(fi)) << (16 * d);
            const long long t = 2 * fi - mkey;
            s2 += t * t;
        }
        if (sphere && !(25 * s2 < 4 * mkey * mkey)) {
            out[f] = cz();
            continue;
        }
        const unsigned long long s = seed ^ (static_cast<unsigned long long>(channel) << 48) ^ key;
        out[f] = make_double2(unit_rand(s), unit_rand(s ^ 0x5bf03635ull));
    }
}

template <int P>
__global__ void k_random_fine(Lvl c, unsigned long long seed, int channel = 0) {  // cycles.cpp:812-840
    for (unsigned f = blockIdx.x * blockDim.x + threadIdx.x; f < c.n; f += gridDim.x * blockDim.x) {
        int idx[P];
        unflat<P>(f, c.n1, idx);
        if (on_boundary<P>(idx, static_cast<int>(c.m))) {
            c.u[f] = cz();
            continue;
        }
        unsigned long long key = 0;
#pragma unroll
        for (int d = 0; d < P; ++d) key |= static_cast<unsigned long long>(static_cast<unsigned short>(idx[d])) << (16 * d);
        const unsigned long long base = seed ^ (static_cast<unsigned long long>(c.level) << 56) ^
                                        (static_cast<unsigned long long>(channel) << 48) ^ key;
        c.u[f] = make_double2(unit_rand(base), unit_rand(base ^ 0x5bf03635ull));
    }
}

// u_l(W) = u_{l+1}(3W) on non-boundary vertices (injection consistency).
template <int P>
__global__ void k_inject_u(Lvl c, Lvl fine, int fineVForm) {
    for (unsigned f = blockIdx.x * blockDim.x + threadIdx.x; f < c.n; f += gridDim.x * blockDim.x) {
        int idx[P];
        unflat<P>(f, c.n1, idx);
        if (on_boundary<P>(idx, static_cast<int>(c.m))) continue;
        int fi[P];
#pragma unroll
        for (int d = 0; d < P; ++d) fi[d] = 3 * idx[d];
        const unsigned ff = flat<P>(fi, fine.n1);
        c.u[f] = fineVForm ? make_double2(fine.u[ff].x - fine.sc[ff].x, fine.u[ff].y - fine.sc[ff].y) : fine.u[ff];
    }
}

// complex64 fine level (precision = fast-complex64): conversions to / from complex128
__global__ void k_f2d(const float2* __restrict__ in, double2* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = make_double2(in[i].x, in[i].y);
}
__global__ void k_d2f(const double2* __restrict__ in, float2* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = make_float2(static_cast<float>(in[i].x), static_cast<float>(in[i].y));
}
// u = v - sc of a complex64 v-form fine level, as complex128
__global__ void k_vform_f2d(const float2* __restrict__ v, const float2* __restrict__ sc, double2* __restrict__ out,
                            size_t n) {
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = make_double2(static_cast<double>(v[i].x) - sc[i].x, static_cast<double>(v[i].y) - sc[i].y);
}

// sc-free fused pass: sc = v - u with the derived u (fused3::derive_u), on [fa, fb)
template <class S2>
__global__ void k_split_derived(S2* __restrict__ v, S2* __restrict__ sc, const double2* __restrict__ u, unsigned fa,
                                unsigned fb, int toU) {  // toU: v <- u as well
    using R = decltype(S2::x);
    for (unsigned f = fa + blockIdx.x * blockDim.x + threadIdx.x; f < fb; f += gridDim.x * blockDim.x) {
        const S2 vf = v[f];
        sc[f] = S2{static_cast<R>(vf.x - u[f].x), static_cast<R>(vf.y - u[f].y)};
        if (toU) v[f] = S2{static_cast<R>(u[f].x), static_cast<R>(u[f].y)};
    }
}

// v-form fine level (fused3.cuh): u = v - sc, in place
__global__ void k_vform_to_u(double2* v, const double2* sc, size_t n) {
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        v[i] = make_double2(v[i].x - sc[i].x, v[i].y - sc[i].y);
}

// Fine interior values (interior lattice order) scattered into the level.
template <int P>
__global__ void k_scatter_interior(Lvl c, const double2* __restrict__ in) {
    for (unsigned f = blockIdx.x * blockDim.x + threadIdx.x; f < c.n; f += gridDim.x * blockDim.x) {
        int idx[P];
        unflat<P>(f, c.n1, idx);
        if (on_boundary<P>(idx, static_cast<int>(c.m))) continue;
        unsigned fl = 0, s = 1;
#pragma unroll
        for (int d = 0; d < P; ++d) {
            fl += static_cast<unsigned>(idx[d] - 1) * s;
            s *= c.m - 1;
        }
        c.u[f] = in[fl];
    }
}

// FMG unfolding: new finest level u = P u_{coarse} (spacetree.cpp:245-270).
template <int P>
__global__ void k_prolong_new(Lvl c, Lvl pr, unsigned fa, unsigned fb) {  // flat indices [fa, fb)
    for (unsigned f = fa + blockIdx.x * blockDim.x + threadIdx.x; f < fb; f += gridDim.x * blockDim.x) {
        int idx[P];
        unflat<P>(f, c.n1, idx);
        int q[P], rel[P];
#pragma unroll
        for (int d = 0; d < P; ++d) {
            q[d] = min(idx[d] / 3, static_cast<int>(pr.m) - 1);
            rel[d] = idx[d] - 3 * q[d];
        }
        double2 cu[1 << P];
#pragma unroll
        for (int e = 0; e < (1 << P); ++e) {
            int pi[P];
#pragma unroll
            for (int d = 0; d < P; ++d) pi[d] = q[d] + ((e >> d) & 1);
            cu[e] = pr.u[flat<P>(pi, pr.n1)];
        }
        c.u[f] = prolong<P>(cu, rel);
    }
}

__global__ void k_test_divdc3(const double2* x, const DivConst* k, double2* out, long long n) {
    for (long long i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = divdc3(x[i].x, x[i].y, k[i]);
}

__global__ void k_flush(double4* buf, size_t n, double v) {
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        buf[i] = make_double4(v, v, v, v);
}

}  // namespace dev

// ============================================================================
// Host side
// ============================================================================

namespace {

int pow3i(int l) {
    int r = 1;
    for (int i = 0; i < l; ++i) r *= 3;
    return r;
}

// proj/src/elemops.cpp:13-18
Cplx cplx_ipow(Cplx z, int e) {
    if (e < 0) return 1.0 / cplx_ipow(z, -e);
    Cplx r = 1.0;
    for (int i = 0; i < e; ++i) r *= z;
    return r;
}

// proj/src/elemops.cpp:29-55, entries for corner pair (0, s): every pair with
// the same XOR pattern has identical entries (per-axis equal/unequal only).
void reference_pattern(int p, int s, double& lap, double& mas) {
    static const double kLap1[2][2] = {{1.0, -1.0}, {-1.0, 1.0}};
    static const double kMass1[2][2] = {{1.0 / 3.0, 1.0 / 6.0}, {1.0 / 6.0, 1.0 / 3.0}};
    const int a = 0, b = s;
    double mass = 1.0;
    for (int d = 0; d < p; ++d) mass *= kMass1[(a >> d) & 1][(b >> d) & 1];
    double l = 0.0;
    for (int d = 0; d < p; ++d) {
        double t = kLap1[(a >> d) & 1][(b >> d) & 1];
        for (int i = 0; i < p; ++i)
            if (i != d) t *= kMass1[(a >> i) & 1][(b >> i) & 1];
        l += t;
    }
    lap = l;
    mas = mass;
}

// libgcc __divdc3 branch structure for a fixed divisor (see exact_ops.cuh).
dev::DivConst div_const(Cplx diag) {
    dev::DivConst k{};
    double c = diag.real(), d = diag.imag();
    const bool swap = !(std::fabs(c) < std::fabs(d));
    k.swap = swap ? 1 : 0;
    const double big = swap ? std::fabs(c) : std::fabs(d);
    k.pre = 0;
    if (big >= dev::kRBIG) {
        c = c / 2;
        d = d / 2;
        k.pre = 1;
    }
    const double big2 = swap ? std::fabs(c) : std::fabs(d);
    if (big2 < dev::kRMIN2) {
        c = c * dev::kRMINSCAL;
        d = d * dev::kRMINSCAL;
        k.pre = k.pre == 1 ? 1 : 2;  // halving and scaling up are exclusive
    }
    k.c = c;
    k.d = d;
    if (!swap) {
        k.ratio = c / d;
        k.denom = (c * k.ratio) + d;
        k.denomTiny = ((c * dev::kRMINSCAL) * k.ratio) + (d * dev::kRMINSCAL);
    } else {
        k.ratio = d / c;
        k.denom = (d * k.ratio) + c;
        k.denomTiny = ((d * dev::kRMINSCAL) * k.ratio) + (c * dev::kRMINSCAL);
    }
    k.sub = std::fabs(k.ratio) > dev::kRMIN ? 0 : 1;
    return k;
}

}  // namespace

Cplx omega_unmasked(const Policy& pol, int succ, int n) {
    Cplx ws = pol.omegaS;
    if (pol.twoPhase) {  // cycles.cpp:11-15
        const Cplx w1 = 0.01 * Cplx(std::sqrt(3.0), -1.0);
        ws = (n % 2 == 1) ? w1 : -std::conj(w1);
    }
    switch (pol.kind) {
        case OmegaKind::JacobiOnly: return succ == 0 ? ws : Cplx(0.0);
        case OmegaKind::UndampedCG: return ws;
        case OmegaKind::LGrid: return succ <= pol.lGrid ? ws : Cplx(0.0);
        case OmegaKind::Exponential: return cplx_ipow(ws, succ + 1);
        case OmegaKind::Transition: {
            const double e = (1.0 - 1.0 / static_cast<double>(n)) * (succ + 1);
            if (e == 0.0) return Cplx(1.0);
            return std::pow(ws, e);
        }
    }
    return Cplx(0.0);
}

struct Hierarchy::Impl {
    Problem prob;
    int p = 2, L = 1;
    std::vector<dev::Lvl> lv;
    std::vector<void*> allocations;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, evf0 = nullptr, evf1 = nullptr;
    double* partials = nullptr;
    int normBlocks = 0;
    double* dNorm = nullptr;
    double* hNorm = nullptr;  // pinned
    unsigned char* restrictTable = nullptr;
    double* restrictWeights = nullptr;
    double2* chiNodal = nullptr;  // device nodal rhs at the finest lattice
    double4* flushBuf = nullptr;
    size_t flushN = 0;
    std::vector<dev::LevelConst> kc;  // per level (exact)
    std::vector<fast::LevelCoef> fc;  // per level (fast)
    std::vector<Cplx> diagInterior;
    std::vector<Cplx> lapScale, massScale;
    bool debugR = false;
    int smCount = 148;
    float lastFineMs = 0.f, lastTdMs = 0.f;
    bool timeFine = false;
    bool coarseUStale = false;
    // fused 3D fine pass (fast precision): double-buffered fine u / sc
    bool fused = false;
    double2* uAlt = nullptr;
    CUtensorMap mapU[2];  // v: [0] current buffer, [1] alternate
    CUtensorMap mapC, mapI;  // coarse sc / si planes (L-1)
    CUtensorMap mapB;        // fine load vector b (the fused pass's b tiles)
    fused3::Geometry geo{};
    double2* partial3 = nullptr;
    std::unique_ptr<AmrTree> amr;  // static adaptive tree (prob.sphereLevels > 0)
    std::vector<double2*> vcScratch;  // verification cycles: per-level residual
    std::vector<double2*> cellA, cellMs;  // gaussian scenario: per-cell operator / massScale
    std::vector<std::vector<dev::Lvl>> chanLv;  // channels 1.. (exact storage)
    std::vector<const double2**> chanU, chanUh;  // per level: device arrays of every channel's u / u-hat
    std::vector<std::array<double2, 8>> couplingM;  // per level: A_ij massScale mas(pattern)
    bool fused2on = false;         // 2D fused fine pass (fast precision)
    fused2::Geometry geo2{};
    double2* partial2 = nullptr;
    int chainGrid = 0;              // cooperative coarse-chain grid (0: per-level launches)
#ifndef TMG_CHAIN_MAXN
#define TMG_CHAIN_MAXN (1u << 16)
#endif
    static constexpr unsigned kChainMaxN = TMG_CHAIN_MAXN;  // levels below this size join the chain
    int fusedResident = 4 * 148;  // replaced by fused3::resident_blocks at construction
    bool fineFused = false;  // the fine level runs a fused pass (decided before allocation)
    // sc-free fine pass (3D fused td-add, fused3::derive_u): the level L-1 top-down values the
    // last pass prolonged (the planes of a slab), and whether the fine (u, sc) must be derived
    double2* scTD = nullptr;
    double2* siTD = nullptr;  // td-bpx: level L-1 si as the pass read it
    bool fineDerived = false, derivedBpx = false;
    // z-slab member (prob.slabLo >= 0): allocated plane ranges [za, zb) of levels L and L-1
    int zaF = 0, zbF = 0, zaC = 0, zbC = 0;
    bool slab() const { return prob.slabLo >= 0; }
    // the fine lattice's allocated flat index range
    std::pair<unsigned, unsigned> fine_flat_range() const {
        const dev::Lvl& F = lv[L];
        if (!slab()) return {0u, F.n};
        const unsigned plane = F.n1 * F.n1;
        return {static_cast<unsigned>(zaF) * plane, static_cast<unsigned>(zbF) * plane};
    }
    // bytes per fine-level element: complex64 storage (precision = fast-complex64) or complex128
    size_t fine_elem() const { return prob.c64 ? sizeof(float2) : sizeof(double2); }
    // a transient complex128 array of the fine lattice (complex64 conversions)
    struct Tmp {
        double2* p = nullptr;
        ~Tmp() {
            if (p) cudaFree(p);
        }
    };
    // complex64 hierarchies convert on their hot paths (the load vector of every new right-hand
    // side, field export): they keep one stand-in for the hierarchy's lifetime instead of a
    // cudaMalloc / cudaFree of the whole lattice per call (6.2 GB at 729^3); complex128
    // hierarchies (and slab members, which must stay at 1 / N of the memory) allocate transiently
    double2* tmpFineKept = nullptr;
    double2* tmp_fine(Tmp& t) {
        const size_t bytes = static_cast<size_t>(lv[L].n) * sizeof(double2);
        double2* p = nullptr;
        if (prob.c64) {
            if (!tmpFineKept) tmpFineKept = alloc<double2>(lv[L].n);
            p = tmpFineKept;
        } else {
            TMG_CUDA(cudaMalloc(&t.p, bytes));
            p = t.p;
        }
        TMG_CUDA(cudaMemsetAsync(p, 0, bytes, stream));
        return p;
    }
    int clusterSize = 0;  // CTAs of a chain cluster (0: grid chains only)
    static constexpr unsigned long long kClusterMaxPts = 1ull << 18;
    unsigned* chainBar = nullptr;

    // ---- CUDA graphs of the fast cycle ----
    // A fast cycle is a handful of launches whose host-side preparation (omega
    // tables, occupancy queries, argument blocks) and launch latency dominate
    // the small levels (cfg1: ~4 launches in ~35 us).  When cycles are issued
    // back to back (time_cycles) and the cycle's arguments do not depend on n
    // (every omega policy but the n-dependent transition / two-phase ones), the
    // cycle is captured once per state of the
    // double-buffered fine level and replayed with one cudaGraphLaunch; the
    // host-side effects of the captured cycle (buffer swaps, flags) are stored
    // with the graph and reapplied on every replay.
    struct CycleGraph {
        std::string sig;          // pre-state + arguments the capture depends on
        cudaGraphExec_t exec = nullptr;
        double2 *fu = nullptr, *ualt = nullptr;  // post-state
        CUtensorMap mu0, mu1;
        bool fineDerived = false, coarseUStale = false;
        int derivedBpx = 0;
    };
    std::vector<CycleGraph> graphs;
    bool graphsBroken = false;  // a capture failed: ordinary launches from then on
    bool capturing = false;
    // graphs only for cycles issued back to back (time_cycles): a cycle that
    // reads its norms back before the next one is issued runs as fast from
    // launches (measured: 47 vs 45 us per cfg1 cycle) and a short solve would
    // pay the ~0.5 ms capture
    bool backToBack = false;
    void clear_graphs() {
        for (CycleGraph& g : graphs)
            if (g.exec) cudaGraphExecDestroy(g.exec);
        graphs.clear();
    }
    // cudaEventRecord inside a capture must become an event-record node
    void record(cudaEvent_t ev) {
        TMG_CUDA(cudaEventRecordWithFlags(ev, stream, capturing ? cudaEventRecordExternal : cudaEventRecordDefault));
    }

    ~Impl() {
        clear_graphs();
        amr.reset();
        for (void* ptr : allocations) cudaFree(ptr);
        if (hNorm) cudaFreeHost(hNorm);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (evf0) cudaEventDestroy(evf0);
        if (evf1) cudaEventDestroy(evf1);
        if (stream) cudaStreamDestroy(stream);
    }

    template <class T>
    T* alloc(size_t count) {
        void* ptr = nullptr;
        TMG_CUDA(cudaMalloc(&ptr, count * sizeof(T)));
        allocations.push_back(ptr);
        TMG_CUDA(cudaMemsetAsync(ptr, 0, count * sizeof(T), stream));
        return static_cast<T*>(ptr);
    }
    // planes [za, zb) of a level whose planes hold `plane` elements, addressed
    // with global lattice indices (the returned base is za planes before the
    // allocation; only indices inside the range are ever touched)
    template <class T>
    T* alloc_planes(long long plane, int za, int zb) {
        T* ptr = alloc<T>(static_cast<size_t>(plane) * static_cast<size_t>(zb - za));
        return ptr - plane * za;
    }

    // grid-stride launches: enough blocks that each thread has only a few
    // points (memory-level parallelism for the bandwidth-bound level passes)
    int blocks_for(unsigned n) const {
        const long long need = (static_cast<long long>(n) + 255) / 256;
        const long long perSm = dev::switches().gridCap;
        return static_cast<int>(std::max<long long>(1, std::min<long long>(need, perSm * smCount)));
    }

    dev::Lvl make_level(int l, bool fine) {
        dev::Lvl v{};
        v.level = l;
        v.m = static_cast<unsigned>(pow3i(l));
        v.n1 = v.m + 1;
        unsigned long long n = 1;
        for (int d = 0; d < p; ++d) n *= v.n1;
        if (n >= (1ull << 32)) throw CapacityError("level lattice exceeds 2^32 vertices");
        v.n = static_cast<unsigned>(n);
        if (slab() && l >= L - 1) {  // z-slab member: the plane range of levels L and L-1 only
            const long long plane = static_cast<long long>(v.n1) * v.n1;
            const int za = fine ? zaF : zaC, zb = fine ? zbF : zbC;
            v.u = alloc_planes<double2>(plane, za, zb);
            v.sc = alloc_planes<double2>(plane, za, zb);
            if (fine) {
                v.chi = alloc_planes<double2>(plane, za, zb);
            } else {
                v.rhat = alloc_planes<double2>(plane, za, zb);
                v.si = alloc_planes<double2>(plane, za, zb);
                v.sinext = alloc_planes<double2>(plane, za, zb);
            }
            return v;
        }
        if (fine && prob.c64) {  // complex64 storage (float2) behind the double2 pointers: fused3 / conversions only
            v.u = reinterpret_cast<double2*>(alloc<float2>(n));
            v.sc = reinterpret_cast<double2*>(alloc<float2>(n));
            v.chi = reinterpret_cast<double2*>(alloc<float2>(n));
            return v;
        }
        v.u = alloc<double2>(n);
        v.sc = alloc<double2>(n);
        // the fused fine passes keep the fine residual in registers: no fine r-hat
        if (!(fine && fineFused)) v.rhat = alloc<double2>(n);
        if (!prob.fast) {  // exact: the full FAS state of cycles.cpp
            v.chi = alloc<double2>(n);
            v.uhat = alloc<double2>(n);
            if (!fine) v.sf = alloc<double2>(n);
        } else if (fine) {  // fast: load vector on the finest level only
            v.chi = alloc<double2>(n);
        }
        if (!fine) {
            v.si = alloc<double2>(n);
            v.sinext = alloc<double2>(n);
        }
        if (debugR) v.r = alloc<double2>(n);
        return v;
    }

    void compute_level_constants() {
        kc.assign(L + 1, dev::LevelConst{});
        fc.assign(L + 1, fast::LevelCoef{});
        diagInterior.assign(L + 1, Cplx(0.0));
        lapScale.assign(L + 1, Cplx(0.0));
        massScale.assign(L + 1, Cplx(0.0));
        for (int l = 0; l <= L; ++l) {
            // make_cell_kernel, kernels.cpp:7-23 (constant theta and phi)
            const double h = std::pow(3.0, -l);
            const Cplx hElem = h * Cplx(std::cos(prob.theta), std::sin(prob.theta));
            const Cplx ls = cplx_ipow(hElem, p - 2);
            const Cplx ms = cplx_ipow(hElem, p);
            lapScale[l] = ls;
            massScale[l] = ms;
            dev::LevelConst& k = kc[l];
            for (int s = 0; s < (1 << p); ++s) {
                double lap, mas;
                reference_pattern(p, s, lap, mas);
                const Cplx A = ls * lap - prob.phi * ms * mas;  // kernels.cpp:43-44
                k.A[s] = make_double2(A.real(), A.imag());
                k.M[s] = mas;
            }
            k.massScale = make_double2(ms.real(), ms.imag());
            // interior diag: 2^p cell contributions A_aa (kernels.cpp:62-64)
            double lap0, mas0;
            reference_pattern(p, 0, lap0, mas0);
            const Cplx Aaa = ls * lap0 - prob.phi * ms * mas0;
            Cplx dg(0.0);
            for (int i = 0; i < (1 << p); ++i) dg += Aaa;
            diagInterior[l] = dg;
            k.div = div_const(dg);
            fast::LevelCoef& fcl = fc[l];
            for (int cls = 0; cls <= p; ++cls) {  // assembled stencil: 2^(p-k) A_k per class
                double lapk, mask;
                reference_pattern(p, (1 << cls) - 1, lapk, mask);
                const Cplx Ak = ls * lapk - prob.phi * ms * mask;
                const Cplx ck = static_cast<double>(1 << (p - cls)) * Ak;
                fcl.c[cls] = make_double2(ck.real(), ck.imag());
            }
            const Cplx inv = 1.0 / dg;
            fcl.invDiag = make_double2(inv.real(), inv.imag());
        }
    }

    // gaussian scenario (problems.cpp:20-24, 78-90; kernels.cpp:7-23): per level
    // and cell the element operator per XOR pattern and the massScale, from the
    // cell's theta (absorbing layer: 30 degrees within 1/3 of the x / y = 1 faces)
    // and phi at the cell centre -- host arithmetic, so the reference's bits.
    void build_cell_constants() {
        cellA.assign(L + 1, nullptr);
        cellMs.assign(L + 1, nullptr);
        const int nc = 1 << p;
        for (int l = 1; l <= L; ++l) {
            const int m = pow3i(l);
            long long cells = 1;
            for (int d = 0; d < p; ++d) cells *= m;
            std::vector<double2> A(static_cast<size_t>(cells) * nc), MS(static_cast<size_t>(cells));
            const double h = std::pow(3.0, -l);
            for (long long cf = 0; cf < cells; ++cf) {
                long long cc = cf;
                int ci[3] = {0, 0, 0};
                for (int d = 0; d < p; ++d) {
                    ci[d] = static_cast<int>(cc % m);
                    cc /= m;
                }
                double theta = prob.theta;
                for (int d = 0; d < p; ++d) {  // cell_theta: openHi on axes 0 and 1
                    const double centre = (ci[d] + 0.5) * h;
                    if (d < 2 && centre > 1.0 - 1.0 / 3.0) {
                        theta = 30.0 * M_PI / 180.0;
                        break;
                    }
                }
                const Cplx hElem = h * Cplx(std::cos(theta), std::sin(theta));
                const Cplx ls = cplx_ipow(hElem, p - 2);
                const Cplx ms = cplx_ipow(hElem, p);
                double centre[3] = {0.0, 0.0, 0.0};
                for (int d = 0; d < p; ++d) centre[d] = (ci[d] + 0.5) * h;
                const double ph = 45.0 * 45.0 + 135.0 * 135.0 * (std::exp(-(15.0 * centre[0]) * (15.0 * centre[0])) +
                                                                 std::exp(-(15.0 * centre[1]) * (15.0 * centre[1])));
                const Cplx phi(ph, 0.0);
                for (int sp = 0; sp < nc; ++sp) {
                    double lap, mas;
                    reference_pattern(p, sp, lap, mas);
                    const Cplx a = ls * lap - phi * ms * mas;  // kernels.cpp:43-44
                    A[static_cast<size_t>(cf) * nc + sp] = make_double2(a.real(), a.imag());
                }
                MS[static_cast<size_t>(cf)] = make_double2(ms.real(), ms.imag());
            }
            cellA[l] = alloc<double2>(A.size());
            cellMs[l] = alloc<double2>(MS.size());
            TMG_CUDA(cudaMemcpyAsync(cellA[l], A.data(), A.size() * sizeof(double2), cudaMemcpyHostToDevice, stream));
            TMG_CUDA(cudaMemcpyAsync(cellMs[l], MS.data(), MS.size() * sizeof(double2), cudaMemcpyHostToDevice, stream));
            TMG_CUDA(cudaStreamSynchronize(stream));
        }
    }

    void build_restrict_tables() {
        const int NT = p == 1 ? 5 : p == 2 ? 25 : 125;
        const int NP = p == 1 ? 1 : p == 2 ? 2 : 6;
        std::vector<unsigned char> table(static_cast<size_t>(NP * NT));
        std::vector<double> w(NT);
        // kW0/kW1 of transfer.cpp:7-8 per offset k in -2..2
        const double k1d[5] = {1.0 / 3.0, 2.0 / 3.0, 1.0, 2.0 / 3.0, 1.0 / 3.0};
        for (int code = 0; code < NT; ++code) {
            double wt = 1.0;  // restriction_weight, cycles.cpp:46-50: product in axis order
            int cc = code;
            for (int d = 0; d < p; ++d) {
                wt *= k1d[cc % 5];
                cc /= 5;
            }
            w[code] = wt;
        }
        for (int id = 0; id < NP; ++id) {
            int pos = 0;
            for (int gi = 0; gi < (1 << p); ++gi) {
                const int fsel = dev::perm_cell(p, id, gi);  // group = parent cell W-1+f
                // within the group: lexicographic, axis p-1 slowest
                int lo[3], cnt[3];
                for (int d = 0; d < p; ++d) {
                    lo[d] = ((fsel >> d) & 1) ? 0 : -2;
                    cnt[d] = ((fsel >> d) & 1) ? 3 : 2;
                }
                int total = 1;
                for (int d = 0; d < p; ++d) total *= cnt[d];
                for (int t = 0; t < total; ++t) {
                    int tt = t, code = 0, mul = 1;
                    for (int d = 0; d < p; ++d) {
                        const int k = lo[d] + tt % cnt[d];
                        tt /= cnt[d];
                        code += (k + 2) * mul;
                        mul *= 5;
                    }
                    table[static_cast<size_t>(id * NT + pos++)] = static_cast<unsigned char>(code);
                }
            }
        }
        restrictTable = alloc<unsigned char>(table.size());
        restrictWeights = alloc<double>(w.size());
        TMG_CUDA(cudaMemcpyAsync(restrictTable, table.data(), table.size(), cudaMemcpyHostToDevice, stream));
        TMG_CUDA(cudaMemcpyAsync(restrictWeights, w.data(), w.size() * sizeof(double), cudaMemcpyHostToDevice, stream));
        TMG_CUDA(cudaStreamSynchronize(stream));
    }

    template <int P>
    void build_rhs_seeded(int ch = 0) {  // channel ch keyed as oracle/refdriver.cpp seeded_f
        const dev::Lvl& F = lv[L];
        const int key = prob.rhsLattice >= 0 ? prob.rhsLattice : L;
        const int scale = pow3i(key - L);
        const auto [fa, fb] = fine_flat_range();
        dev::k_seeded_chi<P><<<blocks_for(fb - fa), 256, 0, stream>>>(chiNodal, fa, fb, F.n1, prob.rhsSeed, scale,
                                                                       static_cast<long long>(pow3i(key)),
                                                                       prob.rhsSphere ? 1 : 0, ch);
        TMG_CUDA(cudaGetLastError());
    }

    void build_rhs_analytic() {
        // chi_at (problems.cpp:55-68) uses glibc sin; evaluated on the host
        // once per setup so the nodal values are the reference's bits.
        const dev::Lvl& F = lv[L];
        std::vector<double2> h(F.n);
        const double hh = std::pow(3.0, -L);
        for (unsigned f = 0; f < F.n; ++f) {
            unsigned ff = f;
            double x[3];
            for (int d = 0; d < p; ++d) {
                x[d] = static_cast<int>(ff % F.n1) * hh;
                ff /= F.n1;
            }
            double v = 0.0;
            if (prob.chi == ChiKind::SinProduct) {
                const double dd = static_cast<double>(p);
                v = dd * M_PI * M_PI;
                for (int d = 0; d < p; ++d) v *= std::sin(M_PI * x[d]);
            } else if (prob.chi == ChiKind::BallIndicator) {
                double r2 = 0.0;
                for (int d = 0; d < p; ++d) r2 += (x[d] - 0.5) * (x[d] - 0.5);
                v = r2 < 0.01 ? 1.0 : 0.0;
            } else if (prob.chi == ChiKind::Gaussian) {  // problems.cpp:20-21
                v = std::exp(-(125.0 * x[0]) * (125.0 * x[0]) - (125.0 * x[1]) * (125.0 * x[1]));
            }
            h[f] = make_double2(v, 0.0);
        }
        const auto [fa, fb] = fine_flat_range();
        TMG_CUDA(cudaMemcpyAsync(chiNodal + fa, h.data() + fa, (fb - fa) * sizeof(double2), cudaMemcpyHostToDevice,
                                 stream));
        TMG_CUDA(cudaStreamSynchronize(stream));
    }

    template <int P>
    void load_vector(unsigned fa, unsigned fb, int ch) {
        const dev::Lvl F = level(ch, L);
        dev::k_load_vector<P><<<blocks_for(fb - fa), 256, 0, stream>>>(F, chiNodal, kc[L], fa, fb,
                                                                     prob.gaussian ? cellMs[L] : nullptr);
        TMG_CUDA(cudaGetLastError());
    }

    // load vector on planes [za, zb) of the last axis (za < 0: everywhere)
    void load_vector_dispatch(int za = -1, int zb = -1, int ch = 0) {
        const dev::Lvl& F = lv[L];
        if (prob.fast && prob.c64) {  // complex128 load vector, stored as complex64
            Tmp t;
            dev::Lvl Fd = F;
            Fd.chi = tmp_fine(t);
            fast::load_vector(p, Fd, chiNodal, kc[L].massScale, blocks_for(F.n), stream, za, zb);
            dev::k_d2f<<<blocks_for(F.n), 256, 0, stream>>>(Fd.chi, reinterpret_cast<float2*>(F.chi), F.n);
            TMG_CUDA(cudaGetLastError());
            TMG_CUDA(cudaStreamSynchronize(stream));
            return;
        }
        if (prob.fast) {  // separable assembled mass stencil (rounding differs from the cell-by-cell sum)
            fast::load_vector(p, F, chiNodal, kc[L].massScale, blocks_for(F.n), stream, za, zb);
            TMG_CUDA(cudaGetLastError());
            return;
        }
        unsigned fa = 0, fb = F.n;
        if (za >= 0) {
            unsigned plane = 1;
            for (int d = 0; d < p - 1; ++d) plane *= F.n1;
            fa = static_cast<unsigned>(za) * plane;
            fb = static_cast<unsigned>(std::min<long long>(zb, F.n1)) * plane;
        }
        if (fb <= fa) return;
        if (p == 1) load_vector<1>(fa, fb, ch);
        else if (p == 2) load_vector<2>(fa, fb, ch);
        else load_vector<3>(fa, fb, ch);
    }

    template <int P>
    void cycle_exact(const Policy& pol, int n, bool timed) {
        const int nch = prob.channels;
        const bool coupled = nch > 1 && prob.coupling != Cplx(0.0);
        // top-down (levels 1..L; level 0 holds only zero boundary corners); channels are independent here
        for (int l = 1; l <= L; ++l) {
            if (timed && l == L) record(evf0);
            for (int ch = 0; ch < nch; ++ch)
                dev::k_topdown<P><<<blocks_for(lv[l].n), 256, 0, stream>>>(level(ch, l), level(ch, l - 1),
                                                                          pol.bpx ? 1 : 0);
        }
        for (int l = L; l >= 1; --l) {
            for (int ch = 0; ch < nch; ++ch) {
                dev::ResArgs a{};
                a.lv = level(ch, l);
                a.par = level(ch, l - 1);
                a.k = kc[l];
                const Cplx w = omega_unmasked(pol, L - l, n);
                a.k.wRaw = make_double2(w.real(), w.imag());
                a.ellMin = prob.ellMin;
                a.isFine = l == L ? 1 : 0;
                a.bpx = pol.bpx ? 1 : 0;
                a.hb = (pol.hbMask && !pol.bpx) ? 1 : 0;
                a.partials = partials + 2 * static_cast<size_t>(normBlocks) * ch;
                const int nb = l == L ? normBlocks : blocks_for(lv[l].n);
                if (prob.gaussian) {
                    dev::k_residual_cells<P><<<nb, 256, 0, stream>>>(a, cellA[l]);
                } else if (coupled) {
                    dev::McArgs mc{};
                    mc.u = chanU[l];
                    mc.uhat = chanUh[l];
                    mc.nch = nch;
                    mc.own = ch;
                    for (int sp = 0; sp < (1 << p); ++sp) mc.Mc[sp] = couplingM[l][sp];
                    dev::k_residual_exact<P, true><<<nb, 256, 0, stream>>>(a, mc);
                } else {
                    dev::k_residual_exact<P, false><<<nb, 256, 0, stream>>>(a, dev::McArgs{});
                }
            }
            if (timed && l == L) record(evf1);
            if (l >= 2) {
                const int zero = l <= prob.ellMin ? 1 : 0;
                for (int ch = 0; ch < nch; ++ch)
                    dev::k_restrict_exact<P><<<blocks_for(lv[l - 1].n), 256, 0, stream>>>(
                        level(ch, l), level(ch, l - 1), restrictTable, restrictWeights, zero);
            }
        }
        for (int ch = 0; ch < nch; ++ch)
            dev::k_norm_final<<<1, 1024, 0, stream>>>(partials + 2 * static_cast<size_t>(normBlocks) * ch, normBlocks,
                                                      dNorm + 2 * ch);
        TMG_CUDA(cudaGetLastError());
    }

    // channel ch's arrays of level l (channel 0: lv)
    dev::Lvl level(int ch, int l) const { return ch == 0 ? lv[l] : chanLv[ch - 1][l]; }

    template <int P>
    void cycle_fast(const Policy& pol, int n, bool timed) {
        const int bpx = pol.bpx ? 1 : 0;
        auto args = [&](int l) {
            fast::ResArgs a{};
            a.lv = lv[l];
            a.par = lv[l - 1];
            a.k = fc[l];
            const Cplx w = omega_unmasked(pol, L - l, n);
            a.k.wRaw = make_double2(w.real(), w.imag());
            a.ellMin = prob.ellMin;
            a.bpx = bpx;
            a.hb = (pol.hbMask && !pol.bpx) ? 1 : 0;
            a.partials = partials;
            return a;
        };
        // levels 1..top (each below kChainMaxN points) run as one cooperative
        // chain per phase; bigger levels keep their own full-grid launches
        const int top = chain_top(L - 1);
        const bool useChain = top >= 1;
        fast::ChainArgs ch{};
        if (useChain) ch = make_chain(pol, n, top);
        // the fused passes read level L-1's top-down values from scTD (written there
        // directly; the staged sc stays in place), and td-bpx's si from siTD:
        // both are what fused3::derive_u / fused2::derive_u re-read later
        const bool toTD = (P == 3 && fused) || (P == 2 && fused2on);
        if (use_pyramid()) {
            topdown_all(bpx, -1, toTD ? scTD : nullptr);
        } else {
            if (useChain) fast::chain_down(P, ch, ch.cluster ? clusterSize : chainGrid, stream);
            for (int l = useChain ? top + 1 : 1; l < L; ++l) {
                dev::Lvl c = lv[l];
                if (l == L - 1 && toTD) c.scOut = scTD;
                fast::topdown_coarse(P, c, lv[l - 1], bpx, blocks_for(lv[l].n), stream);
            }
            if (toTD && useChain && top == L - 1) save_coarse_td(0, static_cast<int>(lv[L - 1].n1), false, true);  // in place
        }
        if (P == 3 && fused && bpx) save_coarse_td(0, static_cast<int>(lv[L - 1].n1), true, false);
        if (timed) record(evf0);
        if (P == 2 && fused2on) {
            fused2::Args fa{};
            dev::Lvl& F = lv[L];
            fa.uNew = uAlt;   // v-form (fused3.cuh)
            fa.scNew = F.sc;
            fa.u = F.u;
            fa.sc = F.sc;
            fa.b = F.chi;
            fa.scC = scTD;  // level L-1 top-down values
            fa.siC = lv[L - 1].si;
            fa.sinextC = lv[L - 1].sinext;
            fa.partial = partial2;
            fa.norms = partials;
            fa.n1 = F.n1;
            fa.n1c = lv[L - 1].n1;
            fa.g = geo2;
            fa.k = fc[L];
            const Cplx w = omega_unmasked(pol, 0, n);
            fa.k.wRaw = make_double2(w.real(), w.imag());
            fa.bpx = bpx;
            fa.hb = (pol.hbMask && !pol.bpx) ? 1 : 0;
            fa.ellMin = prob.ellMin;
            fa.level = L;
            // the 2D pass is bound by its per-row barrier, not by HBM: it keeps the
            // stored fine sc (no derive, no si copy for td-bpx)
            fa.writeSc = 1;
            fa.c64 = prob.c64 ? 1 : 0;
            fused2::launch(fa, stream);
            if (timed) record(evf1);
            if (use_up()) {  // combine + level L-1 smoothing, then the whole bottom-up in one launch
                const fast::ResArgs sL = args(L - 1);
                fused2::combine(fa, lv[L - 1].rhat, stream, &sL);
                std::swap(F.u, uAlt);
                up_all(pol, n, fused2::blocks(geo2));
                TMG_CUDA(cudaGetLastError());
                coarseUStale = true;
                return;
            }
            fused2::combine(fa, lv[L - 1].rhat, stream);
            std::swap(F.u, uAlt);
            for (int l = L - 1; l >= (useChain ? top + 1 : 1); --l) {
                if (l < L - 1 && l >= prob.ellMin)
                    fast::restrict_level(P, lv[l + 1], lv[l], nullptr, blocks_for(lv[l].n), stream);
                fast::smooth_coarse(P, args(l), blocks_for(lv[l].n), stream);
            }
            if (useChain) {
                if (top < L - 1 && top >= prob.ellMin)
                    fast::restrict_level(P, lv[top + 1], lv[top], nullptr, blocks_for(lv[top].n), stream);
                ch.firstRestrict = 0;
                ch.normBlocks = fused2::blocks(geo2);
                fast::chain_up(P, ch, ch.cluster ? clusterSize : chainGrid, stream);
            } else {
                dev::k_norm_final<<<1, 1024, 0, stream>>>(partials, fused2::blocks(geo2), dNorm);
            }
            TMG_CUDA(cudaGetLastError());
            coarseUStale = true;
            return;
        }
        if (P == 3 && fused) {
            fused3::Args fa{};
            dev::Lvl& F = lv[L];
            fa.writeSc = 0;  // the fine sc is re-derived on demand (fused3::derive_u)
            fa.uNew = uAlt;   // next v (v-form, fused3.cuh)
            fa.scNew = F.sc;  // write-only
            fa.b = F.chi;
            fa.scC = scTD;  // level L-1 top-down values (read through mapC)
            fa.siC = lv[L - 1].si;
            fa.sinextC = lv[L - 1].sinext;
            fa.partial = partial3;
            fa.norms = partials;
            fa.n1 = F.n1;
            fa.n1c = lv[L - 1].n1;
            fa.g = geo;
            fa.k = fc[L];
            const Cplx w = omega_unmasked(pol, 0, n);
            fa.k.wRaw = make_double2(w.real(), w.imag());
            fa.bpx = bpx;
            fa.hb = (pol.hbMask && !pol.bpx) ? 1 : 0;
            fa.ellMin = prob.ellMin;
            fa.level = L;
            fa.c64 = prob.c64 ? 1 : 0;
            fused3::launch(fa, mapU[0], mapC, mapI, mapB, stream);
            if (timed) record(evf1);
            const int lo = useChain ? top + 1 : 1;
            const fast::ResArgs sL = args(L - 1);
            fused3::combine(fa, lv[L - 1].rhat, blocks_for(lv[L - 1].n), stream, -1, -1,
                            (use_up() || lo <= L - 1) ? &sL : nullptr);
            std::swap(F.u, uAlt);
            std::swap(mapU[0], mapU[1]);
            fineDerived = true;
            derivedBpx = bpx;
            if (use_up()) {
                up_all(pol, n, fused3::blocks(geo));
                TMG_CUDA(cudaGetLastError());
                coarseUStale = true;
                return;
            }
            for (int l = L - 1; l >= lo; --l) {
                if (l < L - 1 && l >= prob.ellMin)
                    fast::restrict_level(P, lv[l + 1], lv[l], nullptr, blocks_for(lv[l].n), stream);
                if (l < L - 1) fast::smooth_coarse(P, args(l), blocks_for(lv[l].n), stream);  // L-1: in the combine
            }
            if (useChain) {
                if (top < L - 1 && top >= prob.ellMin)
                    fast::restrict_level(P, lv[top + 1], lv[top], nullptr, blocks_for(lv[top].n), stream);
                ch.firstRestrict = 0;
                ch.normBlocks = fused3::blocks(geo);
                fast::chain_up(P, ch, ch.cluster ? clusterSize : chainGrid, stream);
            } else {
                dev::k_norm_final<<<1, 1024, 0, stream>>>(partials, fused3::blocks(geo), dNorm);
            }
            TMG_CUDA(cudaGetLastError());
            coarseUStale = true;
            return;
        }
        fast::correct_fine(P, lv[L], lv[L - 1], bpx, blocks_for(lv[L].n), stream);
        const int nb = fast::residual_fine(P, args(L), smCount, stream);
        if (timed) record(evf1);
        for (int l = L - 1; l >= (useChain ? top + 1 : 1); --l) {
            if (l >= prob.ellMin) fast::restrict_level(P, lv[l + 1], lv[l], nullptr, blocks_for(lv[l].n), stream);
            fast::smooth_coarse(P, args(l), blocks_for(lv[l].n), stream);
        }
        if (useChain) {
            ch.firstRestrict = 1;  // fine = lv[top + 1] into lv[top]
            ch.normBlocks = nb;
            fast::chain_up(P, ch, ch.cluster ? clusterSize : chainGrid, stream);
        } else {
            dev::k_norm_final<<<1, 1024, 0, stream>>>(partials, nb, dNorm);
        }
        TMG_CUDA(cudaGetLastError());
        coarseUStale = true;
    }

    template <int P>
    void inject_coarse_u() {
        Tmp t;
        for (int l = L - 1; l >= 1; --l) {
            if (l == L - 1 && fineDerived) {  // the derived fine u (sc-free fused pass)
                dev::Lvl Fd = lv[L];
                Fd.u = tmp_fine(t);
                const auto [fa, fb] = fine_flat_range();
                derive_fine_u(Fd.u, fa, fb);
                dev::k_inject_u<P><<<blocks_for(lv[l].n), 256, 0, stream>>>(lv[l], Fd, 0);
                continue;
            }
            if (l == L - 1 && prob.c64) {  // u = v - sc of the complex64 fine level, as complex128
                dev::Lvl Fd = lv[L];
                Fd.u = tmp_fine(t);
                dev::k_vform_f2d<<<blocks_for(Fd.n), 256, 0, stream>>>(reinterpret_cast<const float2*>(lv[L].u),
                                                                       reinterpret_cast<const float2*>(lv[L].sc),
                                                                       Fd.u, Fd.n);
                dev::k_inject_u<P><<<blocks_for(lv[l].n), 256, 0, stream>>>(lv[l], Fd, 0);
                continue;
            }
            dev::k_inject_u<P><<<blocks_for(lv[l].n), 256, 0, stream>>>(lv[l], lv[l + 1], l == L - 1 && vForm() ? 1 : 0);
        }
        TMG_CUDA(cudaStreamSynchronize(stream));
    }

    // the finest level holds v = u + sc (fused fast paths, fused3.cuh)
    bool vForm() const { return prob.fast && (fused || fused2on); }

    // planes [za, zb) of level L-1's top-down sc, as the sc-free fused pass is about to read them
    // planes (2D: rows) [za, zb) of level L-1's si (td-bpx) and / or top-down sc as
    // the sc-free fused pass is about to read them (sc: only where the top-down
    // ran in place -- the coarse chains)
    void save_coarse_td(int za, int zb, bool si, bool sc) {
        const dev::Lvl& C = lv[L - 1];
        const long long plane = p == 3 ? static_cast<long long>(C.n1) * C.n1 : C.n1;
        const size_t bytes = static_cast<size_t>((zb - za) * plane) * sizeof(double2);
        if (zb <= za) return;
        if (sc) TMG_CUDA(cudaMemcpyAsync(scTD + za * plane, C.sc + za * plane, bytes, cudaMemcpyDeviceToDevice, stream));
        if (si) TMG_CUDA(cudaMemcpyAsync(siTD + za * plane, C.si + za * plane, bytes, cudaMemcpyDeviceToDevice, stream));
    }

    // the fine u of the last sc-free pass on the flat range [fa, fb) into out (global indices)
    void derive_fine_u(double2* out, unsigned fa, unsigned fb) {
        const dev::Lvl& F = lv[L];
        const double2* si = derivedBpx ? siTD : nullptr;
        if (p == 2) fused2::derive_u(uAlt, scTD, si, F.n1, lv[L - 1].n1, fa, fb, out, prob.c64, stream);
        else fused3::derive_u(uAlt, scTD, si, F.n1, lv[L - 1].n1, fa, fb, out, prob.c64, stream);
        TMG_CUDA(cudaGetLastError());
    }

    // fineDerived -> the fine arrays hold (v, sc) again, sc = v - u with the derived u;
    // toU: (u, sc) instead (what Hierarchy::unfold makes of the old finest level)
    void split_fine(bool toU) {
        if (!fineDerived) return;
        const dev::Lvl& F = lv[L];
        const auto [fa, fb] = fine_flat_range();
        Tmp t;
        double2* u = tmp_fine(t);
        derive_fine_u(u, fa, fb);
        if (prob.c64)
            dev::k_split_derived<float2><<<blocks_for(fb - fa), 256, 0, stream>>>(
                reinterpret_cast<float2*>(F.u), reinterpret_cast<float2*>(F.sc), u, fa, fb, toU ? 1 : 0);
        else
            dev::k_split_derived<double2><<<blocks_for(fb - fa), 256, 0, stream>>>(F.u, F.sc, u, fa, fb, toU ? 1 : 0);
        TMG_CUDA(cudaGetLastError());
        TMG_CUDA(cudaStreamSynchronize(stream));
        fineDerived = false;
    }

    void materialize_coarse_u() {
        if (!prob.fast || !coarseUStale) return;
        if (p == 1) inject_coarse_u<1>();
        else if (p == 2) inject_coarse_u<2>();
        else inject_coarse_u<3>();
        coarseUStale = false;
    }

    void cycle_fast_dispatch(const Policy& pol, int n, bool timed) {
        if (p == 1) cycle_fast<1>(pol, n, timed);
        else if (p == 2) cycle_fast<2>(pol, n, timed);
        else cycle_fast<3>(pol, n, timed);
    }

    // the cycle's launch arguments as bytes, or "" when they depend on n
    std::string cycle_signature(const Policy& pol, int n, bool timed) const {
        std::string sig;
        auto put = [&](const void* ptr, size_t bytes) { sig.append(static_cast<const char*>(ptr), bytes); };
        for (int succ = 0; succ <= L; ++succ) {
            const Cplx w = omega_unmasked(pol, succ, n);
            if (w != omega_unmasked(pol, succ, n + 1)) return std::string();
            put(&w, sizeof(w));
        }
        (void)timed;  // a captured cycle always records the fine-pass events (time_cycles and cycle share it)
        const int flags[3] = {pol.bpx ? 1 : 0, pol.hbMask ? 1 : 0, prob.ellMin};
        put(flags, sizeof(flags));
        put(&lv[L].u, sizeof(double2*));
        put(&uAlt, sizeof(double2*));
        return sig;
    }

    void cycle_fast_graph(const Policy& pol, int n, bool timed) {
        const std::string sig =
            dev::switches().graph && !graphsBroken && backToBack ? cycle_signature(pol, n, timed) : std::string();
        if (sig.empty()) {
            cycle_fast_dispatch(pol, n, timed);
            return;
        }
        for (CycleGraph& g : graphs) {
            if (g.sig != sig) continue;
            TMG_CUDA(cudaGraphLaunch(g.exec, stream));
            lv[L].u = g.fu;
            uAlt = g.ualt;
            mapU[0] = g.mu0;
            mapU[1] = g.mu1;
            fineDerived = g.fineDerived;
            derivedBpx = g.derivedBpx;
            coarseUStale = g.coarseUStale;
            return;
        }
        // capture: the host-side state is restored if the capture fails
        double2 *fu = lv[L].u, *ua = uAlt;
        const CUtensorMap m0 = mapU[0], m1 = mapU[1];
        const bool fd = fineDerived, cs = coarseUStale;
        const int db = derivedBpx;
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        bool ok = cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
        if (ok) {
            capturing = true;
            try {
                cycle_fast_dispatch(pol, n, true);
            } catch (...) {
                ok = false;
            }
            capturing = false;
            ok = cudaStreamEndCapture(stream, &graph) == cudaSuccess && ok && graph;
        }
        if (ok) ok = cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
        if (graph) cudaGraphDestroy(graph);
        if (!ok) {
            (void)cudaGetLastError();
            graphsBroken = true;
            lv[L].u = fu;
            uAlt = ua;
            mapU[0] = m0;
            mapU[1] = m1;
            fineDerived = fd;
            derivedBpx = db;
            coarseUStale = cs;
            cycle_fast_dispatch(pol, n, timed);
            return;
        }
        if (graphs.size() >= 4) {
            cudaGraphExecDestroy(graphs.front().exec);
            graphs.erase(graphs.begin());
        }
        CycleGraph g;
        g.sig = sig;
        g.exec = exec;
        g.fu = lv[L].u;
        g.ualt = uAlt;
        g.mu0 = mapU[0];
        g.mu1 = mapU[1];
        g.fineDerived = fineDerived;
        g.derivedBpx = derivedBpx;
        g.coarseUStale = coarseUStale;
        graphs.push_back(g);
        TMG_CUDA(cudaGraphLaunch(exec, stream));
    }

    void run_cycle(const Policy& pol, int n, bool timed) {
        if (prob.fast) {
            cycle_fast_graph(pol, n, timed);
        } else {
            if (p == 1) cycle_exact<1>(pol, n, timed);
            else if (p == 2) cycle_exact<2>(pol, n, timed);
            else cycle_exact<3>(pol, n, timed);
        }
    }

    // bottom-up below level L-1 (r_{L-1} complete and smoothed) as one cooperative launch
    // (levels above the chain top S: restriction + smoothing kernels; S-1 .. 1:
    // fast::up_coop, which restricts out of S)
    bool use_up() const { return use_up_from(L - 1); }
    bool use_up_from(int from) const {
        return dev::switches().up && chainBar && (p == 2 || p == 3) && from >= 2 && chain_top(from) >= 2;
    }
    // from: the level whose r is complete and smoothed (L-1 after the combine; the
    // slab path's replicated top L-2); norms = false: up_coop reduces no norms
    void up_all(const Policy& pol, int n, int normBlocks, int from = -1, bool norms = true) {
        if (from < 0) from = L - 1;
        const int S = chain_top(from);
        for (int l = from - 1; l >= S; --l) {
            fast::ResArgs sl{};
            sl.lv = lv[l];
            sl.par = lv[l - 1];
            sl.k = fc[l];
            const Cplx w = omega_unmasked(pol, L - l, n);
            sl.k.wRaw = make_double2(w.real(), w.imag());
            sl.ellMin = prob.ellMin;
            sl.bpx = pol.bpx ? 1 : 0;
            sl.hb = (pol.hbMask && !pol.bpx) ? 1 : 0;
            sl.partials = partials;
            if (l >= prob.ellMin) fast::restrict_level(p, lv[l + 1], lv[l], nullptr, blocks_for(lv[l].n), stream, -1, -1, &sl);
            else fast::smooth_coarse(p, sl, blocks_for(lv[l].n), stream);
        }
        fast::ChainArgs ch = make_chain(pol, n, S - 1);  // fine = level S
        ch.firstRestrict = 1;
        ch.normBlocks = normBlocks;
        if (!norms) ch.normOut = nullptr;
        fast::up_coop(p, ch, chainBar + 2, smCount, stream);
    }

    // coarse top-down of levels 1..L-1 as one pyramid launch (fast::topdown_pyramid)
    bool use_pyramid() const {
        return dev::switches().pyr && (p == 2 || p == 3) && L >= 2 && L - 1 < fast::kPyrMaxLevels;
    }
    // pyramid up to the highest level below kPyrMaxN points, per-level launches above it
#ifndef TMG_PYR_MAXN
#define TMG_PYR_MAXN (1u << 21)
#endif
    static constexpr unsigned kPyrMaxN = TMG_PYR_MAXN;
    int pyramid_top() const {
        int T = L - 1;
        while (T > 1 && lv[T].n > kPyrMaxN) --T;
        return T;
    }
    // levels 1 .. last-1 (default: every coarse level); the slab path passes
    // last = L-1 (level L-1 is sharded and done per plane range)
    // outL1: level L-1's top-down values go there instead of in place (the fused
    // passes read them from scTD: the staged sc stays, nothing to save)
    void topdown_all(int bpx, int last = -1, double2* outL1 = nullptr) {
        if (last < 0) last = L;
        fast::PyrArgs a{};
        const int T = std::min(pyramid_top(), last - 1);
        for (int l = 0; l <= T; ++l) {
            a.lv[l].sc = lv[l].sc;
            a.lv[l].si = lv[l].si ? lv[l].si : lv[l].sc;  // si is read only under BPX
            a.lv[l].m = static_cast<int>(lv[l].m);
            a.lv[l].n1 = static_cast<int>(lv[l].n1);
        }
        a.scTin = lv[T].sc;
        a.scT = (T == L - 1 && outL1) ? outL1 : lv[T].sc;
        a.bpx = bpx;
        const size_t smem = fast::pyramid_setup(p, a, T);
        fast::topdown_pyramid(p, a, smem, stream);
        for (int l = T + 1; l < last; ++l) {
            dev::Lvl c = lv[l];
            if (l == L - 1) c.scOut = outL1;
            fast::topdown_coarse(p, c, lv[l - 1], bpx, blocks_for(lv[l].n), stream);
        }
    }

    // highest level <= maxLevel of the coarse chain (every level below kChainMaxN
    // points joins it); 0 when chains are off
    int chain_top(int maxLevel) const {
        int top = maxLevel;
        while (top >= 1 && lv[top].n >= kChainMaxN) --top;
        return (chainGrid > 0 && top >= 1 && top < fast::kMaxChainLevels) ? top : 0;
    }

    fast::ChainArgs make_chain(const Policy& pol, int n, int top) const {
        fast::ChainArgs ch{};
        for (int l = 0; l <= top; ++l) {
            ch.lv[l] = lv[l];
            ch.k[l] = fc[l];
            const Cplx w = omega_unmasked(pol, L - l, n);
            ch.k[l].wRaw = make_double2(w.real(), w.imag());
        }
        ch.fine = lv[top + 1];
        ch.top = top;
        ch.ellMin = prob.ellMin;
        ch.bpx = pol.bpx ? 1 : 0;
        ch.hb = (pol.hbMask && !pol.bpx) ? 1 : 0;
        ch.bar = chainBar;
        ch.normPartials = partials;
        ch.normOut = dNorm;
        unsigned long long pts = 0;  // small chains run as one thread-block cluster
        for (int l = 1; l <= top; ++l) pts += lv[l].n;
        ch.cluster = (clusterSize > 0 && pts <= kClusterMaxPts) ? 1 : 0;
        return ch;
    }

    // kernel launches of one cycle (bench.py "gpu_launches"), mirroring cycle_fast / cycle_exact
    int launches_per_cycle() const {
        if (!prob.fast) return 3 * L;  // top-down 1..L, residual L..1, restriction L..2, norm
        const int top = chain_top(L - 1);
        const bool useChain = top >= 1;
        const bool fusedPath = (p == 3 && fused) || (p == 2 && fused2on);
        const int lo = useChain ? top + 1 : 1;
        int n = use_pyramid() ? 1 + (L - 1 - pyramid_top()) : useChain ? 1 + (L - 1 - top) : (L - 1);  // top-down
        n += 2;                                            // fine pass (+ combine, or correction + residual)
        if (fusedPath && use_up()) return n + (L - 1 - top) + 1;  // restrict + smooth above the chain top, up_coop
        for (int l = L - 1; l >= lo; --l)
            n += (p == 3 && fused && l == L - 1 ? 0 : 1) + ((fusedPath ? l < L - 1 : true) && l >= prob.ellMin ? 1 : 0);
        if (useChain) n += 1 + (fusedPath && top < L - 1 && top >= prob.ellMin ? 1 : 0);
        else n += 1;                                       // norm reduction
        return n;
    }

    void check_diag() {
        if (prob.gaussian) return;  // cell-varying diagonals: checked by construction (phi > 0)
        // jacobi (kernels.cpp:102-106) runs on interior vertices of levels
        // >= ellMin; the interior diagonal is constant per level here.
        for (int l = std::max(1, prob.ellMin); l <= L; ++l)
            if (std::abs(diagInterior[l]) < 1e-300)
                throw SingularDiagonalError("vanishing operator diagonal (phi*h^2 resonance?)");
    }

    // Morton (DFS) order of the interior fine vertices = their touch-last order
    // (exact_ops.cuh rule (2)); the reference sums norms in this order.
    std::vector<unsigned> finishOrder;

    void build_finish_order() {
        const dev::Lvl& F = lv[L];
        std::vector<std::pair<unsigned long long, unsigned>> keys;
        for (unsigned f = 0; f < F.n; ++f) {
            unsigned ff = f;
            int idx[3];
            bool interior = true;
            for (int d = 0; d < p; ++d) {
                idx[d] = static_cast<int>(ff % F.n1);
                ff /= F.n1;
                interior &= idx[d] > 0 && idx[d] < static_cast<int>(F.m);
            }
            if (!interior) continue;
            unsigned long long key = 0;
            for (int k = L - 1; k >= 0; --k) {
                int slot = 0, mul = 1;
                for (int d = 0; d < p; ++d) {
                    slot += ((idx[d] / pow3i(k)) % 3) * mul;
                    mul *= 3;
                }
                key = key * static_cast<unsigned long long>(pow3i(p)) + static_cast<unsigned long long>(slot);
            }
            keys.emplace_back(key, f);
        }
        std::sort(keys.begin(), keys.end());
        finishOrder.resize(keys.size());
        for (size_t i = 0; i < keys.size(); ++i) finishOrder[i] = keys[i].second;
    }

    // proj/src/cycles.cpp:248-258 + 94-97 on the host, bit-for-bit.
    void host_norms(SweepStats& st) {
        if (finishOrder.empty()) build_finish_order();
        const dev::Lvl& F = lv[L];
        std::vector<Cplx> r(F.n);
        TMG_CUDA(cudaMemcpyAsync(r.data(), F.r, static_cast<size_t>(F.n) * sizeof(double2), cudaMemcpyDeviceToHost,
                                 stream));
        TMG_CUDA(cudaStreamSynchronize(stream));
        const double hp = std::pow(std::pow(3.0, -L), p);
        double mx = 0.0, eu = 0.0, hn = 0.0;
        for (unsigned f : finishOrder) {
            const double m = std::abs(r[f]);
            mx = std::max(mx, m);
            eu += m * m;
            hn += hp * m * m;
        }
        st.maxNorm = mx;
        st.euclidNorm = std::sqrt(eu);
        st.hNorm = std::sqrt(hn);
    }

    SweepStats cycle(const Policy& pol, int n, bool timed = false) {
        if (amr) return amr->cycle(pol, n);
        check_diag();
        run_cycle(pol, n, timed);
        const int nch = prob.channels;
        TMG_CUDA(cudaMemcpyAsync(hNorm, dNorm, 2 * sizeof(double) * nch, cudaMemcpyDeviceToHost, stream));
        TMG_CUDA(cudaStreamSynchronize(stream));
        SweepStats st;
        const double hp = std::pow(std::pow(3.0, -L), p);
        st.maxNorm = std::sqrt(hNorm[0]);
        st.euclidNorm = std::sqrt(hNorm[1]);
        st.hNorm = std::sqrt(hp * hNorm[1]);
        if (nch > 1) {  // per channel, aggregated as runner.cpp:68-77 (max; l2 over channels)
            double mx = 0.0, se = 0.0, sh = 0.0;
            for (int ch = 0; ch < nch; ++ch) {
                const double cm = std::sqrt(hNorm[2 * ch]), ce = std::sqrt(hNorm[2 * ch + 1]),
                             chh = std::sqrt(hp * hNorm[2 * ch + 1]);
                st.chMax.push_back(cm);
                st.chEuclid.push_back(ce);
                st.chH.push_back(chh);
                mx = std::max(mx, cm);
                se += ce * ce;
                sh += chh * chh;
            }
            st.maxNorm = mx;
            st.euclidNorm = std::sqrt(se);
            st.hNorm = std::sqrt(sh);
        }
        long long inner = 1;
        for (int d = 0; d < p; ++d) inner *= pow3i(L) - 1;
        st.updatedFineVertices = inner;
        if (prob.hostNorms && !prob.fast) host_norms(st);
        return st;
    }
};

Hierarchy::Hierarchy(const Problem& prob) : impl_(new Impl()) {
    Impl& I = *impl_;
    dev::refresh_switches();  // developer A/B environment, read here, not on the launch path
    I.prob = prob;
    I.p = prob.dim;
    I.L = prob.levels;
    if (prob.dim < 1 || prob.dim > 3) throw UnsupportedConfigError("B200 path: dim must be 1, 2 or 3");
    if (prob.levels < 1) throw ConfigError("build_regular needs levels >= 1");
    if (prob.levels > 9) throw ConfigError("tree depth exceeds supported maximum");
    if (prob.sphereLevels < 0 || prob.sphereLevels >= prob.levels) throw ConfigError("sphere_levels out of range");
    if (prob.channels > 1 && (prob.sphereLevels > 0 || prob.dynStart > 0 || prob.hostNorms))
        throw UnsupportedConfigError("B200 path: several channels run on regular trees with device norms");
    // build_regular's capacity estimate (spacetree.cpp:53-63)
    std::size_t estimate = 0;
    const int regularTop = prob.dynStart > 0 ? prob.dynStart : prob.levels - prob.sphereLevels;
    for (int l = 0; l <= regularTop; ++l) {
        std::size_t perAxis = static_cast<std::size_t>(pow3i(l)) + 1, n = 1;
        for (int d = 0; d < prob.dim; ++d) n *= perAxis;
        estimate += n;
    }
    if (estimate > prob.maxVertices)
        throw CapacityError("regular grid would hold " + std::to_string(estimate) + " vertices, cap is " +
                            std::to_string(prob.maxVertices));
    TMG_CUDA(cudaSetDevice(prob.device));
    cudaDeviceProp props{};
    TMG_CUDA(cudaGetDeviceProperties(&props, prob.device));
    I.smCount = props.multiProcessorCount;
    TMG_CUDA(cudaStreamCreateWithFlags(&I.stream, cudaStreamNonBlocking));
    TMG_CUDA(cudaEventCreate(&I.ev0));
    TMG_CUDA(cudaEventCreate(&I.ev1));
    TMG_CUDA(cudaEventCreate(&I.evf0));
    TMG_CUDA(cudaEventCreate(&I.evf1));
    if (prob.sphereLevels > 0 || prob.dynStart > 0) {
        if (prob.hostNorms) throw UnsupportedConfigError("norms = host is not available on adaptive trees");
        I.compute_level_constants();
        I.amr = std::make_unique<AmrTree>(prob, I.kc, I.diagInterior, I.stream, I.smCount);
        return;
    }
    const char* dbg = std::getenv("TMG_DEBUG_R");
    I.debugR = (dbg && dbg[0] == '1') || (prob.hostNorms && !prob.fast);
    {
        const char* f3 = std::getenv("TMG_FUSED");
        const char* f2 = std::getenv("TMG_FUSED2");
        I.fineFused = prob.fast && ((I.p == 3 && I.L >= 2 && !(f3 && f3[0] == '0')) ||
                                    (I.p == 2 && I.L >= 3 && !(f2 && f2[0] == '0')));
    }
    if (prob.c64) {
        if (!prob.fast) throw ConfigError("complex64 storage is a fast-precision mode");
        if ((I.p != 3 && I.p != 2) || !I.fineFused || prob.channels > 1 || prob.gaussian)
            throw UnsupportedConfigError(
                "precision = fast-complex64 runs the fused fine passes (dim = 2 with level >= 3, dim = 3 with level >= 2; "
                "one channel)");
    }
    if (I.slab()) {
        if (!prob.fast || I.p != 3 || !I.fineFused || prob.c64 || prob.channels > 1 || I.L < 3)
            throw UnsupportedConfigError("z-slabs: 3D fast precision (complex128), fused fine pass");
        const int n1 = pow3i(I.L) + 1, n1c = pow3i(I.L - 1) + 1;
        const int Zs = (prob.slabLo + 2) / 3, Ze = (prob.slabHi + 2) / 3;
        I.zaF = std::max(0, prob.slabLo - 1);
        I.zbF = std::min(n1, prob.slabHi + 1);
        I.zaC = std::max(0, Zs - 2);
        I.zbC = std::min(n1c, Ze + 2);
    }
    I.lv.resize(I.L + 1);
    for (int l = 0; l <= I.L; ++l) I.lv[l] = I.make_level(l, l == I.L);
    I.normBlocks = std::max(I.blocks_for(I.lv[I.L].n), fast::residual_fine_blocks(I.p, I.lv[I.L], I.smCount));
    if (prob.fast && I.p == 3 && I.L >= 2) {
        I.fusedResident = fused3::resident_blocks(I.smCount);
        I.normBlocks = std::max(I.normBlocks, fused3::blocks(fused3::geometry(static_cast<int>(I.lv[I.L].m),
                                                                              static_cast<int>(I.lv[I.L - 1].m),
                                                                              prob.zParts, I.fusedResident)));
    }
    {
        const char* f2 = std::getenv("TMG_FUSED2");
        if (prob.fast && I.p == 2 && I.L >= 3 && !(f2 && f2[0] == '0')) {
            I.fused2on = true;
            I.geo2 = fused2::geometry(static_cast<int>(I.lv[I.L].m), static_cast<int>(I.lv[I.L - 1].m), I.smCount);
            I.normBlocks = std::max(I.normBlocks, fused2::blocks(I.geo2));
        }
    }
    if (prob.channels < 1 || prob.channels > 16) throw ConfigError("channels must lie in [1, 16]");
    if (prob.channels > 1) {
        if (prob.fast) throw UnsupportedConfigError("B200 path: several channels run in precision = exact");
        for (int ch = 1; ch < prob.channels; ++ch) {
            std::vector<dev::Lvl> v(I.L + 1);
            for (int l = 0; l <= I.L; ++l) v[l] = I.make_level(l, l == I.L);
            I.chanLv.push_back(v);
        }
    }
    I.partials = I.alloc<double>(2 * static_cast<size_t>(I.normBlocks) * prob.channels);
    if (I.fused2on) {
        I.uAlt = prob.c64 ? reinterpret_cast<double2*>(I.alloc<float2>(I.lv[I.L].n)) : I.alloc<double2>(I.lv[I.L].n);
        I.partial2 = I.alloc<double2>(fused2::partial_count(I.geo2));
        I.scTD = I.alloc<double2>(I.lv[I.L - 1].n);
        I.siTD = I.alloc<double2>(I.lv[I.L - 1].n);
    }
    if (prob.fast) {
        const char* cz = std::getenv("TMG_CHAIN");
        int coop = 0;
        TMG_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, prob.device));
        if (coop && !(cz && cz[0] == '0')) {
            I.chainGrid = fast::chain_grid(I.p, I.smCount);
            I.chainBar = I.alloc<unsigned>(3);  // grid barrier (2) + up_coop's last-CTA counter
            const char* cl = std::getenv("TMG_CHAIN_CLUSTER");
            if (!(cl && cl[0] == '0')) I.clusterSize = fast::chain_cluster_size();
        }
    }
    I.dNorm = I.alloc<double>(2 * static_cast<size_t>(prob.channels));
    TMG_CUDA(cudaMallocHost(&I.hNorm, 2 * sizeof(double) * prob.channels));
    I.chiNodal = I.slab() ? I.alloc_planes<double2>(static_cast<long long>(I.lv[I.L].n1) * I.lv[I.L].n1, I.zaF, I.zbF)
                          : I.alloc<double2>(I.lv[I.L].n);
    I.compute_level_constants();
    I.build_restrict_tables();
    if (prob.gaussian) {
        if (prob.dim != 2) throw ConfigError("the gaussian scenario is two-dimensional");
        if (prob.fast) throw UnsupportedConfigError("the gaussian scenario (cell-varying phi / theta) runs in precision = exact");
        I.build_cell_constants();
    }
    {
        const char* fz = std::getenv("TMG_FUSED");
        if (prob.fast && I.p == 3 && I.L >= 2 && !(fz && fz[0] == '0')) {
            const dev::Lvl& F = I.lv[I.L];
            // v double buffer; sc is write-only (v-form)
            const long long plane = static_cast<long long>(F.n1) * F.n1;
            I.uAlt = prob.c64  ? reinterpret_cast<double2*>(I.alloc<float2>(F.n))
                     : I.slab() ? I.alloc_planes<double2>(plane, I.zaF, I.zbF)
                                : I.alloc<double2>(F.n);
            I.geo = fused3::geometry(static_cast<int>(F.m), static_cast<int>(I.lv[I.L - 1].m), prob.zParts,
                                     I.fusedResident);
            I.partial3 = I.alloc<double2>(fused3::partial_count(I.geo));
            const dev::Lvl& C = I.lv[I.L - 1];
            I.scTD = I.slab() ? I.alloc_planes<double2>(static_cast<long long>(C.n1) * C.n1, I.zaC, I.zbC)
                              : I.alloc<double2>(C.n);
            I.siTD = I.slab() ? I.alloc_planes<double2>(static_cast<long long>(C.n1) * C.n1, I.zaC, I.zbC)
                              : I.alloc<double2>(C.n);
            // slab members: maps over the allocated plane ranges, z coordinates shifted by the kernel
            const long long planeC = static_cast<long long>(C.n1) * C.n1;
            const int nzF = I.slab() ? I.zbF - I.zaF : static_cast<int>(F.n1);
            const int nzC = I.slab() ? I.zbC - I.zaC : static_cast<int>(C.n1);
            const long long offF = I.slab() ? plane * I.zaF : 0, offC = I.slab() ? planeC * I.zaC : 0;
            bool ok = fused3::encode_map(&I.mapU[0], F.u + offF, F.n1, 0, prob.c64, nzF) &&
                      fused3::encode_map(&I.mapU[1], I.uAlt + offF, F.n1, 0, prob.c64, nzF) &&
                      fused3::encode_map(&I.mapC, I.scTD + offC, C.n1, 2, false, nzC) &&
                      fused3::encode_map(&I.mapI, C.si + offC, C.n1, 2, false, nzC) &&
                      fused3::encode_map(&I.mapB, F.chi + offF, F.n1, 1, prob.c64, nzF);
            if (!ok) throw CudaError("cuTensorMapEncodeTiled failed for the fused fine pass");
            I.fused = true;
        }
    }
    if (prob.chi == ChiKind::Seeded) {
        // the seeded rhs keys every channel apart (oracle/refdriver.cpp seeded_f: seed ^ c << 48);
        // channel 0 last so chiNodal keeps its values
        for (int ch = prob.channels - 1; ch >= 0; --ch) {
            if (I.p == 1) I.build_rhs_seeded<1>(ch);
            else if (I.p == 2) I.build_rhs_seeded<2>(ch);
            else I.build_rhs_seeded<3>(ch);
            if (I.slab()) I.load_vector_dispatch(prob.slabLo, prob.slabHi, ch);
            else I.load_vector_dispatch(-1, -1, ch);
        }
    } else {
        I.build_rhs_analytic();
        if (I.slab()) I.load_vector_dispatch(prob.slabLo, prob.slabHi);
        else I.load_vector_dispatch();
        // every channel carries the same fields (runner.cpp:152): same load vector
        for (int ch = 1; ch < prob.channels; ++ch)
            TMG_CUDA(cudaMemcpyAsync(I.chanLv[ch - 1][I.L].chi, I.lv[I.L].chi,
                                     static_cast<size_t>(I.lv[I.L].n) * sizeof(double2), cudaMemcpyDeviceToDevice,
                                     I.stream));
    }
    if (prob.channels > 1) {
        I.chanU.assign(I.L + 1, nullptr);
        I.chanUh.assign(I.L + 1, nullptr);
        I.couplingM.assign(I.L + 1, std::array<double2, 8>{});
        for (int l = 0; l <= I.L; ++l) {
            std::vector<const double2*> pu(prob.channels), ph(prob.channels);
            for (int ch = 0; ch < prob.channels; ++ch) {
                pu[ch] = I.level(ch, l).u;
                ph[ch] = I.level(ch, l).uhat;
            }
            auto** du = I.alloc<const double2*>(prob.channels);
            auto** dh = I.alloc<const double2*>(prob.channels);
            TMG_CUDA(cudaMemcpyAsync(du, pu.data(), pu.size() * sizeof(void*), cudaMemcpyHostToDevice, I.stream));
            TMG_CUDA(cudaMemcpyAsync(dh, ph.data(), ph.size() * sizeof(void*), cudaMemcpyHostToDevice, I.stream));
            I.chanU[l] = du;
            I.chanUh[l] = dh;
            const Cplx aij = prob.coupling * I.massScale[l];  // kernels.cpp:52-53
            for (int sp = 0; sp < (1 << I.p); ++sp) {
                double lap, mas;
                reference_pattern(I.p, sp, lap, mas);
                const Cplx mcpl = aij * mas;
                I.couplingM[l][sp] = make_double2(mcpl.real(), mcpl.imag());
            }
        }
    }
    TMG_CUDA(cudaStreamSynchronize(I.stream));
}

Hierarchy::~Hierarchy() = default;

SweepStats Hierarchy::cycle(const Policy& pol, int n) { return impl_->cycle(pol, n); }

namespace {
vc::Ctx vc_ctx(Hierarchy::Impl& I, std::vector<double2*>& scratch) {
    if (I.amr) throw UnsupportedConfigError("verification cycles run on regular trees (runner.cpp:232)");
    if (I.prob.fast) throw UnsupportedConfigError("verification cycles need the exact storage (precision = exact)");
    if (scratch.empty())
        for (int l = 0; l <= I.L; ++l) scratch.push_back(I.alloc<double2>(I.lv[l].n));
    vc::Ctx x{};
    x.lv = I.lv.data();
    x.L = I.L;
    x.ellMin = I.prob.ellMin;
    x.fc = I.fc.data();
    x.r = scratch.data();
    x.partials = I.partials;
    x.dNorm = I.dNorm;
    x.stream = I.stream;
    x.smCount = I.smCount;
    return x;
}

SweepStats vc_norms(Hierarchy::Impl& I, const vc::Ctx& x) {
    double out[2];
    vc::residual_norms(I.p, x, out);
    SweepStats st;
    const double hp = std::pow(std::pow(3.0, -I.L), I.p);
    st.maxNorm = std::sqrt(out[0]);
    st.euclidNorm = std::sqrt(out[1]);
    st.hNorm = std::sqrt(hp * out[1]);
    long long inner = 1;
    for (int d = 0; d < I.p; ++d) inner *= pow3i(I.L) - 1;
    st.updatedFineVertices = inner;
    return st;
}
}  // namespace

SweepStats Hierarchy::bu_fas(const Policy& pol, int n) {
    Impl& I = *impl_;
    const vc::Ctx x = vc_ctx(I, I.vcScratch);
    I.check_diag();
    std::vector<double2> wn(I.L + 1), wc(I.L + 1);
    for (int l = 0; l <= I.L; ++l) {  // omega_of (cycles.cpp:33-36) with succ = L - l
        const Cplx w = omega_unmasked(pol, I.L - l, n);
        wn[l] = make_double2(w.real(), w.imag());
        wc[l] = pol.hbMask ? make_double2(0.0, 0.0) : wn[l];
    }
    vc::bu_fas(I.p, x, wn.data(), wc.data(), pol.bpx ? 1 : 0);
    TMG_CUDA(cudaGetLastError());
    I.coarseUStale = false;
    return vc_norms(I, x);
}

SweepStats Hierarchy::textbook_add(Cplx omegaS, Cplx omegaCG) {
    Impl& I = *impl_;
    const vc::Ctx x = vc_ctx(I, I.vcScratch);
    I.check_diag();
    vc::textbook_add(I.p, x, make_double2(omegaS.real(), omegaS.imag()), make_double2(omegaCG.real(), omegaCG.imag()));
    TMG_CUDA(cudaGetLastError());
    return vc_norms(I, x);
}

int Hierarchy::dim() const { return impl_->p; }
int Hierarchy::levels() const { return impl_->amr ? impl_->amr->levels() : impl_->L; }

void Hierarchy::set_cell_marks(int level, const unsigned char* cells) {
    if (!impl_->amr) throw UnsupportedConfigError("set_cell_marks: the tree is not dynamically adaptive");
    impl_->amr->set_cell_marks(level, cells);
}

void Hierarchy::dyn_phase_ms(double* out6) const {
    for (int i = 0; i < 6; ++i) out6[i] = 0.0;
    if (!impl_->amr || !impl_->amr->dynamic()) return;
    for (int i = 0; i < 6; ++i) out6[i] = impl_->amr->phase_ms()[i];
}

long long Hierarchy::existing_vertices() const { return impl_->amr ? impl_->amr->existing_vertices() : 0; }

AmrMarkStats Hierarchy::mark() {
    if (!impl_->amr) throw UnsupportedConfigError("mark: the tree is not dynamically adaptive (h_max / h_min)");
    return impl_->amr->mark();
}

long long Hierarchy::lattice_size(int level) const {
    if (level < 0 || level > impl_->L) return 0;
    if (impl_->amr) {
        long long n = 1;
        for (int d = 0; d < impl_->p; ++d) n *= pow3i(level) + 1;
        return n;
    }
    return impl_->lv[level].n;
}

bool Hierarchy::get_flags(int level, unsigned char* flags, signed char* succ, unsigned char* cells) const {
    if (!impl_->amr) return false;
    impl_->amr->get_flags(level, flags, succ, cells);
    return true;
}

long long Hierarchy::hanging_vertices() const { return impl_->amr ? impl_->amr->hanging_vertices() : 0; }

long long Hierarchy::interior_fine_vertices() const {
    if (impl_->amr) return impl_->amr->leaf_vertices();
    long long n = 1;
    for (int d = 0; d < impl_->p; ++d) n *= pow3i(impl_->L) - 1;
    return n;
}

namespace {
double2* field_ptr(const dev::Lvl& v, const std::string& f) {
    if (f == "u") return v.u;
    if (f == "sc") return v.sc;
    if (f == "sf") return v.sf;
    if (f == "si") return v.si;
    if (f == "sinext") return v.sinext;
    if (f == "chi") return v.chi;
    if (f == "uhat") return v.uhat;
    if (f == "rhat") return v.rhat;
    if (f == "r") return v.r;
    return nullptr;
}
}  // namespace

void Hierarchy::get_field(int level, const std::string& name, double* host) const {
    Impl& I = *impl_;
    if (level < 0 || level > I.L) throw ConfigError("get_field: level out of range");
    if (I.amr) {
        I.amr->get_field(level, name, host);
        return;
    }
    // "<field>#<channel>": another channel's arrays (channels > 1)
    int ch = 0;
    std::string field = name;
    if (const auto hash = name.find('#'); hash != std::string::npos) {
        ch = std::stoi(name.substr(hash + 1));
        field = name.substr(0, hash);
        if (ch < 0 || ch >= I.prob.channels) throw ConfigError("get_field: channel out of range");
    }
    const dev::Lvl v = I.level(ch, level);
    if (I.slab() && level >= I.L - 1 && field != "diag")
        throw UnsupportedConfigError("get_field: a z-slab member holds a plane range of levels L and L-1 (SlabGroup)");
    if (field == "diag") {
        // host-side: per vertex the sum of A_aa over its existing cells
        const Cplx a = I.diagInterior[level] / static_cast<double>(1 << I.p);
        (void)a;
        double lap0, mas0;
        reference_pattern(I.p, 0, lap0, mas0);
        const Cplx Aaa = I.lapScale[level] * lap0 - I.prob.phi * I.massScale[level] * mas0;
        for (unsigned f = 0; f < v.n; ++f) {
            unsigned ff = f;
            int cells = 1;
            for (int d = 0; d < I.p; ++d) {
                const int x = static_cast<int>(ff % v.n1);
                ff /= v.n1;
                cells *= (x > 0 ? 1 : 0) + (x < static_cast<int>(v.m) ? 1 : 0);
            }
            Cplx dg(0.0);
            for (int i = 0; i < cells; ++i) dg += Aaa;
            host[2 * f] = dg.real();
            host[2 * f + 1] = dg.imag();
        }
        return;
    }
    if (field == "u" && level < I.L) I.materialize_coarse_u();
    if (level == I.L && I.fineDerived && (field == "u" || field == "sc")) {  // sc-free pass: u derived, sc = v - u
        Impl::Tmp t;
        double2* u = I.tmp_fine(t);
        I.derive_fine_u(u, 0, v.n);
        TMG_CUDA(cudaMemcpyAsync(host, u, static_cast<size_t>(v.n) * sizeof(double2), cudaMemcpyDeviceToHost, I.stream));
        std::vector<double> vv;
        if (field == "sc") {
            vv.resize(2 * static_cast<size_t>(v.n));
            if (I.prob.c64) {
                std::vector<float> vf(vv.size());
                TMG_CUDA(cudaMemcpyAsync(vf.data(), v.u, vf.size() * sizeof(float), cudaMemcpyDeviceToHost, I.stream));
                TMG_CUDA(cudaStreamSynchronize(I.stream));
                for (size_t i = 0; i < vv.size(); ++i) vv[i] = vf[i];
            } else {
                TMG_CUDA(cudaMemcpyAsync(vv.data(), v.u, vv.size() * sizeof(double), cudaMemcpyDeviceToHost, I.stream));
            }
        }
        TMG_CUDA(cudaStreamSynchronize(I.stream));
        if (field == "sc") {
            for (size_t i = 0; i < vv.size(); ++i) {
                const double r = vv[i] - host[i];
                host[i] = I.prob.c64 ? static_cast<double>(static_cast<float>(r)) : r;
            }
        }
        return;
    }
    if (level == I.L && I.prob.c64 && (field == "u" || field == "sc" || field == "chi")) {  // complex64 storage
        std::vector<float2> a(v.n), b;
        TMG_CUDA(cudaMemcpyAsync(a.data(), field == "chi" ? v.chi : field == "sc" ? v.sc : v.u,
                                 a.size() * sizeof(float2), cudaMemcpyDeviceToHost, I.stream));
        if (field == "u") {  // u = v - sc
            b.resize(v.n);
            TMG_CUDA(cudaMemcpyAsync(b.data(), v.sc, b.size() * sizeof(float2), cudaMemcpyDeviceToHost, I.stream));
        }
        TMG_CUDA(cudaStreamSynchronize(I.stream));
        for (size_t i = 0; i < a.size(); ++i) {
            host[2 * i] = static_cast<double>(a[i].x) - (b.empty() ? 0.0 : static_cast<double>(b[i].x));
            host[2 * i + 1] = static_cast<double>(a[i].y) - (b.empty() ? 0.0 : static_cast<double>(b[i].y));
        }
        return;
    }
    if (field == "u" && level == I.L && I.vForm()) {  // u = v - sc
        std::vector<double2> sc(v.n);
        TMG_CUDA(cudaMemcpyAsync(host, v.u, static_cast<size_t>(v.n) * sizeof(double2), cudaMemcpyDeviceToHost, I.stream));
        TMG_CUDA(cudaMemcpyAsync(sc.data(), v.sc, sc.size() * sizeof(double2), cudaMemcpyDeviceToHost, I.stream));
        TMG_CUDA(cudaStreamSynchronize(I.stream));
        for (size_t i = 0; i < sc.size(); ++i) {
            host[2 * i] -= sc[i].x;
            host[2 * i + 1] -= sc[i].y;
        }
        return;
    }
    double2* ptr = field_ptr(v, field);
    if (!ptr) {
        if (field == "uhat" || field == "chi" || field == "sf" || field == "si" || field == "sinext" || field == "r" ||
            field == "rhat") {
            std::fill(host, host + 2 * static_cast<size_t>(v.n), 0.0);
            return;
        }
        throw ConfigError("get_field: unknown field '" + field + "'");
    }
    TMG_CUDA(cudaMemcpyAsync(host, ptr, static_cast<size_t>(v.n) * sizeof(double2), cudaMemcpyDeviceToHost, I.stream));
    TMG_CUDA(cudaStreamSynchronize(I.stream));
}

void Hierarchy::set_field(int level, const std::string& field, const double* host) {
    if (impl_->amr) throw UnsupportedConfigError("set_field is not available on adaptive trees");
    Impl& I = *impl_;
    if (level < 0 || level > I.L) throw ConfigError("set_field: level out of range");
    const dev::Lvl& v = I.lv[level];
    double2* ptr = field_ptr(v, field);
    if (!ptr) throw ConfigError("set_field: unknown field '" + field + "'");
    if (level == I.L && I.vForm() && (field == "u" || field == "sc")) {
        // the device keeps v = u + sc on the finest level
        I.split_fine(false);
        std::vector<double> u(2 * static_cast<size_t>(v.n)), sc(2 * static_cast<size_t>(v.n));
        get_field(level, "u", u.data());
        get_field(level, "sc", sc.data());
        const double* nu = field == "u" ? host : u.data();
        const double* ns = field == "sc" ? host : sc.data();
        std::vector<double> vv(u.size());
        for (size_t i = 0; i < vv.size(); ++i) vv[i] = nu[i] + ns[i];
        if (I.prob.c64) {  // complex64 storage
            std::vector<float> fv(vv.size()), fs(vv.size());
            for (size_t i = 0; i < vv.size(); ++i) {
                fv[i] = static_cast<float>(vv[i]);
                fs[i] = static_cast<float>(ns[i]);
            }
            TMG_CUDA(cudaMemcpyAsync(v.u, fv.data(), fv.size() * sizeof(float), cudaMemcpyHostToDevice, I.stream));
            TMG_CUDA(cudaMemcpyAsync(v.sc, fs.data(), fs.size() * sizeof(float), cudaMemcpyHostToDevice, I.stream));
            TMG_CUDA(cudaStreamSynchronize(I.stream));
            return;
        }
        TMG_CUDA(cudaMemcpyAsync(v.u, vv.data(), vv.size() * sizeof(double), cudaMemcpyHostToDevice, I.stream));
        TMG_CUDA(cudaMemcpyAsync(v.sc, ns, vv.size() * sizeof(double), cudaMemcpyHostToDevice, I.stream));
        TMG_CUDA(cudaStreamSynchronize(I.stream));
        return;
    }
    if (level == I.L && I.prob.c64) throw UnsupportedConfigError("set_field: complex64 fine level holds u / sc only");
    TMG_CUDA(cudaMemcpyAsync(ptr, host, static_cast<size_t>(v.n) * sizeof(double2), cudaMemcpyHostToDevice, I.stream));
    TMG_CUDA(cudaStreamSynchronize(I.stream));
}

namespace {
// callers reset sc afterwards: plain u injection; fineD: the fine level's u as
// complex128 (complex64 storage) instead of the level itself
template <int P>
void inject_up(Hierarchy::Impl& I, int ch = 0, const dev::Lvl* fineD = nullptr) {
    for (int l = I.L - 1; l >= 1; --l)
        dev::k_inject_u<P><<<I.blocks_for(I.lv[l].n), 256, 0, I.stream>>>(
            I.level(ch, l), (l == I.L - 1 && fineD) ? *fineD : I.level(ch, l + 1), 0);
}

// complex64 fine level: a complex128 stand-in whose u is written by the caller,
// then stored as complex64 (store_fine_u) and injected from (inject_up's fineD)
dev::Lvl c64_stage(Hierarchy::Impl& I, Hierarchy::Impl::Tmp& t) {
    dev::Lvl Fd = I.lv[I.L];
    Fd.u = I.tmp_fine(t);
    return Fd;
}
void store_fine_u(Hierarchy::Impl& I, const dev::Lvl& Fd) {
    const dev::Lvl& F = I.lv[I.L];
    dev::k_d2f<<<I.blocks_for(F.n), 256, 0, I.stream>>>(Fd.u, reinterpret_cast<float2*>(F.u), F.n);
    TMG_CUDA(cudaGetLastError());
}
}  // namespace

struct HierarchyAccess {
    static void reset_pipeline(Hierarchy::Impl& I) {  // reset_pipeline_state, cycles.cpp:843-853
        for (int ch = 0; ch < I.prob.channels; ++ch)
            for (int l = 0; l <= I.L; ++l) {
                const dev::Lvl v = I.level(ch, l);
                const size_t bytes = static_cast<size_t>(v.n) * (l == I.L ? I.fine_elem() : sizeof(double2));
                for (double2* ptr : {v.sc, v.sf, v.si, v.sinext, v.uhat})
                    if (ptr) TMG_CUDA(cudaMemsetAsync(ptr, 0, bytes, I.stream));
            }
    }
};

void Hierarchy::set_fine_interior_u(const double* host) {
    if (impl_->amr) throw UnsupportedConfigError("set_fine_interior_u is not available on adaptive trees");
    Impl& I = *impl_;
    Impl::Tmp t;
    const dev::Lvl F = I.prob.c64 ? c64_stage(I, t) : I.lv[I.L];
    const dev::Lvl* fineD = I.prob.c64 ? &F : nullptr;
    const long long ni = interior_fine_vertices();
    double2* tmp = nullptr;
    TMG_CUDA(cudaMalloc(&tmp, static_cast<size_t>(ni) * sizeof(double2)));
    TMG_CUDA(cudaMemcpyAsync(tmp, host, static_cast<size_t>(ni) * sizeof(double2), cudaMemcpyHostToDevice, I.stream));
    if (I.p == 1) dev::k_scatter_interior<1><<<I.blocks_for(F.n), 256, 0, I.stream>>>(F, tmp);
    else if (I.p == 2) dev::k_scatter_interior<2><<<I.blocks_for(F.n), 256, 0, I.stream>>>(F, tmp);
    else dev::k_scatter_interior<3><<<I.blocks_for(F.n), 256, 0, I.stream>>>(F, tmp);
    if (fineD) store_fine_u(I, F);
    if (I.p == 1) inject_up<1>(I, 0, fineD);
    else if (I.p == 2) inject_up<2>(I, 0, fineD);
    else inject_up<3>(I, 0, fineD);
    HierarchyAccess::reset_pipeline(I);
    I.fineDerived = false;
    TMG_CUDA(cudaStreamSynchronize(I.stream));
    cudaFree(tmp);
}

void Hierarchy::set_random_initial_guess(std::uint64_t seed) {
    Impl& I = *impl_;
    if (I.amr) {
        I.amr->set_random_initial_guess(seed);
        return;
    }
    for (int ch = 0; ch < I.prob.channels; ++ch) {
        Impl::Tmp t;
        const dev::Lvl F = I.prob.c64 ? c64_stage(I, t) : I.level(ch, I.L);
        const dev::Lvl* fineD = I.prob.c64 ? &F : nullptr;
        if (I.p == 1) dev::k_random_fine<1><<<I.blocks_for(F.n), 256, 0, I.stream>>>(F, seed, ch);
        else if (I.p == 2) dev::k_random_fine<2><<<I.blocks_for(F.n), 256, 0, I.stream>>>(F, seed, ch);
        else dev::k_random_fine<3><<<I.blocks_for(F.n), 256, 0, I.stream>>>(F, seed, ch);
        if (fineD) store_fine_u(I, F);
        if (I.p == 1) inject_up<1>(I, ch, fineD);
        else if (I.p == 2) inject_up<2>(I, ch, fineD);
        else inject_up<3>(I, ch, fineD);
        TMG_CUDA(cudaStreamSynchronize(I.stream));
    }
    HierarchyAccess::reset_pipeline(I);
    I.fineDerived = false;
    TMG_CUDA(cudaStreamSynchronize(I.stream));
}

void Hierarchy::set_fine_rhs(const double* hostNodalChi) {
    if (impl_->amr) throw UnsupportedConfigError("set_fine_rhs is not available on adaptive trees");
    Impl& I = *impl_;
    const dev::Lvl& F = I.lv[I.L];
    TMG_CUDA(cudaMemcpyAsync(I.chiNodal, hostNodalChi, static_cast<size_t>(F.n) * sizeof(double2),
                             cudaMemcpyHostToDevice, I.stream));
    I.load_vector_dispatch();
    for (int ch = 1; ch < I.prob.channels; ++ch)  // same fields on every channel (runner.cpp:152)
        TMG_CUDA(cudaMemcpyAsync(I.chanLv[ch - 1][I.L].chi, I.lv[I.L].chi,
                                 static_cast<size_t>(I.lv[I.L].n) * sizeof(double2), cudaMemcpyDeviceToDevice,
                                 I.stream));
    TMG_CUDA(cudaStreamSynchronize(I.stream));
}

// FNV-1a over the bit patterns (sign of zero folded), tests/golden/make_goldens.py
std::uint64_t fnv_hash(const std::vector<double>& buf) {
    std::uint64_t h = 1469598103934665603ull;
    for (double x : buf) {
        const double y = x + 0.0;
        std::uint64_t bits;
        std::memcpy(&bits, &y, 8);
        for (int b = 0; b < 8; ++b) {
            h ^= (bits >> (8 * b)) & 0xffu;
            h *= 1099511628211ull;
        }
    }
    return h;
}

std::uint64_t Hierarchy::field_hash(int level, const std::string& field) const {
    if (impl_->amr) return impl_->amr->field_hash(level, field);
    const long long n = lattice_size(level);
    std::vector<double> buf(2 * static_cast<size_t>(n));
    get_field(level, field, buf.data());
    return fnv_hash(buf);
}

int fused3_resident_blocks(int smCount) { return fused3::resident_blocks(smCount); }

DeviceScope::DeviceScope(int device) : want(device) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != want) cudaSetDevice(want);
}
DeviceScope::~DeviceScope() {
    if (prev >= 0 && prev != want) cudaSetDevice(prev);
}

void test_divdc3(const double* x, const double* y, double* out, long long n) {
    std::vector<dev::DivConst> k(static_cast<size_t>(n));
    for (long long i = 0; i < n; ++i) k[static_cast<size_t>(i)] = div_const(Cplx(y[2 * i], y[2 * i + 1]));
    double2 *dx = nullptr, *dout = nullptr;
    dev::DivConst* dk = nullptr;
    TMG_CUDA(cudaMalloc(&dx, n * sizeof(double2)));
    TMG_CUDA(cudaMalloc(&dout, n * sizeof(double2)));
    TMG_CUDA(cudaMalloc(&dk, n * sizeof(dev::DivConst)));
    TMG_CUDA(cudaMemcpy(dx, x, n * sizeof(double2), cudaMemcpyHostToDevice));
    TMG_CUDA(cudaMemcpy(dk, k.data(), n * sizeof(dev::DivConst), cudaMemcpyHostToDevice));
    dev::k_test_divdc3<<<64, 256>>>(dx, dk, dout, n);
    TMG_CUDA(cudaGetLastError());
    TMG_CUDA(cudaMemcpy(out, dout, n * sizeof(double2), cudaMemcpyDeviceToHost));
    cudaFree(dx);
    cudaFree(dout);
    cudaFree(dk);
}

// FMG unfolding: the reference refines every leaf cell in
// sorted key order (spacetree.cpp:272-329), giving new vertices p-linearly
// prolonged u (create_vertex_if_missing, :245-270) and zero payload, keeps the
// existing levels' u / sc / sf / si, and re-classifies (succ = L+1-l).  The
// canonical-parent prolongation used here equals the creating cell's for
// every vertex (coinciding components are exact copies, transfer.cpp:26-38).
void Hierarchy::unfold(bool toComplex64) {
    if (impl_->amr) throw UnsupportedConfigError("FMG unfolding is not available on adaptive trees");
    if (impl_->prob.c64) throw UnsupportedConfigError("FMG unfolding: only the final level may be complex64");
    Impl& old = *impl_;
    Problem p2 = old.prob;
    p2.levels = old.L + 1;
    p2.c64 = toComplex64;
    if (p2.rhsLattice < 0) p2.rhsLattice = p2.levels;
    if (old.fineDerived) {  // the old finest level becomes a coarse level: (u, sc) with the derived u
        old.split_fine(true);
    } else if (old.vForm()) {  // back to (u, sc)
        const dev::Lvl& F = old.lv[old.L];
        dev::k_vform_to_u<<<old.blocks_for(F.n), 256, 0, old.stream>>>(F.u, F.sc, F.n);
        TMG_CUDA(cudaGetLastError());
    }
    TMG_CUDA(cudaStreamSynchronize(old.stream));
    Hierarchy deeper(p2);
    Impl& nw = *deeper.impl_;
    const int L = old.L;
    for (int l = 0; l <= L; ++l) {
        const dev::Lvl& a = old.lv[l];
        const dev::Lvl& b = nw.lv[l];
        const size_t bytes = static_cast<size_t>(a.n) * sizeof(double2);
        auto copy = [&](double2* dst, const double2* src) {
            if (dst && src) TMG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, nw.stream));
        };
        copy(b.u, a.u);
        copy(b.sc, a.sc);
        copy(b.sf, a.sf);
        copy(b.si, a.si);
        copy(b.sinext, a.sinext);
    }
    Impl::Tmp t;
    // complex64 fine level: prolonged in complex128 into a stand-in, then stored as complex64
    const dev::Lvl F = nw.prob.c64 ? c64_stage(nw, t) : nw.lv[L + 1];
    if (nw.p == 1) dev::k_prolong_new<1><<<nw.blocks_for(F.n), 256, 0, nw.stream>>>(F, nw.lv[L], 0u, F.n);
    else if (nw.p == 2) dev::k_prolong_new<2><<<nw.blocks_for(F.n), 256, 0, nw.stream>>>(F, nw.lv[L], 0u, F.n);
    else dev::k_prolong_new<3><<<nw.blocks_for(F.n), 256, 0, nw.stream>>>(F, nw.lv[L], 0u, F.n);
    TMG_CUDA(cudaGetLastError());
    if (nw.prob.c64) store_fine_u(nw, F);
    nw.coarseUStale = nw.prob.fast;
    TMG_CUDA(cudaStreamSynchronize(nw.stream));
    std::swap(impl_, deeper.impl_);
}

void Hierarchy::time_cycles(const Policy& pol, int n0, int count, bool flushL2, double* out4) {
    Impl& I = *impl_;
    if (I.amr) {
        I.amr->time_cycles(pol, n0, count, out4);
        return;
    }
    I.check_diag();
    if (flushL2 && !I.flushBuf) {
        I.flushN = (256ull << 20) / sizeof(double4);  // 256 MB > 126 MB L2
        I.flushBuf = I.alloc<double4>(I.flushN);
    }
    double totalMs = 0.0, fineMs = 0.0;
    I.backToBack = true;
    struct Reset {
        bool& b;
        ~Reset() { b = false; }
    } reset{I.backToBack};
    for (int i = 0; i < count; ++i) {
        if (flushL2) dev::k_flush<<<4 * I.smCount, 256, 0, I.stream>>>(I.flushBuf, I.flushN, 0.0);
        TMG_CUDA(cudaEventRecord(I.ev0, I.stream));
        I.run_cycle(pol, n0 + i, true);
        TMG_CUDA(cudaEventRecord(I.ev1, I.stream));
        TMG_CUDA(cudaEventSynchronize(I.ev1));
        float ms = 0.f, fms = 0.f;
        TMG_CUDA(cudaEventElapsedTime(&ms, I.ev0, I.ev1));
        TMG_CUDA(cudaEventElapsedTime(&fms, I.evf0, I.evf1));
        totalMs += ms;
        fineMs += fms;
    }
    out4[0] = totalMs;
    out4[1] = count ? fineMs / count : 0.0;
    out4[2] = 0.0;
    out4[3] = static_cast<double>(I.launches_per_cycle());
}

void Hierarchy::e2e_step(const Policy& pol, int n, const double* hostChi, double* out3) {
    if (impl_->amr) throw UnsupportedConfigError("e2e_step is not available on adaptive trees");
    Impl& I = *impl_;
    const dev::Lvl& F = I.lv[I.L];
    TMG_CUDA(cudaMemcpyAsync(I.chiNodal, hostChi, static_cast<size_t>(F.n) * sizeof(double2), cudaMemcpyHostToDevice,
                             I.stream));
    I.load_vector_dispatch();
    const SweepStats st = I.cycle(pol, n);
    out3[0] = st.maxNorm;
    out3[1] = st.euclidNorm;
    out3[2] = st.hNorm;
}

}  // namespace tmg
#include "slabs.inc"
