// Static adaptive spacetree cycle (exact precision).  See amr.hpp for the
// layout and the ordering rules; the per-vertex semantics follow
//   touch_first      proj/src/cycles.cpp:102-141
//   create_hanging   proj/src/cycles.cpp:143-171
//   enter_cell       proj/src/cycles.cpp:173-220 (residual, diag, leaf loads)
//   touch_last       proj/src/cycles.cpp:243-303
//   destroy_hanging  proj/src/cycles.cpp:305-321
// and the classification of proj/src/spacetree.cpp:438-489.

#include "amr.hpp"

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <array>
#include <chrono>
#include <cstdio>
#include <thread>

#include "exact_ops.cuh"
#include "lattice.cuh"

namespace tmg {

#define AMR_CUDA(call)                                                                          \
    do {                                                                                        \
        cudaError_t err_ = (call);                                                              \
        if (err_ != cudaSuccess) {                                                              \
            if (err_ == cudaErrorMemoryAllocation)                                              \
                throw CapacityError(std::string("device memory exhausted: ") + #call);          \
            throw CudaError(std::string("CUDA error ") + cudaGetErrorString(err_) + " at " + #call); \
        }                                                                                       \
    } while (0)

namespace adev {

using namespace dev;

struct ALvl {
    double2 *u, *sc, *sf, *si, *sinext, *chi, *uhat, *rhat, *r, *nodal;
    const unsigned char* vflag;
    const unsigned char* cflag;
    const unsigned char* estar;
    const signed char* succ;
    const unsigned* list;  // existing vertices: interior non-hanging first, then the rest
    unsigned nlist;
    // dynamic adaptivity (dyn.hpp): sweep tables beyond the static ones, the
    // classification after the sweep, and the mark pass's per-vertex data
    double2* dg;                  // accumulated operator diagonal (mark's convergence indicator)
    const unsigned char* fmask;   // finish cells (bit e: cell = v - 1 + bits(e))
    const unsigned char* skip;    // cells entered before the vertex was created
    const int* xoff;              // special vertices: first slot of their finish values in extras
    double2* extras;              // r-hat at each finish of a special vertex, in traversal order
    const unsigned* slist;        // special vertices
    unsigned nslist;
    const unsigned char* fflag;   // classification after the sweep (amr::k* bits)
    const unsigned char* fcell;   // cells after the sweep (kCellExists | kCellRefined)
    double* feat;                 // mark: feature s per candidate
    double* ind;                  // mark: |r| / |diag|
    unsigned char* vmark;         // mark: 1 refine, 2 erase, 4 candidate
    unsigned* cmark;              // mark: per cell, dyn::kRM | dyn::kEM
    unsigned* mlist;              // mark: cells whose mark flipped (cell | kind << 31), for the host
    unsigned* mcount;
    int lo[3];
    int n1[3];
    unsigned n;
    int m;
    int level;
};

struct AResArgs {
    ALvl lv, par;
    LevelConst k;
    double2 wTab[12];  // omega_unmasked(pol, succ, n) for succ = 0..11
    double2 dgTab[9];  // diag after k cells: ((A_aa + A_aa) + ...) k times (zero_accumulators, then +=)
    int ellMin, bpx, hb;
    double* partials;
    double2 kAsm[8];  // precision = fast: assembled stencil entry per offset class s, 2^(P - |s|) A[s]
    double2 invDiag;  // precision = fast: 1 / (the diagonal after 2^P cells), Jacobi as a complex multiply
};

template <int P>
__device__ __forceinline__ void aunflat(unsigned f, const ALvl& c, int* g) {
#pragma unroll
    for (int d = 0; d < P; ++d) {
        g[d] = c.lo[d] + static_cast<int>(f % static_cast<unsigned>(c.n1[d]));
        f /= static_cast<unsigned>(c.n1[d]);
    }
}

// box position of lattice point g, -1 outside the box
template <int P>
__device__ __forceinline__ int aflat(const ALvl& c, const int* g) {
    int f = 0, s = 1;
#pragma unroll
    for (int d = 0; d < P; ++d) {
        const int x = g[d] - c.lo[d];
        if (x < 0 || x >= c.n1[d]) return -1;
        f += x * s;
        s *= c.n1[d];
    }
    return f;
}

// aunflat with the divisions by the box extents as multiply-high by
// M = ceil(2^64 / n1) (exact for 32-bit operands; Lemire & Kaser 2019): the two
// magic numbers are formed once per thread, the per-vertex cost is two
// 64-bit multiply-highs instead of two 32-bit divisions and remainders.
template <int P>
struct FastUnflat {
    unsigned long long m0 = 0, m1 = 0;
    unsigned n0 = 1, n1 = 1;
    int lo[3] = {0, 0, 0};
    __device__ explicit FastUnflat(const ALvl& c) {
        n0 = static_cast<unsigned>(c.n1[0]);
        n1 = P >= 2 ? static_cast<unsigned>(c.n1[1]) : 1u;
        m0 = n0 > 1 ? ~0ull / n0 + 1ull : 0ull;  // n = 1: quotient is f itself (handled below)
        m1 = n1 > 1 ? ~0ull / n1 + 1ull : 0ull;
#pragma unroll
        for (int d = 0; d < P; ++d) lo[d] = c.lo[d];
    }
    __device__ __forceinline__ void operator()(unsigned f, int* g) const {
        const unsigned q0 = n0 > 1 ? static_cast<unsigned>(__umul64hi(m0, f)) : f;
        g[0] = lo[0] + static_cast<int>(f - q0 * n0);
        if (P == 1) return;
        if (P == 2) {
            g[1] = lo[1] + static_cast<int>(q0);  // aunflat takes q0 % n1[1]; q0 < n1[1] inside the box
            return;
        }
        const unsigned q1 = n1 > 1 ? static_cast<unsigned>(__umul64hi(m1, q0)) : q0;
        g[1] = lo[1] + static_cast<int>(q0 - q1 * n1);
        // the last axis: aunflat takes q1 % n1[2]; q1 < n1[2] for every index inside the box
        g[2] = lo[2] + static_cast<int>(q1);
    }
};

// Grid-stride walk over a level's vertex list with the list entry loaded two
// iterations ahead and the vertex's flags one ahead: the per-vertex chain
// list -> flags -> data was three dependent memory latencies per iteration.
struct ListWalk {
    const unsigned* list;
    const unsigned char* vflag;
    unsigned n, stride;
    unsigned f = 0, fN = 0;  // this / the next iteration's vertex
    unsigned char vf = 0;    // this iteration's flags
    __device__ explicit ListWalk(const ALvl& c) : list(c.list), vflag(c.vflag), n(c.nlist), stride(gridDim.x * blockDim.x) {}
    __device__ unsigned first() {
        const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
        if (i < n) {
            f = __ldg(list + i);
            vf = __ldg(vflag + f);
        }
        if (i + stride < n) fN = __ldg(list + i + stride);
        return i;
    }
    // issue the loads of the iterations after i (call once per iteration, before any `continue`)
    __device__ void prefetch(unsigned i) {
        const unsigned i1 = i + stride, i2 = i1 + stride;
        unsigned char vfN = 0;
        if (i1 < n) vfN = __ldg(vflag + fN);
        const unsigned fNN = i2 < n ? __ldg(list + i2) : 0u;
        pendF = fN;
        pendVf = vfN;
        fN = fNN;
    }
    __device__ unsigned next(unsigned i) {
        f = pendF;
        vf = pendVf;
        return i + stride;
    }
    unsigned pendF = 0;
    unsigned char pendVf = 0;
};

// ---- top-down: touch_first / create_hanging ----------------------------------
#ifndef TMG_AMR_TD_MINB
#define TMG_AMR_TD_MINB 3
#endif
template <int P, bool STATIC = false, bool FAST = false>
// FAST (precision = fast on static trees): the regular vertices' interpolation as
// fma(rel / 3, c1 - c0, c0) -- no exact-copy select (weight 0 copies c0), within rounding
// finestStatic: the finest level of a static tree, where the residual pass
// restages sc of every non-hanging vertex and no finer top-down reads it -- the
// top-down's sc is dead there and not stored (the sum still feeds u)
__global__ void __launch_bounds__(256, TMG_AMR_TD_MINB) k_amr_topdown(ALvl c, ALvl pr, int bpx, int finestStatic = 0) {
    ListWalk w(c);
    const FastUnflat<P> unflat(c);
    for (unsigned i = w.first(); i < c.nlist; i = w.next(i)) {
        const unsigned f = w.f;
        const unsigned char vf = w.vf;
        w.prefetch(i);
        if (!(vf & amr::kExists)) continue;
        const bool bnd = vf & amr::kBoundary, cp = vf & amr::kCPoint, hang = vf & amr::kHanging;
        if (STATIC && c.level > 0 && (vf & amr::kParentsAll) && !hang) {
            // Static tree, every parent corner present, regular vertex: the same values
            // and operations as the general path below with less bookkeeping.  The parent
            // cell is taken as q = g / 3 with rel = g % 3 in {0, 1, 2} (at the upper
            // boundary the general path's (q - 1, rel 3) names the same corner q as
            // (q, rel 0)); an axis with rel 0 reads its lower corner twice (stride 0)
            // and copies it, so the interpolation needs one exact-copy select instead
            // of two and no existence look-ups.
            int g[P];
            unflat(f, g);
            int q[P], rel[P];
#pragma unroll
            for (int d = 0; d < P; ++d) {
                q[d] = g[d] / 3;
                rel[d] = g[d] - 3 * q[d];
            }
            const int p0 = aflat<P>(pr, q);
            const int s0 = rel[0] ? 1 : 0;
            const int s1 = (P >= 2 && rel[P >= 2 ? 1 : 0]) ? pr.n1[0] : 0;
            const int s2 = (P == 3 && rel[P == 3 ? 2 : 0]) ? pr.n1[0] * pr.n1[1] : 0;
            auto prolong012 = [&](const double2* __restrict__ src) {
                double2 v[1 << P];
#pragma unroll
                for (int e = 0; e < (1 << P); ++e)
                    v[e] = src[p0 + (e & 1) * s0 + ((e >> 1) & 1) * s1 + ((e >> 2) & 1) * s2];
#pragma unroll
                for (int d = 0; d < P; ++d) {
                    const double w0 = rel[d] == 1 ? (2.0 / 3.0) : (1.0 / 3.0);
                    const double w1 = rel[d] == 1 ? (1.0 / 3.0) : (2.0 / 3.0);
#pragma unroll
                    for (int k = 0; k < (1 << (P - 1 - d)); ++k) {
                        if (FAST) {
                            const double wr = rel[d] == 0 ? 0.0 : w1;
                            v[k] = make_double2(fma(wr, v[2 * k + 1].x - v[2 * k].x, v[2 * k].x),
                                                fma(wr, v[2 * k + 1].y - v[2 * k].y, v[2 * k].y));
                        } else {
                            const double2 r = xadd(xscale(w0, v[2 * k]), xscale(w1, v[2 * k + 1]));  // lerp_rel
                            v[k] = rel[d] == 0 ? v[2 * k] : r;
                        }
                    }
                }
                return v[0];
            };
            const double2 pu = prolong012(pr.u);
            double2 sc = xadd(c.sc[f], prolong012(pr.sc));
            if (bpx && !cp) sc = xsub(sc, prolong012(pr.si));
            const double2 sf = c.sf ? c.sf[f] : cz();
            double2 u = xadd(c.u[f], xadd(sc, sf));
            double2 uh = xsub(u, pu);
            if (bnd) {
                u = cz();
                uh = cz();
            }
            c.u[f] = u;
            if (!finestStatic) c.sc[f] = sc;
            c.uhat[f] = uh;
            if (c.sf) c.sf[f] = cz();
            continue;
        }
        if (c.level == 0) {  // cycles.cpp:128-133
            double2 u = xadd(c.u[f], xadd(c.sc[f], c.sf ? c.sf[f] : cz()));
            if (bnd) u = cz();
            c.u[f] = u;
            c.uhat[f] = cz();
            if (c.sf) c.sf[f] = cz();
            continue;
        }
        int g[P];
        aunflat<P>(f, c, g);
        int q[P], rel[P];
#pragma unroll
        for (int d = 0; d < P; ++d) {
            q[d] = min(g[d] / 3, pr.m - 1);  // parent_stencil, spacetree.cpp:164-174
            rel[d] = g[d] - 3 * q[d];
        }
        // parent corners (find_vertex: absent -> 0); one field at a time keeps
        // the register footprint small
        int pfs[1 << P];
        if (STATIC && (vf & amr::kParentsAll)) {  // every parent corner exists: box strides
            const int p0 = aflat<P>(pr, q);
            const int s1 = P >= 2 ? pr.n1[0] : 0, s2 = P == 3 ? pr.n1[0] * pr.n1[1] : 0;
#pragma unroll
            for (int e = 0; e < (1 << P); ++e) pfs[e] = p0 + (e & 1) + ((e >> 1) & 1) * s1 + ((e >> 2) & 1) * s2;
        } else {
#pragma unroll
            for (int e = 0; e < (1 << P); ++e) {
                int pi[P];
#pragma unroll
                for (int d = 0; d < P; ++d) pi[d] = q[d] + ((e >> d) & 1);
                const int pf = aflat<P>(pr, pi);
                pfs[e] = (pf >= 0 && (pr.vflag[pf] & amr::kExists)) ? pf : -1;
            }
        }
        auto parent_prolong = [&](const double2* src) {
            double2 v[1 << P];
#pragma unroll
            for (int e = 0; e < (1 << P); ++e) v[e] = pfs[e] >= 0 ? src[pfs[e]] : cz();
            return prolong<P>(v, rel);
        };
        const double2 pu = parent_prolong(pr.u);
        if (!STATIC && (vf & dyn::kSCreated)) {  // create_vertex_if_missing inside the sweep (spacetree.cpp:245-270, 310-318)
            c.u[f] = pu;
            c.sc[f] = cz();
            c.uhat[f] = cz();
            if (c.sf) c.sf[f] = cz();
            if (c.si) c.si[f] = cz();
            if (c.sinext) c.sinext[f] = cz();
            continue;
        }
        const double2 ps = parent_prolong(pr.sc);
        if (hang) {  // create_hanging
            double2 u = pu, sc = ps;
            if (bpx && !cp) sc = xsub(sc, parent_prolong(pr.si));
            if (bnd) {
                u = cz();
                sc = cz();
            }
            c.u[f] = u;
            c.sc[f] = sc;
            c.uhat[f] = cz();
            if (c.sf) c.sf[f] = cz();
            if (c.si) c.si[f] = cz();
            if (c.sinext) c.sinext[f] = cz();
            continue;
        }
        double2 sc = xadd(c.sc[f], ps);
        if (bpx && !cp) sc = xsub(sc, parent_prolong(pr.si));
        const double2 sf = c.sf ? c.sf[f] : cz();
        double2 u = xadd(c.u[f], xadd(sc, sf));
        double2 uh = xsub(u, pu);
        if (bnd) {
            u = cz();
            uh = cz();
        }
        c.u[f] = u;
        if (!(STATIC && finestStatic)) c.sc[f] = sc;
        c.uhat[f] = uh;
        if (c.sf) c.sf[f] = cz();
    }
}

// ---- chi: leaf loads and restriction in traversal time order ---------------
// r-hat value fine vertex vf restricts from its finish in the child cell where
// it is corner ec; false if it does not finish there.  A special vertex
// (dynamic adaptivity) may finish in several cells, in traversal (Morton)
// order of the cells around it, each with its own value.
template <int P>
__device__ __forceinline__ bool fine_finish_value(const ALvl& fl, int vf, int ec, double2& val) {
    constexpr int NC = 1 << P;
    if (fl.fmask && (fl.vflag[vf] & dyn::kSSpecial)) {
        const unsigned char fm = fl.fmask[vf];
        const int ep = (~ec) & (NC - 1);
        if (!((fm >> ep) & 1)) return false;
        int g[P];
        aunflat<P>(static_cast<unsigned>(vf), fl, g);
        const int pid = perm_id<P>(g);
        int k = 0;
        for (int i = 0; i < NC; ++i) {
            const int e = perm_cell(P, pid, i);
            if (e == ep) break;
            k += (fm >> e) & 1;
        }
        val = fl.extras[fl.xoff[vf] + k];
        return true;
    }
    if (fl.estar[vf] != ec) return false;
    val = fl.rhat[vf];
    return true;
}

// chi contribution of one existing cell around g (g is corner a of it):
// the leaf load on entering it (kernels.cpp:69-87), or, for a cell refined on
// entry, the restriction of the fine vertices touched last inside it, in
// child order, then by their corner index in the child (visit_cell's finish loop)
template <int P>
__device__ __forceinline__ void cell_chi(double2& acc, const ALvl& c, const ALvl& fl, const LevelConst& k,
                                         const double* __restrict__ w5, const int* g, const int* cell, int a,
                                         unsigned char cfl, int restrictOn) {
    constexpr int NC = 1 << P;
    constexpr int NT = P == 1 ? 3 : P == 2 ? 9 : 27;
    if (!(cfl & amr::kCellRefined)) {
        double2 acc2 = cz();
#pragma unroll
        for (int bb = 0; bb < NC; ++bb) {
            int vb[P];
#pragma unroll
            for (int d = 0; d < P; ++d) vb[d] = cell[d] + ((bb >> d) & 1);
            acc2 = xadd(acc2, xscale(k.M[a ^ bb], c.nodal[aflat<P>(c, vb)]));
        }
        acc = xadd(acc, xmul(k.massScale, acc2));
        return;
    }
    if (!restrictOn) return;
    if (!fl.fmask) {
        // static tree (no special vertices): the 3^P fine vertices of this cell
        // inside g's restriction window (w = v - 3 cell in [wlo, wlo + 2] per axis)
        // have their finish corners loaded once, packed 4 bits each (15: absent /
        // off the domain); then (child t, corner ec) ascending as below, touching
        // only the pairs whose vertex lies in the window
        int wlo[3] = {0, 0, 0};
#pragma unroll
        for (int d = 0; d < P; ++d) wlo[d] = cell[d] == g[d] - 1 ? 1 : 0;
        constexpr int NW = P == 1 ? 3 : P == 2 ? 9 : 27;
        unsigned long long pk[2] = {0ull, 0ull};
        int vfw[NW];
#pragma unroll
        for (int pw = 0; pw < NW; ++pw) {
            int v[P];
            int rr = pw;
            bool in = true;
#pragma unroll
            for (int d = 0; d < P; ++d) {
                v[d] = 3 * cell[d] + wlo[d] + rr % 3;
                rr /= 3;
                in &= (v[d] >= 1) & (v[d] <= fl.m - 1);
            }
            const int vf = in ? aflat<P>(fl, v) : -1;
            vfw[pw] = vf;
            const unsigned e = vf >= 0 ? static_cast<unsigned>(fl.estar[vf]) & 15u : 15u;
            pk[pw >> 4] |= static_cast<unsigned long long>(e) << (4 * (pw & 15));
        }
        for (int t = 0; t < NT; ++t) {
            int j[P];
            int tt = t;
            unsigned must0 = 0, must1 = 0;
#pragma unroll
            for (int d = 0; d < P; ++d) {
                j[d] = tt % 3;
                tt /= 3;
                const int dj = j[d] - wlo[d];  // i_d = dj + ec_d must lie in [0, 2]
                if (dj < 0) must1 |= 1u << d;
                if (dj > 1) must0 |= 1u << d;
            }
            const unsigned freeb = ~(must0 | must1) & static_cast<unsigned>(NC - 1);
            unsigned sub = 0;
            do {  // ec = must1 | sub, ascending
                const int ec = static_cast<int>(must1 | sub);
                int pw = 0, mul = 1, code = 0, cm = 1;
#pragma unroll
                for (int d = 0; d < P; ++d) {
                    const int bit = (ec >> d) & 1;
                    pw += (j[d] - wlo[d] + bit) * mul;
                    mul *= 3;
                    code += (3 * cell[d] + j[d] + bit - 3 * g[d] + 2) * cm;
                    cm *= 5;
                }
                const unsigned e = static_cast<unsigned>(pk[pw >> 4] >> (4 * (pw & 15))) & 15u;
                if (e == static_cast<unsigned>(ec)) acc = xadd(acc, xscale(w5[code], fl.rhat[vfw[pw]]));
                sub = (sub - freeb) & freeb;
            } while (sub);
        }
        return;
    }
    for (int t = 0; t < NT; ++t) {
        int j[P];
        int tt = t;
#pragma unroll
        for (int d = 0; d < P; ++d) {
            j[d] = tt % 3;
            tt /= 3;
        }
        for (int ec = 0; ec < NC; ++ec) {
            int v[P];
            int code = 0, mul = 1;
            bool in = true;
#pragma unroll
            for (int d = 0; d < P; ++d) {
                v[d] = 3 * cell[d] + j[d] + ((ec >> d) & 1);
                const int off = v[d] - 3 * g[d];
                in &= (off >= -2) & (off <= 2) & (v[d] >= 1) & (v[d] <= fl.m - 1);
                code += (off + 2) * mul;
                mul *= 5;
            }
            if (!in) continue;
            const int vf = aflat<P>(fl, v);
            if (vf < 0) continue;
            double2 val;
            if (!fine_finish_value<P>(fl, vf, ec, val)) continue;
            acc = xadd(acc, xscale(w5[code], val));
        }
    }
}

template <int P>
__global__ void __launch_bounds__(256) k_amr_chi(ALvl c, ALvl fl, LevelConst k, const double* __restrict__ w5,
                                                 int restrictOn) {
    constexpr int NC = 1 << P;
    constexpr int NT = P == 1 ? 3 : P == 2 ? 9 : 27;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < c.nlist; i += gridDim.x * blockDim.x) {
        const unsigned f = c.list[i];
        if (!(c.vflag[f] & amr::kExists)) continue;
        int g[P];
        aunflat<P>(f, c, g);
        const int pid = perm_id<P>(g);
        double2 acc = cz();
        for (int i = 0; i < NC; ++i) {
            const int e = perm_cell(P, pid, i);  // cells around g in Morton order
            int cell[P];
            bool ok = true;
#pragma unroll
            for (int d = 0; d < P; ++d) {
                cell[d] = g[d] - 1 + ((e >> d) & 1);
                ok &= (cell[d] >= 0) & (cell[d] <= c.m - 1);
            }
            if (!ok) continue;
            const int cf = aflat<P>(c, cell);
            if (cf < 0) continue;
            const unsigned char cfl = c.cflag[cf];
            if (!(cfl & amr::kCellExists)) continue;
            const int a = (~e) & (NC - 1);  // corner of g in the cell
            if ((c.vflag[f] & amr::kRegularChi) && restrictOn) {
                // regular neighbourhood: fine vertices 3*cell + j in child order (t = j0 + 3 j1 + 9 j2),
                // loaded a batch of 3^min(P,2) at a time so the loads are in flight together; the
                // sum keeps the child order
                constexpr int NB = P == 1 ? 3 : 9;  // batch: one j_{P-1} slice (P = 3) / everything
                int gc[3] = {0, 0, 0};
#pragma unroll
                for (int d = 0; d < P; ++d) gc[d] = 3 * g[d];
                const int sy = P >= 2 ? fl.n1[0] : 0, sz = P == 3 ? fl.n1[0] * fl.n1[1] : 0;
                const int centre = aflat<P>(fl, gc);
#pragma unroll 1
                for (int t0 = 0; t0 < NT; t0 += NB) {
                    double2 val[NB];
                    double wt[NB];
                    bool act[NB];
#pragma unroll
                    for (int q = 0; q < NB; ++q) {
                        int tt = t0 + q, off[3] = {0, 0, 0}, code = 0, mul = 1;
                        bool in = true;
#pragma unroll
                        for (int d = 0; d < P; ++d) {
                            const int vd = 3 * cell[d] + tt % 3;
                            tt /= 3;
                            off[d] = vd - gc[d];
                            in &= (off[d] >= -2) & (off[d] <= 2) & (vd >= 1) & (vd <= fl.m - 1);
                            code += (off[d] + 2) * mul;
                            mul *= 5;
                        }
                        act[q] = in;
                        val[q] = in ? __ldg(fl.rhat + (centre + off[0] + sy * off[1] + sz * off[2])) : cz();
                        wt[q] = in ? __ldg(w5 + code) : 0.0;
                    }
#pragma unroll
                    for (int q = 0; q < NB; ++q)
                        if (act[q]) acc = xadd(acc, xscale(wt[q], val[q]));
                }
                continue;
            }
            cell_chi<P>(acc, c, fl, k, w5, g, cell, a, cfl, restrictOn);
        }
        c.chi[f] = acc;
    }
}


// ---- chi gather lists (static trees) -----------------------------------------
// The chi walk of k_amr_chi visits the same fine vertices and leaf cells in the
// same order every cycle on a static tree.  k_amr_chi_list replays it once at
// setup and records, per vertex, its terms in order: (fine box index << 7 |
// weight code) for a restriction term, (k << 7 | 127) for its k-th leaf-load term,
// whose value (massScale * sum M nodal) is stored aside -- nodal is constant.
// Storage is warp-interleaved (term k of list position i at base[i >> 5] +
// 32 k + (i & 31)), so the per-cycle k_amr_chi_gather reads it coalesced and
// adds the terms in the recorded order: the same xadd / xscale sequence as
// k_amr_chi, bit for bit.
struct ChiList {
    int* cnt;               // terms per list position (-1: vertex absent, kChiDirect: no stored list)
    int* lcnt;              // leaf terms per list position
    const long long* base;  // per warp group: first term slot
    const long long* lbase; // per warp group: first leaf-value slot
    unsigned* ent;
    double2* leaf;
    const unsigned char* order;  // direct vertices: weight codes in term order, [perm id][5^P]
    int direct;                  // record interior kRegularChi vertices as kChiDirect
};
constexpr unsigned kLeafCode = 127;  // restriction weight codes are 0 .. 5^P - 1
// An interior kRegularChi vertex (amr.hpp) has no loads and no finish-corner
// look-ups: its terms are the 5^P fine vertices 3 g + off, off in [-2, 2]^P, in
// an order that depends only on its permutation id (cells in perm_cell order,
// the 3^P lower-corner vertices of each cell lexicographically).  No list is
// stored for it; k_amr_chi_gather walks the per-id order table instead (the
// weight code gives the offset: code = sum (off_d + 2) 5^d).  Same terms, same
// order, same xscale / xadd sequence as the stored list.
constexpr int kChiDirect = -2;

template <int P, bool WRITE>
__global__ void __launch_bounds__(256) k_amr_chi_list(ALvl c, ALvl fl, LevelConst k, int restrictOn, ChiList L) {
    constexpr int NC = 1 << P;
    constexpr int NT = P == 1 ? 3 : P == 2 ? 9 : 27;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < c.nlist; i += gridDim.x * blockDim.x) {
        const unsigned f = c.list[i];
        if (!(c.vflag[f] & amr::kExists)) {
            if (!WRITE) L.cnt[i] = -1, L.lcnt[i] = 0;
            continue;
        }
        int n = 0, nl = 0;
        const long long eb = WRITE ? L.base[i >> 5] + (i & 31) : 0, lb = WRITE ? L.lbase[i >> 5] + (i & 31) : 0;
        auto term = [&](int vf, int code) {
            if (WRITE) L.ent[eb + 32LL * n] = (static_cast<unsigned>(vf) << 7) | static_cast<unsigned>(code);
            ++n;
        };
        auto leafTerm = [&](double2 v) {
            if (WRITE) {
                L.leaf[lb + 32LL * nl] = v;
                L.ent[eb + 32LL * n] = (static_cast<unsigned>(nl) << 7) | kLeafCode;
            }
            ++n;
            ++nl;
        };
        int g[P];
        aunflat<P>(f, c, g);
        const int pid = perm_id<P>(g);
        if (L.direct && restrictOn && (c.vflag[f] & amr::kRegularChi)) {
            bool interior = true;
#pragma unroll
            for (int d = 0; d < P; ++d) interior &= (g[d] >= 1) & (g[d] <= c.m - 1);
            if (interior) {  // every term is 3 g + off inside the fine box: walked from the order table
                if (!WRITE) L.cnt[i] = kChiDirect, L.lcnt[i] = 0;
                continue;
            }
        }
        for (int ic = 0; ic < NC; ++ic) {
            const int e = perm_cell(P, pid, ic);
            int cell[P];
            bool ok = true;
#pragma unroll
            for (int d = 0; d < P; ++d) {
                cell[d] = g[d] - 1 + ((e >> d) & 1);
                ok &= (cell[d] >= 0) & (cell[d] <= c.m - 1);
            }
            if (!ok) continue;
            const int cf = aflat<P>(c, cell);
            if (cf < 0) continue;
            const unsigned char cfl = c.cflag[cf];
            if (!(cfl & amr::kCellExists)) continue;
            const int a = (~e) & (NC - 1);
            if ((c.vflag[f] & amr::kRegularChi) && restrictOn) {
                for (int t = 0; t < NT; ++t) {
                    int v[P], tt = t, code = 0, mul = 1;
                    bool in = true;
#pragma unroll
                    for (int d = 0; d < P; ++d) {
                        v[d] = 3 * cell[d] + tt % 3;
                        tt /= 3;
                        const int off = v[d] - 3 * g[d];
                        in &= (off >= -2) & (off <= 2) & (v[d] >= 1) & (v[d] <= fl.m - 1);
                        code += (off + 2) * mul;
                        mul *= 5;
                    }
                    if (in) term(aflat<P>(fl, v), code);
                }
                continue;
            }
            if (!(cfl & amr::kCellRefined)) {  // leaf load (cell_chi)
                double2 acc2 = cz();
#pragma unroll
                for (int bb = 0; bb < NC; ++bb) {
                    int vb[P];
#pragma unroll
                    for (int d = 0; d < P; ++d) vb[d] = cell[d] + ((bb >> d) & 1);
                    acc2 = xadd(acc2, xscale(k.M[a ^ bb], c.nodal[aflat<P>(c, vb)]));
                }
                leafTerm(xmul(k.massScale, acc2));
                continue;
            }
            if (!restrictOn) continue;
            for (int t = 0; t < NT; ++t) {  // cell_chi's refined cell: (child, corner) ascending
                int j[P], tt = t;
#pragma unroll
                for (int d = 0; d < P; ++d) {
                    j[d] = tt % 3;
                    tt /= 3;
                }
                for (int ec = 0; ec < NC; ++ec) {
                    int v[P], code = 0, mul = 1;
                    bool in = true;
#pragma unroll
                    for (int d = 0; d < P; ++d) {
                        v[d] = 3 * cell[d] + j[d] + ((ec >> d) & 1);
                        const int off = v[d] - 3 * g[d];
                        in &= (off >= -2) & (off <= 2) & (v[d] >= 1) & (v[d] <= fl.m - 1);
                        code += (off + 2) * mul;
                        mul *= 5;
                    }
                    if (!in) continue;
                    const int vf = aflat<P>(fl, v);
                    if (vf < 0 || fl.estar[vf] != ec) continue;
                    term(vf, code);
                }
            }
        }
        if (!WRITE) {
            L.cnt[i] = n;
            L.lcnt[i] = nl;
        }
    }
}

template <int P>
__global__ void __launch_bounds__(256) k_amr_chi_gather(ALvl c, ALvl fl, const double* __restrict__ w5, ChiList L) {
    const double2* __restrict__ frhat = fl.rhat;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < c.nlist; i += gridDim.x * blockDim.x) {
        const int n = L.cnt[i];
        if (n == kChiDirect) {  // interior kRegularChi vertex: the order table instead of a stored list
            constexpr int K = P == 1 ? 5 : P == 2 ? 25 : 125;
            const unsigned f = c.list[i];
            int g[P], v0[P];
            aunflat<P>(f, c, g);
            const unsigned char* __restrict__ ord = L.order + perm_id<P>(g) * K;
#pragma unroll
            for (int d = 0; d < P; ++d) v0[d] = 3 * g[d];
            const int fb = aflat<P>(fl, v0);
            const int sy = P >= 2 ? fl.n1[0] : 0, sz = P >= 3 ? fl.n1[0] * fl.n1[1] : 0;
            double2 acc = cz();
            constexpr int B = 5;  // terms in flight (K is a multiple of 5)
            for (int k0 = 0; k0 < K; k0 += B) {
                double2 val[B];
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    const int code = ord[k0 + b];
                    const int off = (code % 5 - 2) + (P >= 2 ? (code / 5 % 5 - 2) * sy : 0) + (P >= 3 ? (code / 25 - 2) * sz : 0);
                    val[b] = xscale(__ldg(w5 + code), __ldg(frhat + (fb + off)));
                }
#pragma unroll
                for (int b = 0; b < B; ++b) acc = xadd(acc, val[b]);
            }
            c.chi[f] = acc;
            continue;
        }
        if (n < 0) continue;
        const unsigned* __restrict__ e = L.ent + L.base[i >> 5] + (i & 31);
        const double2* __restrict__ lv = L.leaf + L.lbase[i >> 5] + (i & 31);
        double2 acc = cz();
        constexpr int B = 8;  // terms in flight
        for (int k0 = 0; k0 < n; k0 += B) {
            double2 val[B];
            unsigned code[B];
#pragma unroll
            for (int b = 0; b < B; ++b) code[b] = k0 + b < n ? __ldg(e + 32LL * (k0 + b)) : kLeafCode;
#pragma unroll
            for (int b = 0; b < B; ++b) {
                const unsigned x = code[b];
                const bool leaf = (x & 127u) == kLeafCode;
                val[b] = k0 + b >= n ? cz() : leaf ? __ldg(lv + 32LL * (x >> 7)) : xscale(__ldg(w5 + (x & 127u)), __ldg(frhat + (x >> 7)));
            }
#pragma unroll
            for (int b = 0; b < B; ++b) {
                if (k0 + b >= n) break;
                acc = xadd(acc, val[b]);
            }
        }
        c.chi[c.list[i]] = acc;
    }
}

// small levels: one warp per vertex -- the lanes fetch and scale 32 terms at a
// time, lane 0 adds them in order
__global__ void __launch_bounds__(256) k_amr_chi_gather_warp(ALvl c, const double2* __restrict__ frhat,
                                                             const double* __restrict__ w5, ChiList L) {
    const unsigned lane = threadIdx.x & 31u;
    const unsigned warps = (gridDim.x * blockDim.x) >> 5;
    for (unsigned i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < c.nlist; i += warps) {
        const int n = L.cnt[i];
        if (n < 0) continue;
        const unsigned* __restrict__ e = L.ent + L.base[i >> 5] + (i & 31);
        const double2* __restrict__ lv = L.leaf + L.lbase[i >> 5] + (i & 31);
        double2 acc = cz();
        for (int k0 = 0; k0 < n; k0 += 32) {
            double2 v = cz();
            if (k0 + static_cast<int>(lane) < n) {
                const unsigned x = __ldg(e + 32LL * (k0 + lane));
                v = (x & 127u) == kLeafCode ? __ldg(lv + 32LL * (x >> 7)) : xscale(__ldg(w5 + (x & 127u)), __ldg(frhat + (x >> 7)));
            }
            const int cntk = min(32, n - k0);
            for (int b = 0; b < cntk; ++b) {
                const double vx = __shfl_sync(0xffffffffu, v.x, b), vy = __shfl_sync(0xffffffffu, v.y, b);
                acc = xadd(acc, make_double2(vx, vy));
            }
        }
        if (lane == 0) c.chi[c.list[i]] = acc;
    }
}

// sum_b A(a, b) x_b over the corners of one cell, b ascending (kernels.cpp:39-47)
template <int P>
__device__ __forceinline__ double2 cell_apply(const double2* __restrict__ x, const ALvl& c, const int* cell, int a,
                                              const double2 (&A)[8]) {
    double2 s = cz();
#pragma unroll
    for (int bb = 0; bb < (1 << P); ++bb) {
        int vb[P];
#pragma unroll
        for (int d = 0; d < P; ++d) vb[d] = cell[d] + ((bb >> d) & 1);
        const double2 prod = xmul(A[a ^ bb], x[aflat<P>(c, vb)]);
        s = bb == 0 ? prod : xadd(s, prod);
    }
    return s;
}

// All 2^P cells around an interior non-hanging vertex exist: the regular
// exact path's shared-product evaluation (hierarchy.cu element_residual) on the
// box strides -- the same per-cell corner order and cell order, bit for bit.
template <int P, int ID>
__device__ __forceinline__ double2 amr_ordered_sum(const double2 (&S)[1 << P]) {
    double2 r = xneg(S[perm_cell(P, ID, 0)]);
#pragma unroll
    for (int i = 1; i < (1 << P); ++i) r = xsub(r, S[perm_cell(P, ID, i)]);
    return r;
}

template <int P>
__device__ __forceinline__ double2 regular_residual(const double2* __restrict__ x, int f, int sy, int sz,
                                                    const double2 (&A)[8], int pid) {
    constexpr int NC = 1 << P;
    double2 S[NC];
#pragma unroll
    for (int j = 0; j < (P == 1 ? 3 : P == 2 ? 9 : 27); ++j) {
        int del[P];
        int off = 0, s = 0;
#pragma unroll
        for (int d = 0; d < P; ++d) {
            del[d] = (j / (d == 0 ? 1 : d == 1 ? 3 : 9)) % 3 - 1;
            off += del[d] * (d == 0 ? 1 : d == 1 ? sy : sz);
            s |= (del[d] != 0 ? 1 : 0) << d;
        }
        const double2 prod = xmul(A[s], __ldg(x + (f + off)));
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
    if (P == 1) return amr_ordered_sum<P, 0>(S);
    if (P == 2) return pid == 0 ? amr_ordered_sum<P, 0>(S) : amr_ordered_sum<P, (P >= 2 ? 1 : 0)>(S);
    switch (pid) {
        case 0: return amr_ordered_sum<P, 0>(S);
        case 1: return amr_ordered_sum<P, (P >= 3 ? 1 : 0)>(S);
        case 2: return amr_ordered_sum<P, (P >= 3 ? 2 : 0)>(S);
        case 3: return amr_ordered_sum<P, (P >= 3 ? 3 : 0)>(S);
        case 4: return amr_ordered_sum<P, (P >= 3 ? 4 : 0)>(S);
        default: return amr_ordered_sum<P, (P >= 3 ? 5 : 0)>(S);
    }
}

// precision = fast: the same residual as the assembled 3^P-point stencil (the
// 2^(P - |s|) cells that share the vertex and its neighbour at offset class s
// each contribute A[s]), complex FMAs in neighbour order -- within rounding of
// the traversal-order element sums, not bit-identical
template <int P>
__device__ __forceinline__ double2 regular_residual_fast(const double2* __restrict__ x, int f, int sy, int sz,
                                                         const double2 (&K)[8]) {
    double2 acc = cz();
#pragma unroll
    for (int j = 0; j < (P == 1 ? 3 : P == 2 ? 9 : 27); ++j) {
        int off = 0, s = 0;
#pragma unroll
        for (int d = 0; d < P; ++d) {
            const int del = (j / (d == 0 ? 1 : d == 1 ? 3 : 9)) % 3 - 1;
            off += del * (d == 0 ? 1 : d == 1 ? sy : sz);
            s |= (del != 0 ? 1 : 0) << d;
        }
        const double2 v = __ldg(x + (f + off));
        acc = make_double2(fma(K[s].x, v.x, fma(-K[s].y, v.y, acc.x)), fma(K[s].x, v.y, fma(K[s].y, v.x, acc.y)));
    }
    return xneg(acc);
}

// Special vertices of a dynamic sweep (dyn.hpp kSSpecial): created after some
// adjacent cells were already entered (those never reach it), or finishing
// more than once (hanging vertices on the rim of blocks refined later in the
// same traversal: each destroy_hanging, cycles.cpp:305-321, folds chi + r-hat
// again), or never.  The accumulators run over the cells in traversal order;
// every finish records its r-hat for the parents' restriction.
template <int P>
__global__ void __launch_bounds__(256) k_dyn_special(ALvl c, ALvl fl, LevelConst k, const double* __restrict__ w5,
                                                     int restrictOn, int ellMin, const double2* __restrict__ dgTab) {
    constexpr int NC = 1 << P;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < c.nslist; i += gridDim.x * blockDim.x) {
        const unsigned f = c.slist[i];
        const unsigned char vf = c.vflag[f];
        const bool bnd = vf & amr::kBoundary, hang = vf & amr::kHanging;
        int g[P];
        aunflat<P>(f, c, g);
        const int pid = perm_id<P>(g);
        const unsigned char skip = c.skip[f], fm = c.fmask[f];
        double2 r = cz(), rh = cz(), chi = cz();
        bool first = true;
        int ncell = 0, kfin = 0;
        for (int ii = 0; ii < NC; ++ii) {
            const int e = perm_cell(P, pid, ii);
            int cell[P];
            bool ok = true;
#pragma unroll
            for (int d = 0; d < P; ++d) {
                cell[d] = g[d] - 1 + ((e >> d) & 1);
                ok &= (cell[d] >= 0) & (cell[d] <= c.m - 1);
            }
            if (!ok || ((skip >> e) & 1)) continue;
            const int cf = aflat<P>(c, cell);
            if (cf < 0) continue;
            const unsigned char cfl = c.cflag[cf];
            if (!(cfl & amr::kCellExists)) continue;
            const int ca = (~e) & (NC - 1);
            const double2 sr = cell_apply<P>(c.u, c, cell, ca, k.A);
            const double2 sh = cell_apply<P>(c.uhat, c, cell, ca, k.A);
            if (first) {
                r = xneg(sr);
                rh = xneg(sh);
                first = false;
            } else {
                r = xsub(r, sr);
                rh = xsub(rh, sh);
            }
            ++ncell;
            cell_chi<P>(chi, c, fl, k, w5, g, cell, ca, cfl, restrictOn);
            if ((fm >> e) & 1) {  // finishes at the end of this cell's visit
                if (hang && c.level > ellMin) rh = bnd ? cz() : xadd(chi, rh);
                c.extras[c.xoff[f] + kfin] = rh;
                ++kfin;
            }
        }
        c.chi[f] = chi;
        c.rhat[f] = rh;
        c.r[f] = r;
        c.dg[f] = ncell > 0 ? dgTab[ncell] : cz();
    }
}

// ---- residual + touch_last / destroy_hanging --------------------------------
#ifndef TMG_AMR_RES_MINB
#define TMG_AMR_RES_MINB 3
#endif
template <int P, bool FAST = false>
__global__ void __launch_bounds__(256, TMG_AMR_RES_MINB) k_amr_residual(AResArgs a) {
    constexpr int NC = 1 << P;
    const ALvl& c = a.lv;
    double nmax = 0.0, nsum = 0.0;
    ListWalk w(c);
    const FastUnflat<P> unflat(c);
    for (unsigned i = w.first(); i < c.nlist; i = w.next(i)) {
        const unsigned f = w.f;
        const unsigned char vf = w.vf;
        w.prefetch(i);
        if (!(vf & amr::kExists)) continue;
        if (c.slist && (vf & dyn::kSSpecial)) continue;  // k_dyn_special
        const bool bnd = vf & amr::kBoundary, cp = vf & amr::kCPoint, hang = vf & amr::kHanging,
                   refined = vf & amr::kRefined;
        int g[P];
        unflat(f, g);
        double2 r = cz(), rh = cz();
        bool first = true;
        int ncell = NC;
        const bool general = hang || bnd;
        // the traversal order of the cells around g: not needed by the assembled stencil
        const int pid = (FAST && !general) ? 0 : perm_id<P>(g);
        if (!general) {  // every cell around g exists
            const int sy = c.n1[0], sz = c.n1[0] * c.n1[1];
            if (FAST) {
                r = regular_residual_fast<P>(c.u, static_cast<int>(f), sy, sz, a.kAsm);
                rh = regular_residual_fast<P>(c.uhat, static_cast<int>(f), sy, sz, a.kAsm);
            } else {
                r = regular_residual<P>(c.u, static_cast<int>(f), sy, sz, a.k.A, pid);
                rh = regular_residual<P>(c.uhat, static_cast<int>(f), sy, sz, a.k.A, pid);
            }
        } else {
            ncell = 0;
        }
        for (int i = 0; i < NC && general; ++i) {
            const int e = perm_cell(P, pid, i);
            int cell[P];
            bool ok = true;
#pragma unroll
            for (int d = 0; d < P; ++d) {
                cell[d] = g[d] - 1 + ((e >> d) & 1);
                ok &= (cell[d] >= 0) & (cell[d] <= c.m - 1);
            }
            if (!ok) continue;
            const int cf = aflat<P>(c, cell);
            if (cf < 0 || !(c.cflag[cf] & amr::kCellExists)) continue;
            const int ca = (~e) & (NC - 1);
            const double2 sr = cell_apply<P>(c.u, c, cell, ca, a.k.A);
            const double2 sh = cell_apply<P>(c.uhat, c, cell, ca, a.k.A);
            if (first) {
                r = xneg(sr);
                rh = xneg(sh);
                first = false;
            } else {
                r = xsub(r, sr);
                rh = xsub(rh, sh);
            }
            ++ncell;
        }
        if (c.dg) c.dg[f] = ncell > 0 ? a.dgTab[ncell] : cz();
        const double2 chi = c.chi[f];
        if (hang) {  // destroy_hanging: only r-hat (plus load) goes down
            double2 rhat = rh;
            if (c.level > a.ellMin) rhat = bnd ? cz() : xadd(chi, rh);
            c.rhat[f] = rhat;
            if (c.r) c.r[f] = r;
            continue;
        }
        if (bnd) {  // finish_vertex, kernels.cpp:89-100
            r = cz();
            rh = cz();
        } else {
            r = xadd(chi, r);
            rh = xadd(chi, rh);
        }
        if (c.si) {
            c.si[f] = c.sinext[f];
            c.sinext[f] = cz();
        }
        if (!refined && !bnd) {
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
        const double2 smooth =
            bnd ? cz()
                : FAST ? make_double2(fma(r.x, a.invDiag.x, -r.y * a.invDiag.y), fma(r.x, a.invDiag.y, r.y * a.invDiag.x))
                       : divdc3(r.x, r.y, a.k.div);
        const double2 wRaw = a.wTab[c.succ[f]];
        double2 sc;
        if (a.bpx) {
            sc = cp ? cz() : xmul(wRaw, smooth);
        } else {
            const bool wz = (a.hb && cp) || xzero(wRaw);
            sc = wz ? cz() : xmul(wRaw, smooth);
        }
        c.sc[f] = sc;
        if (c.level > a.ellMin && cp) {
            int wi[P];
#pragma unroll
            for (int d = 0; d < P; ++d) wi[d] = g[d] / 3;
            const int wf = aflat<P>(a.par, wi);
            if (wf >= 0 && (a.par.vflag[wf] & amr::kExists)) {
                const double2 sf = c.sf ? c.sf[f] : cz();
                a.par.sf[wf] = xadd(sf, sc);
                if (a.bpx) a.par.sinext[wf] = xmul(wRaw, smooth);
            }
        }
    }
    block_norms(nmax, nsum, a.partials);
}

// per-level (max, sum) from the block partials of every level
__global__ void k_amr_norm_final(const double* __restrict__ partials, const int* __restrict__ offs, int nlev,
                                 double* out) {
    __shared__ double smax[1024], ssum[1024];
    for (int l = blockIdx.x; l < nlev; l += gridDim.x) {  // one block per level (same tree per level)
        double mx = 0.0, sm = 0.0;
        for (int i = offs[l] + threadIdx.x; i < offs[l + 1]; i += blockDim.x) {
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
            out[2 * l] = smax[0];
            out[2 * l + 1] = ssum[0];
        }
        __syncthreads();
    }
}

// ---- setup -------------------------------------------------------------------
template <int P>
__global__ void k_amr_seeded(ALvl c, unsigned long long seed, long long scale, long long mkey, int sphere, int all) {
    for (unsigned f = blockIdx.x * blockDim.x + threadIdx.x; f < c.n; f += gridDim.x * blockDim.x) {
        if (!all && !(c.vflag[f] & amr::kExists)) continue;
        int g[P];
        aunflat<P>(f, c, g);
        unsigned long long key = 0;
        long long s2 = 0;
#pragma unroll
        for (int d = 0; d < P; ++d) {
            const long long fi = static_cast<long long>(g[d]) * scale;
            key |= static_cast<unsigned long long>(static_cast<unsigned short>(fi)) << (16 * d);
            const long long t = 2 * fi - mkey;
            s2 += t * t;
        }
        if (sphere && !(25 * s2 < 4 * mkey * mkey)) {
            c.nodal[f] = cz();
            continue;
        }
        const unsigned long long s = seed ^ key;
        c.nodal[f] = make_double2(unit_rand(s), unit_rand(s ^ 0x5bf03635ull));
    }
}

// set_random_initial_guess, cycles.cpp:812-840: leaves random, boundary 0
template <int P>
__global__ void k_amr_random(ALvl c, unsigned long long seed) {
    for (unsigned f = blockIdx.x * blockDim.x + threadIdx.x; f < c.n; f += gridDim.x * blockDim.x) {
        const unsigned char vf = c.vflag[f];
        if (!(vf & amr::kExists) || (vf & amr::kHanging)) continue;
        if (vf & amr::kBoundary) {
            c.u[f] = cz();
            continue;
        }
        if (vf & amr::kRefined) continue;  // injected from the finer level afterwards
        int g[P];
        aunflat<P>(f, c, g);
        unsigned long long key = 0;
#pragma unroll
        for (int d = 0; d < P; ++d) key |= static_cast<unsigned long long>(static_cast<unsigned short>(g[d])) << (16 * d);
        const unsigned long long base = seed ^ (static_cast<unsigned long long>(c.level) << 56) ^ key;
        c.u[f] = make_double2(unit_rand(base), unit_rand(base ^ 0x5bf03635ull));
    }
}

template <int P>
__global__ void k_amr_inject(ALvl c, ALvl fine) {
    for (unsigned f = blockIdx.x * blockDim.x + threadIdx.x; f < c.n; f += gridDim.x * blockDim.x) {
        const unsigned char vf = c.vflag[f];
        if (!(vf & amr::kExists) || (vf & (amr::kHanging | amr::kBoundary)) || !(vf & amr::kRefined)) continue;
        int g[P];
        aunflat<P>(f, c, g);
        int fi[P];
#pragma unroll
        for (int d = 0; d < P; ++d) fi[d] = 3 * g[d];
        const int ff = aflat<P>(fine, fi);
        c.u[f] = (ff >= 0 && (fine.vflag[ff] & amr::kExists)) ? fine.u[ff] : cz();
    }
}

// ---- dynamic adaptivity: mark (amr.cpp:18-222) ------------------------------
// |z| as the host's libm computes it (std::abs(complex) -> hypot): glibc's
// hypot, Borges' algorithm with the non-FMA correction kernel; pinned
// bit-for-bit against the host libm (tests/test_dyn_structure.py).  Every
// operation is an explicit round-to-nearest intrinsic (no contraction).
__device__ __forceinline__ double hypot_kernel(double ax, double ay) {
    double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
    double t1, t2;
    if (h <= 2.0 * ay) {
        const double delta = __dsub_rn(h, ay);
        t1 = __dmul_rn(ax, __dsub_rn(2.0 * delta, ax));
        t2 = __dmul_rn(__dsub_rn(delta, 2.0 * __dsub_rn(ax, ay)), delta);
    } else {
        const double delta = __dsub_rn(h, ax);
        t1 = __dmul_rn(2.0 * delta, __dsub_rn(ax, 2.0 * ay));
        t2 = __dadd_rn(__dmul_rn(__dsub_rn(4.0 * delta, ay), ay), __dmul_rn(delta, delta));
    }
    return __dsub_rn(h, __ddiv_rn(__dadd_rn(t1, t2), 2.0 * h));
}

__device__ double host_hypot(double x, double y) {
    x = fabs(x);
    y = fabs(y);
    if (isinf(x) || isinf(y)) return INFINITY;
    if (isnan(x) || isnan(y)) return x + y;
    const double ax = x < y ? y : x, ay = x < y ? x : y;
    const double kScale = 0x1p-600, kLarge = 0x1p+511, kTiny = 0x1p-511, kEps = 0x1p-54;
    if (ax > kLarge) {
        if (ay <= __dmul_rn(ax, kEps)) return __dadd_rn(ax, ay);
        return __ddiv_rn(hypot_kernel(__dmul_rn(ax, kScale), __dmul_rn(ay, kScale)), kScale);
    }
    if (ay < kTiny) {
        if (ax >= __ddiv_rn(ay, kEps)) return __dadd_rn(ax, ay);
        return __dmul_rn(hypot_kernel(__ddiv_rn(ax, kScale), __ddiv_rn(ay, kScale)), kScale);
    }
    if (ay <= __dmul_rn(ax, kEps)) return __dadd_rn(ax, ay);
    return hypot_kernel(ax, ay);
}

// Spacetree::u_at (spacetree.cpp:191-205): the vertex's u if it exists and is
// not hanging after the sweep, else the prolongation of u_at on the parent
// stencil -- the same recursion, evaluated with an explicit frame stack (one
// frame per level) so the depth never depends on the device call stack
template <int P>
__device__ double2 u_at(const ALvl* __restrict__ lvs, int level, const int* idx) {
    constexpr int NC = 1 << P;
    struct Frame {
        int level, e;
        int q[P], rel[P];
        double2 v[NC];
    };
    auto direct = [&](int l, const int* id, double2& out) -> bool {
        const ALvl& c = lvs[l];
        const int f = aflat<P>(c, id);
        if (f >= 0 && (c.fflag[f] & amr::kExists) && !(c.fflag[f] & amr::kHanging)) {
            out = c.u[f];
            return true;
        }
        if (l == 0) {
            out = cz();
            return true;
        }
        return false;
    };
    double2 res;
    if (direct(level, idx, res)) return res;
    Frame st[10];
    int sp = 0;
    auto push = [&](int l, const int* id) {
        Frame& F = st[sp++];
        F.level = l;
        F.e = 0;
        const int mc = lvs[l - 1].m;
#pragma unroll
        for (int d = 0; d < P; ++d) {
            F.q[d] = min(id[d] / 3, mc - 1);
            F.rel[d] = id[d] - 3 * F.q[d];
        }
    };
    push(level, idx);
    while (true) {
        Frame& F = st[sp - 1];
        if (F.e == NC) {
            const double2 val = prolong<P>(F.v, F.rel);
            if (--sp == 0) return val;
            Frame& U = st[sp - 1];
            U.v[U.e++] = val;
            continue;
        }
        int vi[P];
#pragma unroll
        for (int d = 0; d < P; ++d) vi[d] = F.q[d] + ((F.e >> d) & 1);
        double2 out;
        if (direct(F.level - 1, vi, out)) {
            F.v[F.e++] = out;
            continue;
        }
        push(F.level - 1, vi);
    }
}

struct MarkCounters {  // device counters of one mark pass
    unsigned long long cand, refineV, eraseV, refineC, eraseC, vetoConv, vetoHMin, vetoHMax;
    unsigned long long sMinBits, sMaxBits;
};

// candidates: non-hanging, unrefined, interior vertices of levels >= ellMin
// (amr.cpp:85-90); feature (amr.cpp:18-31) and convergence indicator
template <int P>
__global__ void k_dyn_features(const ALvl* __restrict__ lvs, int level, int candOn, MarkCounters* cnt) {
    const ALvl& c = lvs[level];
    for (unsigned f = blockIdx.x * blockDim.x + threadIdx.x; f < c.n; f += gridDim.x * blockDim.x) {
        const unsigned char vf = c.fflag[f];
        const bool cand =
            candOn && (vf & amr::kExists) && !(vf & (amr::kHanging | amr::kRefined | amr::kBoundary));
        c.vmark[f] = cand ? 4 : 0;
        if (!cand) continue;
        int g[P];
        aunflat<P>(f, c, g);
        const double2 centre = c.u[f];
        double s = 0.0;
        for (int d = 0; d < P; ++d) {
            if (g[d] - 1 < 0 || g[d] + 1 > c.m) continue;
            int lo[P], hi[P];
#pragma unroll
            for (int dd = 0; dd < P; ++dd) {
                lo[dd] = g[dd];
                hi[dd] = g[dd];
            }
            --lo[d];
            ++hi[d];
            const double2 a = u_at<P>(lvs, level, lo), b = u_at<P>(lvs, level, hi);
            const double2 second = xadd(xsub(a, xscale(2.0, centre)), b);
            s = fmax(s, host_hypot(second.x, second.y));
        }
        const double2 r = c.r[f], dg = c.dg[f];
        const double ad = host_hypot(dg.x, dg.y);
        c.feat[f] = s;
        c.ind[f] = ad > 0.0 ? __ddiv_rn(host_hypot(r.x, r.y), ad) : 0.0;
        const unsigned long long sb = __double_as_longlong(s);  // s >= 0: bit order is value order
        atomicMin(&cnt->sMinBits, sb);
        atomicMax(&cnt->sMaxBits, sb);
        atomicAdd(&cnt->cand, 1ull);
    }
}

__device__ __forceinline__ int mark_bin(double s, double smin, double span, int bins) {
    const int b = static_cast<int>(__dmul_rn(__ddiv_rn(__dsub_rn(s, smin), span), static_cast<double>(bins)));
    return min(max(b, 0), bins - 1);
}

template <int P>
__global__ void k_dyn_hist(const ALvl* __restrict__ lvs, int level, double smin, double span, int bins,
                           unsigned long long* hist) {
    const ALvl& c = lvs[level];
    for (unsigned f = blockIdx.x * blockDim.x + threadIdx.x; f < c.n; f += gridDim.x * blockDim.x)
        if (c.vmark[f] & 4) atomicAdd(&hist[mark_bin(c.feat[f], smin, span, bins)], 1ull);
}

// amr.cpp:104-119: top bins refine, bottom bins erase, both vetoed by |r|/|diag|
template <int P>
__global__ void k_dyn_classify(const ALvl* __restrict__ lvs, int level, double smin, double span, int bins, int kRef,
                               int kErase, double veto, MarkCounters* cnt) {
    const ALvl& c = lvs[level];
    for (unsigned f = blockIdx.x * blockDim.x + threadIdx.x; f < c.n; f += gridDim.x * blockDim.x) {
        if (!(c.vmark[f] & 4)) continue;
        const int b = mark_bin(c.feat[f], smin, span, bins);
        const bool vetoed = c.ind[f] > veto;
        if (b >= bins - kRef) {
            if (vetoed) atomicAdd(&cnt->vetoConv, 1ull);
            else {
                c.vmark[f] |= 1;
                atomicAdd(&cnt->refineV, 1ull);
            }
        } else if (b < kErase) {
            if (vetoed) atomicAdd(&cnt->vetoConv, 1ull);
            else {
                c.vmark[f] |= 2;
                atomicAdd(&cnt->eraseV, 1ull);
            }
        }
    }
}

// amr.cpp:134-161: every unrefined cell around a refine-marked vertex, above the h floor
template <int P>
__global__ void k_dyn_refine_cells(const ALvl* __restrict__ lvs, int level, double h, double hMin,
                                   MarkCounters* cnt) {
    const ALvl& c = lvs[level];
    for (unsigned f = blockIdx.x * blockDim.x + threadIdx.x; f < c.n; f += gridDim.x * blockDim.x) {
        if (!(c.vmark[f] & 1)) continue;
        int g[P];
        aunflat<P>(f, c, g);
        for (int e = 0; e < (1 << P); ++e) {
            int ci[P];
            bool ok = true;
#pragma unroll
            for (int d = 0; d < P; ++d) {
                ci[d] = g[d] - ((e >> d) & 1);
                ok &= (ci[d] >= 0) & (ci[d] <= c.m - 1);
            }
            if (!ok) continue;
            const int cf = aflat<P>(c, ci);
            const unsigned char cfl = c.fcell[cf];
            if (!(cfl & amr::kCellExists) || (cfl & amr::kCellRefined)) continue;
            if (!(h > hMin)) {
                atomicAdd(&cnt->vetoHMin, 1ull);
                continue;
            }
            const unsigned old = atomicOr(&c.cmark[cf], static_cast<unsigned>(dyn::kRM));
            if (!(old & dyn::kRM)) {
                atomicAdd(&cnt->refineC, 1ull);
                c.mlist[atomicAdd(c.mcount, 1u)] = static_cast<unsigned>(cf);
            }
        }
    }
}

// amr.cpp:163-221: a refined cell with unrefined children erases when every
// strictly interior child-block vertex is erase-marked and none of the block is
// refine-marked, unless its h exceeds h_max
template <int P>
__global__ void k_dyn_erase_cells(const ALvl* __restrict__ lvs, int level, double h, double hMax, MarkCounters* cnt) {
    const ALvl& c = lvs[level];
    const ALvl& fl = lvs[level + 1];
    constexpr int NB = P == 1 ? 4 : P == 2 ? 16 : 64;
    constexpr int NT = P == 1 ? 3 : P == 2 ? 9 : 27;
    for (unsigned f = blockIdx.x * blockDim.x + threadIdx.x; f < c.n; f += gridDim.x * blockDim.x) {
        const unsigned char cfl = c.fcell[f];
        if (!(cfl & amr::kCellExists) || !(cfl & amr::kCellRefined)) continue;
        int g[P];
        aunflat<P>(f, c, g);
        int innerTotal = 0, innerMarked = 0;
        bool anyRefine = false, childRefined = false;
        for (int t = 0; t < NB; ++t) {
            int vi[P];
            bool inner = true;
            int tt = t;
#pragma unroll
            for (int d = 0; d < P; ++d) {
                const int rel = tt % 4;
                tt /= 4;
                vi[d] = 3 * g[d] + rel;
                inner &= rel == 1 || rel == 2;
            }
            const int vf = aflat<P>(fl, vi);
            if (vf < 0) continue;
            const unsigned char vm = fl.vmark[vf];
            if (vm & 1) anyRefine = true;
            if (!inner) continue;
            const unsigned char ff = fl.fflag[vf];
            if (!(ff & amr::kExists) || (ff & (amr::kHanging | amr::kBoundary))) continue;
            ++innerTotal;
            if (vm & 2) ++innerMarked;
        }
        for (int t = 0; t < NT; ++t) {
            int ci[P];
            int tt = t;
#pragma unroll
            for (int d = 0; d < P; ++d) {
                ci[d] = 3 * g[d] + tt % 3;
                tt /= 3;
            }
            const int cf = aflat<P>(fl, ci);
            if (cf >= 0 && (fl.fcell[cf] & amr::kCellRefined)) childRefined = true;
        }
        if (childRefined || anyRefine || innerTotal == 0 || innerMarked != innerTotal) continue;
        if (h > hMax) {
            atomicAdd(&cnt->vetoHMax, 1ull);
            continue;
        }
        const unsigned old = atomicOr(&c.cmark[f], static_cast<unsigned>(dyn::kEM));
        if (!(old & dyn::kEM)) {
            atomicAdd(&cnt->eraseC, 1ull);
            c.mlist[atomicAdd(c.mcount, 1u)] = f | 0x80000000u;
        }
    }
}

// sweep-table maintenance: clear the previous sweep's entries, scatter the new ones
struct SweepRec {
    unsigned f;
    unsigned char flag, estar, fmask, skip;
    signed char succ;
    unsigned char pad[3];
    int xoff;
};

__global__ void k_dyn_clear(unsigned char* vflag, unsigned char* estar, const unsigned* prev, unsigned n) {
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        vflag[prev[i]] = 0;
        estar[prev[i]] = 0xFF;
    }
}

__global__ void k_dyn_scatter(const SweepRec* __restrict__ rec, unsigned n, unsigned char* vflag, unsigned char* estar,
                              unsigned char* fmask, unsigned char* skip, signed char* succ, int* xoff) {
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const SweepRec r = rec[i];
        vflag[r.f] = r.flag;
        estar[r.f] = r.estar;
        fmask[r.f] = r.fmask;
        skip[r.f] = r.skip;
        succ[r.f] = r.succ;
        xoff[r.f] = r.xoff;
    }
}

// dst[idx[i]] = val[i] (val null: 0)
__global__ void k_scatter_bytes(const unsigned* __restrict__ idx, const unsigned char* __restrict__ val, unsigned n,
                                unsigned char* dst) {
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        dst[idx[i]] = val ? val[i] : 0;
}

__global__ void k_clear_marks(const unsigned* __restrict__ mlist, unsigned n, unsigned* cmark) {
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        cmark[mlist[i] & 0x7FFFFFFFu] = 0;
}

__global__ void k_test_hypot(const double* x, const double* y, double* out, long long n) {
    for (long long i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = host_hypot(x[i], y[i]);
}

}  // namespace adev

void test_hypot(const double* x, const double* y, double* out, long long n) {
    double *dx = nullptr, *dy = nullptr, *dout = nullptr;
    const size_t bytes = static_cast<size_t>(std::max<long long>(n, 1)) * sizeof(double);
    AMR_CUDA(cudaMalloc(&dx, bytes));
    AMR_CUDA(cudaMalloc(&dy, bytes));
    AMR_CUDA(cudaMalloc(&dout, bytes));
    AMR_CUDA(cudaMemcpy(dx, x, static_cast<size_t>(n) * sizeof(double), cudaMemcpyHostToDevice));
    AMR_CUDA(cudaMemcpy(dy, y, static_cast<size_t>(n) * sizeof(double), cudaMemcpyHostToDevice));
    adev::k_test_hypot<<<256, 256>>>(dx, dy, dout, n);
    AMR_CUDA(cudaGetLastError());
    AMR_CUDA(cudaMemcpy(out, dout, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToHost));
    cudaFree(dx);
    cudaFree(dy);
    cudaFree(dout);
}

// ============================================================================
// Host: tree structure
// ============================================================================

namespace amr {
namespace {

int pow3(int l) {
    int r = 1;
    for (int i = 0; i < l; ++i) r *= 3;
    return r;
}

// fn(begin, end) over [0, n) on the host's cores (the setup loops write only
// their own element)
template <class F>
void parallel_for(long long n, F&& fn) {
    const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    if (n < 65536 || hw == 1) {
        fn(0LL, n);
        return;
    }
    std::vector<std::thread> ts;
    const long long chunk = (n + hw - 1) / hw;
    for (unsigned t = 0; t < hw; ++t) {
        const long long a = static_cast<long long>(t) * chunk, b = std::min(n, a + chunk);
        if (a < b) ts.emplace_back([&fn, a, b] { fn(a, b); });
    }
    for (auto& t : ts) t.join();
}

int tz3h(int x) {
    if (x == 0) return 31;
    int t = 0;
    while (x % 3 == 0) {
        x /= 3;
        ++t;
    }
    return t;
}

// host twin of dev::perm_id (exact_ops.cuh)
int perm_id_host(int p, const int* idx) {
    if (p == 1) return 0;
    if (p == 2) return tz3h(idx[1]) >= tz3h(idx[0]) ? 0 : 1;
    const int k0 = tz3h(idx[0]) * 4 + 0, k1 = tz3h(idx[1]) * 4 + 1, k2 = tz3h(idx[2]) * 4 + 2;
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

// cell centre in |x - 1/2|^2 < 0.04 (oracle/refdriver.cpp cell_centre_in_sphere)
bool centre_in_sphere(int p, int level, const int* c) {
    const long long m = pow3(level);
    long long s = 0;
    for (int d = 0; d < p; ++d) {
        const long long t = 2LL * c[d] + 1 - m;
        s += t * t;
    }
    return 25 * s < 4 * m * m;
}

long long box_flat(const HostLevel& h, int p, const int* g) {
    long long f = 0, s = 1;
    for (int d = 0; d < p; ++d) {
        const int x = g[d] - h.lo[d];
        if (x < 0 || x >= h.n1[d]) return -1;
        f += static_cast<long long>(x) * s;
        s *= h.n1[d];
    }
    return f;
}

void box_unflat(const HostLevel& h, int p, long long f, int* g) {
    for (int d = 0; d < p; ++d) {
        g[d] = h.lo[d] + static_cast<int>(f % h.n1[d]);
        f /= h.n1[d];
    }
}

}  // namespace

std::vector<HostLevel> build_sphere_tree(int p, int base, int L) {
    std::vector<HostLevel> lv(static_cast<size_t>(L) + 1);
    for (int l = 0; l <= L; ++l) {
        HostLevel& h = lv[l];
        h.level = l;
        h.m = pow3(l);
        if (l <= base) {
            for (int d = 0; d < p; ++d) {
                h.lo[d] = 0;
                h.n1[d] = h.m + 1;
            }
        } else {
            const HostLevel& pr = lv[l - 1];
            int mn[3] = {INT_MAX, INT_MAX, INT_MAX}, mx[3] = {-1, -1, -1};
            int g[3] = {0, 0, 0};
            for (long long f = 0; f < pr.n; ++f) {
                if (!(pr.cflag[f] & kCellRefined)) continue;
                box_unflat(pr, p, f, g);
                for (int d = 0; d < p; ++d) {
                    mn[d] = std::min(mn[d], g[d]);
                    mx[d] = std::max(mx[d], g[d]);
                }
            }
            if (mx[0] < 0) throw ConfigError("sphere refinement: no cell to refine at level " + std::to_string(l - 1));
            for (int d = 0; d < p; ++d) {
                h.lo[d] = 3 * mn[d];
                h.n1[d] = 3 * (mx[d] + 1) - h.lo[d] + 1;
            }
        }
        h.n = 1;
        for (int d = 0; d < p; ++d) h.n *= h.n1[d];
        if (h.n >= (1LL << 31)) throw CapacityError("adaptive level box exceeds 2^31 vertices");
        h.cflag.assign(static_cast<size_t>(h.n), 0);
        parallel_for(h.n, [&](long long fa, long long fb) {
        int g[3] = {0, 0, 0};
        for (long long f = fa; f < fb; ++f) {
            box_unflat(h, p, f, g);
            bool inDomain = true;
            for (int d = 0; d < p; ++d) inDomain &= g[d] <= h.m - 1;
            if (!inDomain) continue;
            bool exists = true;
            if (l > base) {
                int pc[3] = {0, 0, 0};
                for (int d = 0; d < p; ++d) pc[d] = g[d] / 3;
                const HostLevel& pr = lv[l - 1];
                const long long pf = box_flat(pr, p, pc);
                exists = pf >= 0 && (pr.cflag[pf] & kCellRefined);
            }
            if (!exists) continue;
            const bool refined = l < L && (l < base || centre_in_sphere(p, l, g));
            h.cflag[f] = static_cast<unsigned char>(kCellExists | (refined ? kCellRefined : 0));
        }
        });
        // vertices: classification (spacetree.cpp:438-466) + finish corner
        h.vflag.assign(static_cast<size_t>(h.n), 0);
        h.estar.assign(static_cast<size_t>(h.n), 0xFF);
        h.succ.assign(static_cast<size_t>(h.n), 0);
        const int nc = 1 << p;
        parallel_for(h.n, [&](long long fa, long long fb) {
        int g[3] = {0, 0, 0};
        for (long long f = fa; f < fb; ++f) {
            box_unflat(h, p, f, g);
            int total = 0, have = 0, refAdj = 0;
            bool cellOk[8] = {false, false, false, false, false, false, false, false};
            for (int e = 0; e < nc; ++e) {  // e: cell = g - 1 + e (exact_ops.cuh convention)
                int c[3] = {0, 0, 0};
                bool in = true;
                for (int d = 0; d < p; ++d) {
                    c[d] = g[d] - 1 + ((e >> d) & 1);
                    in &= c[d] >= 0 && c[d] <= h.m - 1;
                }
                if (!in) continue;
                ++total;
                const long long cf = box_flat(h, p, c);
                if (cf < 0 || !(h.cflag[cf] & kCellExists)) continue;
                ++have;
                cellOk[e] = true;
                if (h.cflag[cf] & kCellRefined) ++refAdj;
            }
            if (have == 0) continue;
            unsigned char fl = kExists;
            const bool hanging = have < total;
            if (hanging) fl |= kHanging;
            if (!hanging && refAdj == have) fl |= kRefined;
            bool bnd = false, cp = l > 0;
            for (int d = 0; d < p; ++d) {
                bnd |= g[d] == 0 || g[d] == h.m;
                cp &= g[d] % 3 == 0;
            }
            if (bnd) fl |= kBoundary;
            if (cp) fl |= kCPoint;
            h.vflag[f] = fl;
            // the latest existing cell around g in traversal (Morton) order
            const int pid = perm_id_host(p, g);
            for (int i = nc - 1; i >= 0; --i) {
                const int e = dev::perm_cell(p, pid, i);
                if (cellOk[e]) {
                    h.estar[f] = static_cast<unsigned char>((~e) & (nc - 1));
                    break;
                }
            }
        }
        });
    }
    // succ, finest level first (Spacetree::classify, spacetree.cpp:491-494)
    for (int l = L; l >= 0; --l) {
        HostLevel& h = lv[l];
        if (l == L) continue;
        parallel_for(h.n, [&](long long fa, long long fb) {
        int g[3] = {0, 0, 0};
        for (long long f = fa; f < fb; ++f) {
            if (!(h.vflag[f] & kExists) || !(h.vflag[f] & kRefined)) continue;
            box_unflat(h, p, f, g);
            const HostLevel& fh = lv[l + 1];
            const int mf = fh.m;
            int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
            for (int d = 0; d < p; ++d) {
                lo[d] = std::max(0, 3 * g[d] - 3);
                hi[d] = std::min(mf, 3 * g[d] + 3);
            }
            int minSucc = INT_MAX;
            int w[3] = {0, 0, 0};
            for (w[2] = p > 2 ? lo[2] : 0; w[2] <= (p > 2 ? hi[2] : 0); ++w[2])
                for (w[1] = p > 1 ? lo[1] : 0; w[1] <= (p > 1 ? hi[1] : 0); ++w[1])
                    for (w[0] = lo[0]; w[0] <= hi[0]; ++w[0]) {
                        const long long wf = box_flat(fh, p, w);
                        if (wf < 0 || !(fh.vflag[wf] & kExists)) continue;
                        const int s = (fh.vflag[wf] & kHanging) ? 0 : fh.succ[wf];
                        minSucc = std::min(minSucc, s);
                    }
            h.succ[f] = static_cast<signed char>(minSucc == INT_MAX ? 0 : 1 + minSucc);
        }
        });
    }
    return lv;
}

void mark_regular_chi(std::vector<HostLevel>& lv, int p) {
    const int L = static_cast<int>(lv.size()) - 1;
    const int nc = 1 << p;
    for (int l = 0; l < L; ++l) {
        HostLevel& h = lv[l];
        const HostLevel& fh = lv[l + 1];
        parallel_for(h.n, [&](long long fa, long long fb) {
        int g[3] = {0, 0, 0};
        for (long long f = fa; f < fb; ++f) {
            if (!(h.vflag[f] & kExists)) continue;
            box_unflat(h, p, f, g);
            bool reg = true;
            for (int e = 0; e < nc && reg; ++e) {
                int c[3] = {0, 0, 0};
                bool in = true;
                for (int d = 0; d < p; ++d) {
                    c[d] = g[d] - 1 + ((e >> d) & 1);
                    in &= c[d] >= 0 && c[d] <= h.m - 1;
                }
                if (!in) continue;
                const long long cf = box_flat(h, p, c);
                reg = cf >= 0 && (h.cflag[cf] & kCellExists) && (h.cflag[cf] & kCellRefined);
            }
            int v[3] = {0, 0, 0};
            const int K = p == 1 ? 5 : p == 2 ? 25 : 125;
            for (int k = 0; k < K && reg; ++k) {
                int kk = k;
                bool interior = true;
                for (int d = 0; d < p; ++d) {
                    v[d] = 3 * g[d] + kk % 5 - 2;
                    kk /= 5;
                    interior &= v[d] >= 1 && v[d] <= fh.m - 1;
                }
                if (!interior) continue;
                const long long vf = box_flat(fh, p, v);
                reg = vf >= 0 && (fh.vflag[vf] & kExists) && fh.estar[vf] == 0;
            }
            if (reg) h.vflag[f] |= kRegularChi;
        }
        });
    }
}

void mark_parents_all(std::vector<HostLevel>& lv, int p) {
    const int L = static_cast<int>(lv.size()) - 1;
    const int nc = 1 << p;
    for (int l = 1; l <= L; ++l) {
        HostLevel& h = lv[l];
        const HostLevel& pr = lv[l - 1];
        parallel_for(h.n, [&](long long fa, long long fb) {
            int g[3] = {0, 0, 0};
            for (long long f = fa; f < fb; ++f) {
                if (!(h.vflag[f] & kExists)) continue;
                box_unflat(h, p, f, g);
                bool all = true;
                for (int e = 0; e < nc && all; ++e) {
                    int pi[3] = {0, 0, 0};
                    for (int d = 0; d < p; ++d) pi[d] = std::min(g[d] / 3, pr.m - 1) + ((e >> d) & 1);
                    const long long pf = box_flat(pr, p, pi);
                    all = pf >= 0 && (pr.vflag[pf] & kExists);
                }
                if (all) h.vflag[f] |= kParentsAll;
            }
        });
    }
}

}  // namespace amr

// ============================================================================
// Host: device state and cycle
// ============================================================================

struct AmrTree::Dev {
    std::vector<dev::LevelConst> kc;
    std::vector<adev::ALvl> lv;
    std::vector<void*> allocations;
    std::vector<int> normOffs;  // block partial offsets per level
    std::vector<adev::ChiList> chiList;  // static trees: per-level chi gather lists (empty: k_amr_chi)
    const unsigned char* chiOrder = nullptr;  // term order of interior kRegularChi vertices (chi_order_table)
    double* partials = nullptr;
    int* dOffs = nullptr;
    double* dNorm = nullptr;
    double* hNorm = nullptr;  // pinned, 2 (L+1)
    double* weights = nullptr;
    std::vector<std::pair<std::string, cudaGraphExec_t>> graphs;  // static-tree cycles (AmrTree::run_cycle)
    bool graphsBroken = false;
    bool backToBack = false;  // graphs only for cycles issued back to back (time_cycles), as Hierarchy
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // dynamic adaptivity: writable views of the per-level tables + staging
    struct DynLevel {
        unsigned char *vflag = nullptr, *cflag = nullptr, *estar = nullptr, *fmask = nullptr, *skip = nullptr,
                      *fflag = nullptr, *fcell = nullptr;
        signed char* succ = nullptr;
        int* xoff = nullptr;
        unsigned *list = nullptr, *slist = nullptr, *cmark = nullptr, *mlist = nullptr;
        double2* extras = nullptr;
        size_t extrasCap = 0;
        // incremental uploads: sweep records, visited cells (kept: the next sweep clears them),
        // changed final vertex / cell bytes; host staging per level
        adev::SweepRec* rec = nullptr;
        unsigned *cidx = nullptr, *fidx = nullptr, *fcidx = nullptr;
        unsigned char *cval = nullptr, *fval = nullptr, *fcval = nullptr;
        unsigned ncells = 0;
        std::vector<adev::SweepRec> hRec;
        std::vector<unsigned> hList, hSlist, hCidx, hFidx, hFcidx, hMark;
        std::vector<unsigned char> hCval, hFval, hFcval;
    };
    unsigned* dMcount = nullptr;
    std::vector<DynLevel> dl;
    std::vector<std::array<double2, 9>> dgTab;
    double2* dgDev = nullptr;  // dgTab per level on the device (k_dyn_special)
    adev::ALvl* dLvs = nullptr;
    adev::MarkCounters* dCnt = nullptr;
    unsigned long long* dHist = nullptr;
    std::vector<unsigned> hList, hSlist, hMark;
    std::vector<int> hXoff;
    std::vector<unsigned char> hFlag, hCell;

    ~Dev() {
        for (auto& g : graphs) cudaGraphExecDestroy(g.second);
        for (void* p : allocations) cudaFree(p);
        if (hNorm) cudaFreeHost(hNorm);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
    }
    template <class T>
    T* alloc(size_t count, cudaStream_t s) {
        void* ptr = nullptr;
        // stream-ordered allocation: a hundred-odd level arrays at setup, each a
        // cudaMalloc otherwise (freed with cudaFree in ~Dev, which is allowed)
        AMR_CUDA(cudaMallocAsync(&ptr, std::max<size_t>(1, count) * sizeof(T), s));
        allocations.push_back(ptr);
        AMR_CUDA(cudaMemsetAsync(ptr, 0, std::max<size_t>(1, count) * sizeof(T), s));
        return static_cast<T*>(ptr);
    }
};

namespace {
// TMG_DYN_CHECK=1: synchronise and check after every dynamic-adaptivity kernel (debugging aid)
void dyn_check(cudaStream_t s, const char* what, int level) {
    static const bool on = [] {
        const char* e = std::getenv("TMG_DYN_CHECK");
        return e && e[0] == '1';
    }();
    if (!on) return;
    const cudaError_t err = cudaStreamSynchronize(s);
    if (err != cudaSuccess)
        throw CudaError(std::string("CUDA error ") + cudaGetErrorString(err) + " after " + what + " at level " +
                        std::to_string(level));
}

int blocks_for_n(long long n, int smCount) {
    const long long need = (n + 255) / 256;
    return static_cast<int>(std::max<long long>(1, std::min<long long>(need, 32LL * smCount)));
}
}  // namespace

AmrTree::AmrTree(const Problem& prob, const std::vector<dev::LevelConst>& kc, const std::vector<Cplx>& diagInterior,
                 cudaStream_t stream, int smCount)
    : prob_(prob), p_(prob.dim), L_(prob.levels), base_(prob.levels - prob.sphereLevels), stream_(stream),
      smCount_(smCount), dev_(new Dev()), diag_(diagInterior) {
    dev_->kc = kc;
    if (prob.fast && (prob.dynStart > 0 || prob.c64))
        throw UnsupportedConfigError("adaptive trees: precision = fast on static (sphere) trees in complex128 only");
    if (prob.dynStart > 0) {
        init_dynamic();
        return;
    }
    if (base_ < 1) throw ConfigError("sphere refinement needs a base level >= 1");
    const char* sp = std::getenv("TMG_AMR_PROFILE");  // setup phase times on stderr
    const bool prof = sp && sp[0] == '1';
    auto tp = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (!prof) return;
        AMR_CUDA(cudaStreamSynchronize(stream_));
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "amr setup %-14s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(t - tp).count());
        tp = t;
    };
    host_ = amr::build_sphere_tree(p_, base_, L_);
    lap("tree");
    amr::mark_regular_chi(host_, p_);
    amr::mark_parents_all(host_, p_);
    lap("marks");
    for (const amr::HostLevel& h : host_)
        for (long long f = 0; f < h.n; ++f) {
            const unsigned char v = h.vflag[f];
            if (!(v & amr::kExists)) continue;
            ++existingCount_;
            if (v & amr::kHanging) ++hangingCount_;
            else if (!(v & amr::kRefined) && !(v & amr::kBoundary)) ++leafCount_;
        }
    if (static_cast<std::size_t>(existingCount_) > prob.maxVertices)
        throw CapacityError("vertex capacity exceeded (" + std::to_string(prob.maxVertices) + ")");
    Dev& D = *dev_;
    D.lv.resize(L_ + 1);
    const char* dbg = std::getenv("TMG_DEBUG_R");
    const bool debugR = dbg && dbg[0] == '1';
    int blocksTotal = 0;
    D.normOffs.push_back(0);
    for (int l = 0; l <= L_; ++l) {
        const amr::HostLevel& h = host_[l];
        adev::ALvl& a = D.lv[l];
        a = adev::ALvl{};
        a.level = l;
        a.m = h.m;
        for (int d = 0; d < 3; ++d) {
            a.lo[d] = h.lo[d];
            a.n1[d] = h.n1[d];
        }
        a.n = static_cast<unsigned>(h.n);
        const size_t n = static_cast<size_t>(h.n);
        a.u = D.alloc<double2>(n, stream_);
        a.sc = D.alloc<double2>(n, stream_);
        a.chi = D.alloc<double2>(n, stream_);
        a.uhat = D.alloc<double2>(n, stream_);
        a.rhat = D.alloc<double2>(n, stream_);
        if (l < L_) {
            a.sf = D.alloc<double2>(n, stream_);
            a.si = D.alloc<double2>(n, stream_);
            a.sinext = D.alloc<double2>(n, stream_);
        }
        if (debugR) a.r = D.alloc<double2>(n, stream_);
        if (l >= base_) a.nodal = D.alloc<double2>(n, stream_);
        auto* vflag = D.alloc<unsigned char>(n, stream_);
        auto* cflag = D.alloc<unsigned char>(n, stream_);
        auto* estar = D.alloc<unsigned char>(n, stream_);
        auto* succ = D.alloc<signed char>(n, stream_);
        AMR_CUDA(cudaMemcpyAsync(vflag, h.vflag.data(), n, cudaMemcpyHostToDevice, stream_));
        AMR_CUDA(cudaMemcpyAsync(cflag, h.cflag.data(), n, cudaMemcpyHostToDevice, stream_));
        AMR_CUDA(cudaMemcpyAsync(estar, h.estar.data(), n, cudaMemcpyHostToDevice, stream_));
        AMR_CUDA(cudaMemcpyAsync(succ, h.succ.data(), n, cudaMemcpyHostToDevice, stream_));
        a.vflag = vflag;
        a.cflag = cflag;
        a.estar = estar;
        a.succ = succ;
        {  // compacted vertex list: warps see uniform work (regular vertices first);
           // chunked count / prefix / fill on the host's cores, same order as a serial scan
            const int nt = static_cast<int>(std::max(1u, std::min(64u, std::thread::hardware_concurrency())));
            const long long chunk = (h.n + nt - 1) / nt;
            std::vector<long long> nreg(nt, 0), nirr(nt, 0);
            auto scan = [&](int t, unsigned* out, long long offReg, long long offIrr) {
                const long long fa = t * chunk, fb = std::min(h.n, fa + chunk);
                long long r = 0, q = 0;
                for (long long f = fa; f < fb; ++f) {
                    const unsigned char v = h.vflag[f];
                    if (!(v & amr::kExists)) continue;
                    const bool regular = !(v & (amr::kHanging | amr::kBoundary));
                    if (out) {
                        if (regular) out[offReg + r] = static_cast<unsigned>(f);
                        else out[offIrr + q] = static_cast<unsigned>(f);
                    }
                    (regular ? r : q) += 1;
                }
                if (!out) {
                    nreg[t] = r;
                    nirr[t] = q;
                }
            };
            {
                std::vector<std::thread> th;
                for (int t = 0; t < nt; ++t) th.emplace_back(scan, t, nullptr, 0, 0);
                for (auto& x : th) x.join();
            }
            long long totReg = 0, totIrr = 0;
            for (int t = 0; t < nt; ++t) {
                totReg += nreg[t];
                totIrr += nirr[t];
            }
            std::vector<unsigned> lst(static_cast<size_t>(totReg + totIrr));
            {
                std::vector<std::thread> th;
                long long oR = 0, oI = totReg;
                for (int t = 0; t < nt; ++t) {
                    th.emplace_back(scan, t, lst.data(), oR, oI);
                    oR += nreg[t];
                    oI += nirr[t];
                }
                for (auto& x : th) x.join();
            }
            auto* dl = D.alloc<unsigned>(lst.size(), stream_);
            AMR_CUDA(cudaMemcpyAsync(dl, lst.data(), lst.size() * sizeof(unsigned), cudaMemcpyHostToDevice, stream_));
            AMR_CUDA(cudaStreamSynchronize(stream_));
            a.list = dl;
            a.nlist = static_cast<unsigned>(lst.size());
        }
        blocksTotal += blocks_for_n(h.n, smCount_);
        D.normOffs.push_back(blocksTotal);
    }
    D.partials = D.alloc<double>(2 * static_cast<size_t>(blocksTotal), stream_);
    D.dOffs = D.alloc<int>(D.normOffs.size(), stream_);
    AMR_CUDA(cudaMemcpyAsync(D.dOffs, D.normOffs.data(), D.normOffs.size() * sizeof(int), cudaMemcpyHostToDevice,
                             stream_));
    D.dNorm = D.alloc<double>(2 * (L_ + 1), stream_);
    AMR_CUDA(cudaMallocHost(&D.hNorm, 2 * (L_ + 1) * sizeof(double)));
    upload_weights();
    AMR_CUDA(cudaEventCreate(&D.ev0));
    AMR_CUDA(cudaEventCreate(&D.ev1));
    lap("alloc+upload");
    if (p_ == 1) build_rhs<1>();
    else if (p_ == 2) build_rhs<2>();
    else build_rhs<3>();
    lap("rhs");
    {  // finest level: every cell is a leaf, chi = the load vector in cell order, constant
        const adev::ALvl& F = D.lv[L_];
        const int nb = blocks_for_n(F.n, smCount_);
        if (p_ == 1) adev::k_amr_chi<1><<<nb, 256, 0, stream_>>>(F, F, D.kc[L_], D.weights, 0);
        else if (p_ == 2) adev::k_amr_chi<2><<<nb, 256, 0, stream_>>>(F, F, D.kc[L_], D.weights, 0);
        else adev::k_amr_chi<3><<<nb, 256, 0, stream_>>>(F, F, D.kc[L_], D.weights, 0);
        AMR_CUDA(cudaGetLastError());
    }
    const char* cl = std::getenv("TMG_CHI_LIST");  // developer A/B
    const char* cd = std::getenv("TMG_CHI_DIRECT");
    chiDirect_ = !(cd && cd[0] == '0');
    if (!(cl && cl[0] == '0')) {
        if (p_ == 1) build_chi_lists<1>();
        else if (p_ == 2) build_chi_lists<2>();
        else build_chi_lists<3>();
    }
    lap("chi lists");
    AMR_CUDA(cudaStreamSynchronize(stream_));
}

// k_amr_chi_list: count pass, warp-group bases on the host, fill pass (static trees;
// the leaf terms use nodal, built once by build_rhs)
// Weight codes of an interior kRegularChi vertex's 5^P terms in traversal order, per
// permutation id: the loops of k_amr_chi_list's kRegularChi branch with every cell present.
template <int P>
const unsigned char* AmrTree::chi_order_table() {
    Dev& D = *dev_;
    if (D.chiOrder) return D.chiOrder;
    constexpr int K = P == 1 ? 5 : P == 2 ? 25 : 125, NC = 1 << P, NT = P == 1 ? 3 : P == 2 ? 9 : 27;
    constexpr int NID = P == 1 ? 1 : P == 2 ? 2 : 6;
    std::vector<unsigned char> tab(static_cast<size_t>(NID) * K);
    for (int pid = 0; pid < NID; ++pid) {
        int k = 0;
        for (int ic = 0; ic < NC; ++ic) {
            const int e = dev::perm_cell(P, pid, ic);
            for (int t = 0; t < NT; ++t) {
                int tt = t, code = 0, mul = 1;
                bool in = true;
                for (int d = 0; d < P; ++d) {
                    const int off = 3 * (((e >> d) & 1) - 1) + tt % 3;
                    tt /= 3;
                    in = in && off >= -2 && off <= 2;
                    code += (off + 2) * mul;
                    mul *= 5;
                }
                if (in) tab[static_cast<size_t>(pid) * K + k++] = static_cast<unsigned char>(code);
            }
        }
        if (k != K) throw CudaError("chi order table: term count");
    }
    unsigned char* d = D.alloc<unsigned char>(tab.size(), stream_);
    AMR_CUDA(cudaMemcpyAsync(d, tab.data(), tab.size(), cudaMemcpyHostToDevice, stream_));
    AMR_CUDA(cudaStreamSynchronize(stream_));
    D.chiOrder = d;
    return d;
}

template <int P>
void AmrTree::build_chi_lists() {
    Dev& D = *dev_;
    D.chiList.assign(L_ + 1, adev::ChiList{});
    for (int l = 0; l < L_; ++l) {
        adev::ALvl& c = D.lv[l];
        const adev::ALvl& fine = D.lv[l + 1];
        if (c.nlist == 0 || fine.n >= (1u << 25)) continue;  // (vf << 7) must fit 32 bits
        const int restrictOn = l + 1 > prob_.ellMin ? 1 : 0;
        adev::ChiList L{};
        L.cnt = D.alloc<int>(c.nlist, stream_);
        L.lcnt = D.alloc<int>(c.nlist, stream_);
        // thread-per-vertex gathers (k_amr_chi_gather) walk interior kRegularChi vertices from the
        // order table; the warp-per-vertex gather of small levels keeps stored lists
        L.direct = (chiDirect_ && c.nlist >= 65536u) ? 1 : 0;
        L.order = chi_order_table<P>();
        const int nb = blocks_for_n(c.nlist, smCount_);
        adev::k_amr_chi_list<P, false><<<nb, 256, 0, stream_>>>(c, fine, D.kc[l], restrictOn, L);
        AMR_CUDA(cudaGetLastError());
        std::vector<int> cnt(c.nlist), lcnt(c.nlist);
        AMR_CUDA(cudaMemcpyAsync(cnt.data(), L.cnt, c.nlist * sizeof(int), cudaMemcpyDeviceToHost, stream_));
        AMR_CUDA(cudaMemcpyAsync(lcnt.data(), L.lcnt, c.nlist * sizeof(int), cudaMemcpyDeviceToHost, stream_));
        AMR_CUDA(cudaStreamSynchronize(stream_));
        const size_t groups = (c.nlist + 31) / 32;
        std::vector<long long> base(groups), lbase(groups);
        long long tb = 0, lt = 0;
        for (size_t w = 0; w < groups; ++w) {
            int mx = 0, lmx = 0;
            for (size_t i = 32 * w; i < std::min<size_t>(32 * w + 32, c.nlist); ++i) {
                mx = std::max(mx, cnt[i]);  // absent (-1) / direct (kChiDirect) positions store nothing
                lmx = std::max(lmx, lcnt[i]);
            }
            base[w] = tb;
            lbase[w] = lt;
            tb += 32LL * mx;
            lt += 32LL * lmx;
        }
        long long* dBase = D.alloc<long long>(groups, stream_);
        long long* dLbase = D.alloc<long long>(groups, stream_);
        AMR_CUDA(cudaMemcpyAsync(dBase, base.data(), groups * sizeof(long long), cudaMemcpyHostToDevice, stream_));
        AMR_CUDA(cudaMemcpyAsync(dLbase, lbase.data(), groups * sizeof(long long), cudaMemcpyHostToDevice, stream_));
        L.base = dBase;
        L.lbase = dLbase;
        L.ent = D.alloc<unsigned>(static_cast<size_t>(std::max<long long>(tb, 1)), stream_);
        L.leaf = D.alloc<double2>(static_cast<size_t>(std::max<long long>(lt, 1)), stream_);
        adev::k_amr_chi_list<P, true><<<nb, 256, 0, stream_>>>(c, fine, D.kc[l], restrictOn, L);
        AMR_CUDA(cudaGetLastError());
        D.chiList[l] = L;
    }
}

void AmrTree::upload_weights() {
    // restriction_weight (cycles.cpp:46-50): per-axis 1/3, 2/3, 1 folded in axis order
    Dev& D = *dev_;
    const int NT = p_ == 1 ? 5 : p_ == 2 ? 25 : 125;
    const double k1d[5] = {1.0 / 3.0, 2.0 / 3.0, 1.0, 2.0 / 3.0, 1.0 / 3.0};
    std::vector<double> w(NT);
    for (int code = 0; code < NT; ++code) {
        double wt = 1.0;
        int cc = code;
        for (int d = 0; d < p_; ++d) {
            wt *= k1d[cc % 5];
            cc /= 5;
        }
        w[code] = wt;
    }
    D.weights = D.alloc<double>(NT, stream_);
    AMR_CUDA(cudaMemcpyAsync(D.weights, w.data(), NT * sizeof(double), cudaMemcpyHostToDevice, stream_));
    AMR_CUDA(cudaStreamSynchronize(stream_));
}

AmrTree::~AmrTree() = default;

namespace {
// TMG_DYN_PROFILE=1: per-sweep wall-clock breakdown of dynamic adaptivity on stderr
struct DynProfile {
    bool on = false;
    std::chrono::steady_clock::time_point t;
    DynProfile() {
        const char* e = std::getenv("TMG_DYN_PROFILE");
        on = e && e[0] == '1';
    }
    void start() { t = std::chrono::steady_clock::now(); }
    double lap(const char* what) {  // ms since the last lap (always measured; printed with TMG_DYN_PROFILE=1)
        const auto now = std::chrono::steady_clock::now();
        const double ms = std::chrono::duration<double, std::milli>(now - t).count();
        if (on) std::fprintf(stderr, " %s %.2fms", what, ms);
        t = now;
        return ms;
    }
};
DynProfile& dyn_profile() {
    static DynProfile p;
    return p;
}
}  // namespace


// ---- dynamic adaptivity (h_max / h_min) ---------------------------------------
// Full-lattice levels 0..reference level; the structure is a dyn::DynTree on
// the host, replayed once per sweep; the numerics stay on the device.
void AmrTree::init_dynamic() {
    Dev& D = *dev_;
    const int Lmax = prob_.levels;
    base_ = prob_.dynStart;
    if (base_ < 1 || base_ > Lmax) throw ConfigError("dynamic adaptivity: bad start level");
    dyn_ = std::make_unique<dyn::DynTree>(p_, base_, Lmax, prob_.ellMin, prob_.hMin, prob_.maxVertices);
    L_ = dyn_->depth();
    host_.assign(static_cast<size_t>(Lmax) + 1, amr::HostLevel{});
    D.lv.resize(static_cast<size_t>(Lmax) + 1);
    D.dl.resize(static_cast<size_t>(Lmax) + 1);
    D.dgTab.resize(static_cast<size_t>(Lmax) + 1);
    int blocksTotal = 0;
    D.normOffs.assign(1, 0);
    for (int l = 0; l <= Lmax; ++l) {
        const dyn::Level& T = dyn_->level(l);
        amr::HostLevel& h = host_[l];
        h.level = l;
        h.m = T.m;
        for (int d = 0; d < 3; ++d) {
            h.lo[d] = 0;
            h.n1[d] = d < p_ ? T.n1 : 1;
        }
        h.n = T.n;
        h.vflag.assign(static_cast<size_t>(h.n), 0);
        h.cflag.assign(static_cast<size_t>(h.n), 0);
        h.estar.assign(static_cast<size_t>(h.n), 0xFF);
        h.succ.assign(static_cast<size_t>(h.n), 0);
        adev::ALvl& a = D.lv[l];
        a = adev::ALvl{};
        a.level = l;
        a.m = h.m;
        for (int d = 0; d < 3; ++d) {
            a.lo[d] = 0;
            a.n1[d] = h.n1[d];
        }
        a.n = static_cast<unsigned>(h.n);
        const size_t n = static_cast<size_t>(h.n);
        a.u = D.alloc<double2>(n, stream_);
        a.sc = D.alloc<double2>(n, stream_);
        a.chi = D.alloc<double2>(n, stream_);
        a.uhat = D.alloc<double2>(n, stream_);
        a.rhat = D.alloc<double2>(n, stream_);
        a.sf = D.alloc<double2>(n, stream_);
        a.si = D.alloc<double2>(n, stream_);
        a.sinext = D.alloc<double2>(n, stream_);
        a.r = D.alloc<double2>(n, stream_);
        a.dg = D.alloc<double2>(n, stream_);
        a.nodal = D.alloc<double2>(n, stream_);  // any level can hold leaf cells (erase marks)
        Dev::DynLevel& w = D.dl[l];
        w.vflag = D.alloc<unsigned char>(n, stream_);
        w.cflag = D.alloc<unsigned char>(n, stream_);
        w.estar = D.alloc<unsigned char>(n, stream_);
        w.fmask = D.alloc<unsigned char>(n, stream_);
        w.skip = D.alloc<unsigned char>(n, stream_);
        w.fflag = D.alloc<unsigned char>(n, stream_);
        w.fcell = D.alloc<unsigned char>(n, stream_);
        w.succ = D.alloc<signed char>(n, stream_);
        w.xoff = D.alloc<int>(n, stream_);
        w.list = D.alloc<unsigned>(n, stream_);
        w.slist = D.alloc<unsigned>(n, stream_);
        w.cmark = D.alloc<unsigned>(n, stream_);
        w.mlist = D.alloc<unsigned>(n, stream_);
        w.rec = D.alloc<adev::SweepRec>(n, stream_);
        w.cidx = D.alloc<unsigned>(n, stream_);
        w.fidx = D.alloc<unsigned>(n, stream_);
        w.fcidx = D.alloc<unsigned>(n, stream_);
        w.cval = D.alloc<unsigned char>(n, stream_);
        w.fval = D.alloc<unsigned char>(n, stream_);
        w.fcval = D.alloc<unsigned char>(n, stream_);
        a.vflag = w.vflag;
        a.cflag = w.cflag;
        a.estar = w.estar;
        a.fmask = w.fmask;
        a.skip = w.skip;
        a.fflag = w.fflag;
        a.fcell = w.fcell;
        a.succ = w.succ;
        a.xoff = w.xoff;
        a.list = w.list;
        a.slist = w.slist;
        a.cmark = w.cmark;
        a.mlist = w.mlist;
        a.feat = D.alloc<double>(n, stream_);
        a.ind = D.alloc<double>(n, stream_);
        a.vmark = D.alloc<unsigned char>(n, stream_);
        // diag after k cells: zero_accumulators, then diag += A_aa per cell (cycles.cpp:205)
        const double2 a0 = D.kc[l].A[0];
        D.dgTab[l][0] = make_double2(0.0, 0.0);
        Cplx acc(0.0);
        for (int k = 1; k <= 8; ++k) {
            acc += Cplx(a0.x, a0.y);
            D.dgTab[l][k] = make_double2(acc.real(), acc.imag());
        }
        blocksTotal += blocks_for_n(h.n, smCount_);
        D.normOffs.push_back(blocksTotal);
    }
    D.partials = D.alloc<double>(2 * static_cast<size_t>(blocksTotal), stream_);
    D.dOffs = D.alloc<int>(D.normOffs.size(), stream_);
    AMR_CUDA(cudaMemcpyAsync(D.dOffs, D.normOffs.data(), D.normOffs.size() * sizeof(int), cudaMemcpyHostToDevice,
                             stream_));
    D.dNorm = D.alloc<double>(2 * (static_cast<size_t>(Lmax) + 1), stream_);
    AMR_CUDA(cudaMallocHost(&D.hNorm, 2 * (static_cast<size_t>(Lmax) + 1) * sizeof(double)));
    D.dLvs = D.alloc<adev::ALvl>(static_cast<size_t>(Lmax) + 1, stream_);
    D.dMcount = D.alloc<unsigned>(static_cast<size_t>(Lmax) + 1, stream_);
    for (int l = 0; l <= Lmax; ++l) D.lv[l].mcount = D.dMcount + l;
    D.dgDev = D.alloc<double2>(9 * (static_cast<size_t>(Lmax) + 1), stream_);
    for (int l = 0; l <= Lmax; ++l)
        AMR_CUDA(cudaMemcpyAsync(D.dgDev + 9 * l, D.dgTab[l].data(), 9 * sizeof(double2), cudaMemcpyHostToDevice,
                                 stream_));
    D.dCnt = D.alloc<adev::MarkCounters>(1, stream_);
    D.dHist = D.alloc<unsigned long long>(64, stream_);
    upload_weights();
    AMR_CUDA(cudaEventCreate(&D.ev0));
    AMR_CUDA(cudaEventCreate(&D.ev1));
    // before the first sweep the tables are the regular tree's classification
    upload_final_flags_full();
    for (int l = 0; l <= Lmax; ++l) {
        Dev::DynLevel& w = D.dl[l];
        const size_t n = static_cast<size_t>(host_[l].n);
        AMR_CUDA(cudaMemcpyAsync(w.vflag, w.fflag, n, cudaMemcpyDeviceToDevice, stream_));
        AMR_CUDA(cudaMemcpyAsync(w.cflag, w.fcell, n, cudaMemcpyDeviceToDevice, stream_));
        D.hList.clear();
        for (long long f = 0; f < host_[l].n; ++f)
            if (host_[l].vflag[f] & amr::kExists) D.hList.push_back(static_cast<unsigned>(f));
        AMR_CUDA(cudaMemcpyAsync(w.list, D.hList.data(), D.hList.size() * sizeof(unsigned), cudaMemcpyHostToDevice,
                                 stream_));
        w.hCidx.clear();  // the cells set in cflag, so that the first sweep clears them
        for (long long f = 0; f < host_[l].n; ++f)
            if (host_[l].cflag[f] & amr::kCellExists) w.hCidx.push_back(static_cast<unsigned>(f));
        AMR_CUDA(cudaMemcpyAsync(w.cidx, w.hCidx.data(), w.hCidx.size() * sizeof(unsigned), cudaMemcpyHostToDevice,
                                 stream_));
        AMR_CUDA(cudaStreamSynchronize(stream_));
        D.lv[l].nlist = static_cast<unsigned>(D.hList.size());
        D.lv[l].nslist = 0;
        w.ncells = static_cast<unsigned>(w.hCidx.size());
    }
    if (p_ == 1) build_rhs<1>();
    else if (p_ == 2) build_rhs<2>();
    else build_rhs<3>();
    AMR_CUDA(cudaStreamSynchronize(stream_));
}

// classification after the sweep -> fflag / fcell (mark) and host_ (field API), in full
void AmrTree::upload_final_flags_full() {
    Dev& D = *dev_;
    existingCount_ = hangingCount_ = leafCount_ = 0;
    for (int l = 0; l <= dyn_->max_level(); ++l) {
        const dyn::Level& T = dyn_->level(l);
        amr::HostLevel& h = host_[l];
        const bool live = l <= dyn_->depth();
        for (long long f = 0; f < h.n; ++f) {
            const unsigned char v = live ? static_cast<unsigned char>(T.vtx[f] & 31) : 0;
            h.vflag[f] = v;
            h.cflag[f] = live ? static_cast<unsigned char>(T.cell[f] & (dyn::kCE | dyn::kCR)) : 0;
            h.succ[f] = T.succ[f];
            if (!(v & amr::kExists)) continue;
            ++existingCount_;
            if (v & amr::kHanging) ++hangingCount_;
            else if (!(v & amr::kRefined) && !(v & amr::kBoundary)) ++leafCount_;
        }
        const size_t n = static_cast<size_t>(h.n);
        AMR_CUDA(cudaMemcpyAsync(D.dl[l].fflag, h.vflag.data(), n, cudaMemcpyHostToDevice, stream_));
        AMR_CUDA(cudaMemcpyAsync(D.dl[l].fcell, h.cflag.data(), n, cudaMemcpyHostToDevice, stream_));
    }
    AMR_CUDA(cudaStreamSynchronize(stream_));
    dyn_->clear_notes();
}

// ... and after a sweep: only the vertices / cells the sweep may have changed
void AmrTree::upload_final_flags() {
    Dev& D = *dev_;
    auto counts = [](unsigned char v, long long& ex, long long& hg, long long& lf) {
        if (!(v & amr::kExists)) return;
        ++ex;
        if (v & amr::kHanging) ++hg;
        else if (!(v & amr::kRefined) && !(v & amr::kBoundary)) ++lf;
    };
    for (int l = 0; l <= dyn_->depth(); ++l) {
        const dyn::Level& T = dyn_->level(l);
        amr::HostLevel& h = host_[l];
        Dev::DynLevel& w = D.dl[l];
        w.hFidx.clear();
        w.hFval.clear();
        w.hFcidx.clear();
        w.hFcval.clear();
        for (long long f : T.vtxNoted) {
            const unsigned char nv = static_cast<unsigned char>(T.vtx[f] & 31), ov = h.vflag[f];
            h.succ[f] = T.succ[f];
            if (nv == ov) continue;
            long long e0 = 0, g0 = 0, f0 = 0, e1 = 0, g1 = 0, f1 = 0;
            counts(ov, e0, g0, f0);
            counts(nv, e1, g1, f1);
            existingCount_ += e1 - e0;
            hangingCount_ += g1 - g0;
            leafCount_ += f1 - f0;
            h.vflag[f] = nv;
            w.hFidx.push_back(static_cast<unsigned>(f));
            w.hFval.push_back(nv);
        }
        for (long long f : T.cellNoted) {
            const unsigned char nc = static_cast<unsigned char>(T.cell[f] & (dyn::kCE | dyn::kCR));
            if (nc == h.cflag[f]) continue;
            h.cflag[f] = nc;
            w.hFcidx.push_back(static_cast<unsigned>(f));
            w.hFcval.push_back(nc);
        }
        const unsigned nv = static_cast<unsigned>(w.hFidx.size()), ncl = static_cast<unsigned>(w.hFcidx.size());
        if (nv) {
            AMR_CUDA(cudaMemcpyAsync(w.fidx, w.hFidx.data(), nv * sizeof(unsigned), cudaMemcpyHostToDevice, stream_));
            AMR_CUDA(cudaMemcpyAsync(w.fval, w.hFval.data(), nv, cudaMemcpyHostToDevice, stream_));
            adev::k_scatter_bytes<<<blocks_for_n(nv, smCount_), 256, 0, stream_>>>(w.fidx, w.fval, nv, w.fflag);
        }
        if (ncl) {
            AMR_CUDA(cudaMemcpyAsync(w.fcidx, w.hFcidx.data(), ncl * sizeof(unsigned), cudaMemcpyHostToDevice,
                                     stream_));
            AMR_CUDA(cudaMemcpyAsync(w.fcval, w.hFcval.data(), ncl, cudaMemcpyHostToDevice, stream_));
            adev::k_scatter_bytes<<<blocks_for_n(ncl, smCount_), 256, 0, stream_>>>(w.fcidx, w.fcval, ncl, w.fcell);
        }
    }
    AMR_CUDA(cudaGetLastError());
    AMR_CUDA(cudaStreamSynchronize(stream_));
    dyn_->clear_notes();
}

// the sweep tables of dyn::DynTree::sweep -> device, proportional to the
// sweep: the previous sweep's entries are cleared, the new records scattered;
// vertex lists (regular first), special list, finish-value slots
void AmrTree::upload_sweep_tables() {
    Dev& D = *dev_;
    L_ = dyn_->depth();
    for (int l = 0; l <= dyn_->max_level(); ++l) {
        adev::ALvl& a = D.lv[l];
        Dev::DynLevel& w = D.dl[l];
        if (a.nlist) adev::k_dyn_clear<<<blocks_for_n(a.nlist, smCount_), 256, 0, stream_>>>(w.vflag, w.estar, w.list,
                                                                                            a.nlist);
        if (w.ncells) adev::k_scatter_bytes<<<blocks_for_n(w.ncells, smCount_), 256, 0, stream_>>>(w.cidx, nullptr,
                                                                                                  w.ncells, w.cflag);
        if (l > L_) {
            a.nlist = a.nslist = 0;
            w.ncells = 0;
            continue;
        }
        const dyn::Level& T = dyn_->level(l);
        w.hRec.clear();
        w.hList.clear();
        w.hSlist.clear();
        int slots = 0;
        std::vector<unsigned>& irregular = w.hFidx;  // scratch: non-regular vertices, listed after the regular ones
        irregular.clear();
        for (long long f : T.sweepList) {
            const unsigned char v = T.sflag[f];
            adev::SweepRec r{};
            r.f = static_cast<unsigned>(f);
            r.flag = v;
            r.estar = T.sestar[f];
            r.fmask = T.sfmask[f];
            r.skip = T.sskip[f];
            r.succ = T.ssucc[f];
            r.xoff = 0;
            if (v & dyn::kSSpecial) {
                w.hSlist.push_back(r.f);
                r.xoff = slots;
                slots += __builtin_popcount(T.sfmask[f]);
            }
            w.hRec.push_back(r);
            if (v & (dyn::kSH | dyn::kSB | dyn::kSSpecial)) irregular.push_back(r.f);
            else w.hList.push_back(r.f);
        }
        w.hList.insert(w.hList.end(), irregular.begin(), irregular.end());
        w.hCidx.assign(T.cellList.begin(), T.cellList.end());
        w.hCval.resize(w.hCidx.size());
        for (size_t i = 0; i < w.hCidx.size(); ++i) w.hCval[i] = T.scell[w.hCidx[i]];
        if (static_cast<size_t>(slots) > w.extrasCap) {
            if (w.extras) AMR_CUDA(cudaFree(w.extras));
            w.extrasCap = std::max<size_t>(static_cast<size_t>(slots), 2 * w.extrasCap);
            AMR_CUDA(cudaMalloc(&w.extras, w.extrasCap * sizeof(double2)));
        }
        a.extras = w.extras;
        const unsigned nrec = static_cast<unsigned>(w.hRec.size()), ncl = static_cast<unsigned>(w.hCidx.size());
        AMR_CUDA(cudaMemcpyAsync(w.rec, w.hRec.data(), nrec * sizeof(adev::SweepRec), cudaMemcpyHostToDevice, stream_));
        AMR_CUDA(cudaMemcpyAsync(w.list, w.hList.data(), w.hList.size() * sizeof(unsigned), cudaMemcpyHostToDevice,
                                 stream_));
        AMR_CUDA(cudaMemcpyAsync(w.slist, w.hSlist.data(), w.hSlist.size() * sizeof(unsigned),
                                 cudaMemcpyHostToDevice, stream_));
        AMR_CUDA(cudaMemcpyAsync(w.cidx, w.hCidx.data(), ncl * sizeof(unsigned), cudaMemcpyHostToDevice, stream_));
        AMR_CUDA(cudaMemcpyAsync(w.cval, w.hCval.data(), ncl, cudaMemcpyHostToDevice, stream_));
        if (nrec)
            adev::k_dyn_scatter<<<blocks_for_n(nrec, smCount_), 256, 0, stream_>>>(w.rec, nrec, w.vflag, w.estar,
                                                                                 w.fmask, w.skip, w.succ, w.xoff);
        if (ncl) adev::k_scatter_bytes<<<blocks_for_n(ncl, smCount_), 256, 0, stream_>>>(w.cidx, w.cval, ncl, w.cflag);
        a.nlist = static_cast<unsigned>(w.hList.size());
        a.nslist = static_cast<unsigned>(w.hSlist.size());
        w.ncells = ncl;
    }
    AMR_CUDA(cudaGetLastError());
    AMR_CUDA(cudaStreamSynchronize(stream_));  // staging vectors are rebuilt next sweep
}

template <int P>
void AmrTree::run_cycle_dyn(const Policy& pol, int n) {
    Dev& D = *dev_;
    const int bpx = pol.bpx ? 1 : 0;
    for (int l = 0; l <= L_; ++l) {
        const adev::ALvl& pr = l > 0 ? D.lv[l - 1] : D.lv[0];
        if (D.lv[l].nlist) {
            adev::k_amr_topdown<P><<<blocks_for_n(D.lv[l].nlist, smCount_), 256, 0, stream_>>>(D.lv[l], pr, bpx);
            phaseMs_[5] += 1;
        }
        dyn_check(stream_, "k_amr_topdown", l);
    }
    AMR_CUDA(cudaMemsetAsync(D.partials, 0, 2 * sizeof(double) * static_cast<size_t>(D.normOffs.back()), stream_));
    adev::AResArgs a{};
    a.ellMin = prob_.ellMin;
    a.bpx = bpx;
    a.hb = (pol.hbMask && !pol.bpx) ? 1 : 0;
    for (int s = 0; s < 12; ++s) {
        const Cplx w = omega_unmasked(pol, s, n);
        a.wTab[s] = make_double2(w.real(), w.imag());
    }
    for (int l = L_; l >= 0; --l) {
        const adev::ALvl& c = D.lv[l];
        if (!c.nlist) continue;
        const int nb = blocks_for_n(c.nlist, smCount_);
        const adev::ALvl& fine = l < L_ ? D.lv[l + 1] : D.lv[l];
        const int restrictOn = (l < L_ && l + 1 > prob_.ellMin) ? 1 : 0;
        adev::k_amr_chi<P><<<nb, 256, 0, stream_>>>(c, fine, D.kc[l], D.weights, restrictOn);
        phaseMs_[5] += c.nslist ? 3 : 2;  // chi, special, residual
        dyn_check(stream_, "k_amr_chi", l);
        if (c.nslist) {
            adev::k_dyn_special<P><<<blocks_for_n(c.nslist, smCount_), 256, 0, stream_>>>(
                c, fine, D.kc[l], D.weights, restrictOn, prob_.ellMin, D.dgDev + 9 * l);
            dyn_check(stream_, "k_dyn_special", l);
        }
        a.lv = c;
        a.par = l > 0 ? D.lv[l - 1] : D.lv[0];
        a.k = D.kc[l];
        for (int k = 0; k < 9; ++k) a.dgTab[k] = D.dgTab[l][k];
        a.partials = D.partials + 2 * static_cast<size_t>(D.normOffs[l]);
        adev::k_amr_residual<P><<<nb, 256, 0, stream_>>>(a);
        dyn_check(stream_, "k_amr_residual", l);
    }
    adev::k_amr_norm_final<<<L_ + 1, 1024, 0, stream_>>>(D.partials, D.dOffs, L_ + 1, D.dNorm);
    phaseMs_[5] += 1;
    AMR_CUDA(cudaGetLastError());
}

namespace {
// select_bins, amr.cpp:43-59
int select_bins(const std::vector<unsigned long long>& hist, unsigned long long total, double goal, bool fromTop) {
    const int bins = static_cast<int>(hist.size());
    int best = 0;
    double bestDist = goal;
    unsigned long long cum = 0;
    for (int k = 1; k <= bins; ++k) {
        const int b = fromTop ? bins - k : k - 1;
        cum += hist[static_cast<size_t>(b)];
        const double dist = std::abs(static_cast<double>(cum) / static_cast<double>(total) - goal);
        if (dist < bestDist - 1e-15) {
            bestDist = dist;
            best = k;
        }
    }
    return best;
}
}  // namespace

template <int P>
AmrMarkStats AmrTree::mark_dyn() {
    Dev& D = *dev_;
    // AmrConfig defaults (amr.hpp:7-15) with the run's h_max / h_min
    constexpr int kBins = 20;
    constexpr double kRefineFraction = 0.10, kEraseFraction = 0.02, kVeto = 1e-2;
    adev::MarkCounters zero{};
    zero.sMinBits = ~0ull;
    AMR_CUDA(cudaMemcpyAsync(D.dCnt, &zero, sizeof(zero), cudaMemcpyHostToDevice, stream_));
    AMR_CUDA(cudaMemcpyAsync(D.dLvs, D.lv.data(), D.lv.size() * sizeof(adev::ALvl), cudaMemcpyHostToDevice, stream_));
    for (int l = 0; l <= L_; ++l)
        adev::k_dyn_features<P><<<blocks_for_n(D.lv[l].n, smCount_), 256, 0, stream_>>>(
            D.dLvs, l, l >= prob_.ellMin ? 1 : 0, D.dCnt);
    dyn_check(stream_, "k_dyn_features", L_);
    adev::MarkCounters cnt{};
    AMR_CUDA(cudaMemcpyAsync(&cnt, D.dCnt, sizeof(cnt), cudaMemcpyDeviceToHost, stream_));
    AMR_CUDA(cudaStreamSynchronize(stream_));
    if (cnt.cand > 0) {
        double smin, smax;
        std::memcpy(&smin, &cnt.sMinBits, 8);
        std::memcpy(&smax, &cnt.sMaxBits, 8);
        const double span = smax - smin;
        if (span > 0.0) {
            AMR_CUDA(cudaMemsetAsync(D.dHist, 0, kBins * sizeof(unsigned long long), stream_));
            for (int l = 0; l <= L_; ++l)
                adev::k_dyn_hist<P><<<blocks_for_n(D.lv[l].n, smCount_), 256, 0, stream_>>>(D.dLvs, l, smin, span,
                                                                                          kBins, D.dHist);
            std::vector<unsigned long long> hist(kBins);
            AMR_CUDA(cudaMemcpyAsync(hist.data(), D.dHist, kBins * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                     stream_));
            AMR_CUDA(cudaStreamSynchronize(stream_));
            const int kRef = select_bins(hist, cnt.cand, kRefineFraction, true);
            const int kErase = select_bins(hist, cnt.cand, kEraseFraction, false);
            for (int l = 0; l <= L_; ++l)
                adev::k_dyn_classify<P><<<blocks_for_n(D.lv[l].n, smCount_), 256, 0, stream_>>>(
                    D.dLvs, l, smin, span, kBins, kRef, kErase, kVeto, D.dCnt);
        }
    }
    AMR_CUDA(cudaMemsetAsync(D.dMcount, 0, D.lv.size() * sizeof(unsigned), stream_));
    for (int l = 0; l <= L_; ++l) {
        adev::k_dyn_refine_cells<P><<<blocks_for_n(D.lv[l].n, smCount_), 256, 0, stream_>>>(
            D.dLvs, l, std::pow(3.0, -l), prob_.hMin, D.dCnt);
        dyn_check(stream_, "k_dyn_refine_cells", l);
    }
    for (int l = std::max(0, prob_.ellMin); l < L_; ++l)
        adev::k_dyn_erase_cells<P><<<blocks_for_n(D.lv[l].n, smCount_), 256, 0, stream_>>>(
            D.dLvs, l, std::pow(3.0, -l), prob_.hMax, D.dCnt);
    dyn_check(stream_, "k_dyn_erase_cells", L_);
    AMR_CUDA(cudaGetLastError());
    AMR_CUDA(cudaMemcpyAsync(&cnt, D.dCnt, sizeof(cnt), cudaMemcpyDeviceToHost, stream_));
    AMR_CUDA(cudaStreamSynchronize(stream_));
    // features, refine translation per level, erase translation per level (+ histogram and classify)
    phaseMs_[5] += 2 * (L_ + 1) + std::max(0, L_ - std::max(0, prob_.ellMin)) + (cnt.cand ? 2 * (L_ + 1) : 0);
    std::vector<unsigned> mcount(D.lv.size());
    AMR_CUDA(cudaMemcpy(mcount.data(), D.dMcount, mcount.size() * sizeof(unsigned), cudaMemcpyDeviceToHost));
    for (int l = 0; l <= L_; ++l) {  // the cell marks take effect in the next traversal
        if (!mcount[l]) continue;
        dyn::Level& T = dyn_->level(l);
        Dev::DynLevel& w = D.dl[l];
        w.hMark.resize(mcount[l]);
        AMR_CUDA(cudaMemcpy(w.hMark.data(), w.mlist, mcount[l] * sizeof(unsigned), cudaMemcpyDeviceToHost));
        for (unsigned e : w.hMark) {
            const long long f = e & 0x7FFFFFFFu;
            if (T.cell[f] & dyn::kCE)
                T.cell[f] = static_cast<unsigned char>(T.cell[f] | ((e >> 31) ? dyn::kEM : dyn::kRM));
        }
        adev::k_clear_marks<<<blocks_for_n(mcount[l], smCount_), 256, 0, stream_>>>(w.mlist, mcount[l], w.cmark);
    }
    AMR_CUDA(cudaGetLastError());
    AmrMarkStats st;
    st.refineVertices = static_cast<long long>(cnt.refineV);
    st.eraseVertices = static_cast<long long>(cnt.eraseV);
    st.refineCells = static_cast<long long>(cnt.refineC);
    st.eraseCells = static_cast<long long>(cnt.eraseC);
    st.vetoConvergence = static_cast<long long>(cnt.vetoConv);
    st.vetoHMin = static_cast<long long>(cnt.vetoHMin);
    st.vetoHMax = static_cast<long long>(cnt.vetoHMax);
    return st;
}

void AmrTree::set_cell_marks(int level, const unsigned char* cells) {
    if (!dyn_) throw UnsupportedConfigError("set_cell_marks: the tree is not dynamically adaptive (h_max / h_min)");
    if (level < 0 || level > dyn_->max_level()) throw ConfigError("set_cell_marks: level out of range");
    dyn::Level& T = dyn_->level(level);
    const unsigned char mk = dyn::kRM | dyn::kEM;
    for (long long f = 0; f < T.n; ++f)
        if (T.cell[f] & dyn::kCE) T.cell[f] = static_cast<unsigned char>((T.cell[f] & ~mk) | (cells[f] & mk));
}

AmrMarkStats AmrTree::mark() {
    if (!dyn_) throw UnsupportedConfigError("mark: the tree is not dynamically adaptive (h_max / h_min)");
    DynProfile& prof = dyn_profile();
    prof.start();
    const AmrMarkStats st = p_ == 1 ? mark_dyn<1>() : p_ == 2 ? mark_dyn<2>() : mark_dyn<3>();
    phaseMs_[4] += prof.lap("mark");
    if (prof.on) std::fprintf(stderr, " | depth %d specials %lld\n", L_, lastCounts_.specialVertices);
    return st;
}

template <int P>
void AmrTree::build_rhs() {
    Dev& D = *dev_;
    const int top = static_cast<int>(host_.size()) - 1;  // static: L_; dynamic: the reference level
    for (int l = dyn_ ? 0 : base_; l <= top; ++l) {
        adev::ALvl& a = D.lv[l];
        const amr::HostLevel& h = host_[l];
        if (prob_.chi == ChiKind::Seeded) {
            const int key = prob_.rhsLattice >= 0 ? prob_.rhsLattice : top;
            long long scale = 1, mkey = 1;
            for (int i = 0; i < key - l; ++i) scale *= 3;
            for (int i = 0; i < key; ++i) mkey *= 3;
            adev::k_amr_seeded<P><<<blocks_for_n(h.n, smCount_), 256, 0, stream_>>>(a, prob_.rhsSeed, scale, mkey,
                                                                                    prob_.rhsSphere ? 1 : 0,
                                                                                    dyn_ ? 1 : 0);
            AMR_CUDA(cudaGetLastError());
            continue;
        }
        // chi_at at x = index * 3^-l (kernels.cpp:72-77, problems.cpp:55-68), glibc sin
        std::vector<double2> nod(static_cast<size_t>(h.n), make_double2(0.0, 0.0));
        const double hh = std::pow(3.0, -l);
        int g[3] = {0, 0, 0};
        for (long long f = 0; f < h.n; ++f) {
            if (!dyn_ && !(h.vflag[f] & amr::kExists)) continue;
            long long ff = f;
            double x[3];
            for (int d = 0; d < p_; ++d) {
                g[d] = h.lo[d] + static_cast<int>(ff % h.n1[d]);
                ff /= h.n1[d];
                x[d] = g[d] * hh;
            }
            double v = 0.0;
            if (prob_.chi == ChiKind::SinProduct) {
                v = static_cast<double>(p_) * M_PI * M_PI;
                for (int d = 0; d < p_; ++d) v *= std::sin(M_PI * x[d]);
            } else if (prob_.chi == ChiKind::BallIndicator) {
                double r2 = 0.0;
                for (int d = 0; d < p_; ++d) r2 += (x[d] - 0.5) * (x[d] - 0.5);
                v = r2 < 0.01 ? 1.0 : 0.0;
            }
            nod[f] = make_double2(v, 0.0);
        }
        AMR_CUDA(cudaMemcpyAsync(a.nodal, nod.data(), nod.size() * sizeof(double2), cudaMemcpyHostToDevice, stream_));
        AMR_CUDA(cudaStreamSynchronize(stream_));
    }
}

// The static tree's cycle is ~3 (L + 1) small launches; when cycles are issued
// back to back (time_cycles) and its arguments do not depend on n (every omega
// policy but the transition / two-phase ones) it is captured once as a CUDA
// graph and replayed with one launch (no host-side state changes in a
// static-tree cycle).  TMG_GRAPH=0: launches.
template <int P>
void AmrTree::run_cycle(const Policy& pol, int n) {
    Dev& D = *dev_;
    std::string sig;
    if (dev::switches().graph && !D.graphsBroken && D.backToBack) {
        for (int s = 0; s < 12; ++s) {
            const Cplx w = omega_unmasked(pol, s, n);
            if (w != omega_unmasked(pol, s, n + 1)) {
                sig.clear();
                break;
            }
            sig.append(reinterpret_cast<const char*>(&w), sizeof(w));
        }
        if (!sig.empty()) {
            const int flags[3] = {pol.bpx ? 1 : 0, pol.hbMask ? 1 : 0, prob_.ellMin};
            sig.append(reinterpret_cast<const char*>(flags), sizeof(flags));
        }
    }
    if (sig.empty()) {
        run_cycle_launches<P>(pol, n);
        return;
    }
    for (auto& g : D.graphs)
        if (g.first == sig) {
            AMR_CUDA(cudaGraphLaunch(g.second, stream_));
            return;
        }
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    bool ok = cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
        try {
            run_cycle_launches<P>(pol, n);
        } catch (...) {
            ok = false;
        }
        ok = cudaStreamEndCapture(stream_, &graph) == cudaSuccess && ok && graph;
    }
    if (ok) ok = cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
    if (graph) cudaGraphDestroy(graph);
    if (!ok) {
        (void)cudaGetLastError();
        D.graphsBroken = true;
        run_cycle_launches<P>(pol, n);
        return;
    }
    if (D.graphs.size() >= 4) {
        cudaGraphExecDestroy(D.graphs.front().second);
        D.graphs.erase(D.graphs.begin());
    }
    D.graphs.emplace_back(sig, exec);
    AMR_CUDA(cudaGraphLaunch(exec, stream_));
}

template <int P>
void AmrTree::run_cycle_launches(const Policy& pol, int n) {
    Dev& D = *dev_;
    const int bpx = pol.bpx ? 1 : 0;
    for (int l = 0; l <= L_; ++l) {
        const adev::ALvl& pr = l > 0 ? D.lv[l - 1] : D.lv[0];
        (prob_.fast ? adev::k_amr_topdown<P, true, true> : adev::k_amr_topdown<P, true, false>)
            <<<blocks_for_n(D.lv[l].nlist, smCount_), 256, 0, stream_>>>(D.lv[l], pr, bpx,
                                                                                               l == L_ ? 1 : 0);
    }
    adev::AResArgs a{};
    a.ellMin = prob_.ellMin;
    a.bpx = bpx;
    a.hb = (pol.hbMask && !pol.bpx) ? 1 : 0;
    for (int s = 0; s < 12; ++s) {
        const Cplx w = omega_unmasked(pol, s, n);
        a.wTab[s] = make_double2(w.real(), w.imag());
    }
    for (int l = L_; l >= 0; --l) {
        const int nb = blocks_for_n(D.lv[l].nlist, smCount_);
        const adev::ALvl& fine = l < L_ ? D.lv[l + 1] : D.lv[l];
        if (l < L_) {  // finest level: chi is the constant load vector (built at setup)
            if (!D.chiList.empty() && D.chiList[l].ent) {
                if (D.lv[l].nlist < 65536u)
                    adev::k_amr_chi_gather_warp<<<blocks_for_n(32LL * D.lv[l].nlist, smCount_), 256, 0, stream_>>>(
                        D.lv[l], fine.rhat, D.weights, D.chiList[l]);
                else
                    adev::k_amr_chi_gather<P><<<nb, 256, 0, stream_>>>(D.lv[l], fine, D.weights, D.chiList[l]);
            }
            else
                adev::k_amr_chi<P><<<nb, 256, 0, stream_>>>(D.lv[l], fine, D.kc[l], D.weights,
                                                             l + 1 > prob_.ellMin ? 1 : 0);
        }
        a.lv = D.lv[l];
        a.par = l > 0 ? D.lv[l - 1] : D.lv[0];
        a.k = D.kc[l];
        a.partials = D.partials + 2 * static_cast<size_t>(D.normOffs[l]);
        if (prob_.fast) {
            for (int s = 0; s < 8; ++s) {
                const double m = static_cast<double>(1 << (P - __builtin_popcount(static_cast<unsigned>(s) & ((1u << P) - 1))));
                a.kAsm[s] = make_double2(m * a.k.A[s].x, m * a.k.A[s].y);
            }
            const Cplx inv = Cplx(1.0) / diag_[static_cast<size_t>(l)];  // the interior diagonal kc[l].div divides by
            a.invDiag = make_double2(inv.real(), inv.imag());
            adev::k_amr_residual<P, true><<<nb, 256, 0, stream_>>>(a);
        } else {
            adev::k_amr_residual<P><<<nb, 256, 0, stream_>>>(a);
        }
    }
    adev::k_amr_norm_final<<<L_ + 1, 1024, 0, stream_>>>(D.partials, D.dOffs, L_ + 1, D.dNorm);
    AMR_CUDA(cudaGetLastError());
}

SweepStats AmrTree::cycle(const Policy& pol, int n) {
    DynProfile& prof = dyn_profile();
    if (dyn_) {
        prof.start();
        lastCounts_ = dyn_->sweep();  // the traversal's structural edits, replayed on the host
        phaseMs_[0] += prof.lap("replay");
        upload_sweep_tables();
        phaseMs_[1] += prof.lap("tables");
    }
    for (int l = std::max(1, prob_.ellMin); l <= L_; ++l)
        if (std::abs(diag_[l]) < 1e-300) throw SingularDiagonalError("vanishing operator diagonal (phi*h^2 resonance?)");
    if (dyn_) {
        if (p_ == 1) run_cycle_dyn<1>(pol, n);
        else if (p_ == 2) run_cycle_dyn<2>(pol, n);
        else run_cycle_dyn<3>(pol, n);
        AMR_CUDA(cudaStreamSynchronize(stream_));  // the norms are read right after anyway
        phaseMs_[2] += prof.lap("device");
        upload_final_flags();
        phaseMs_[3] += prof.lap("final");
    } else if (p_ == 1) run_cycle<1>(pol, n);
    else if (p_ == 2) run_cycle<2>(pol, n);
    else run_cycle<3>(pol, n);
    Dev& D = *dev_;
    AMR_CUDA(cudaMemcpyAsync(D.hNorm, D.dNorm, 2 * (L_ + 1) * sizeof(double), cudaMemcpyDeviceToHost, stream_));
    AMR_CUDA(cudaStreamSynchronize(stream_));
    double mx = 0.0, eu = 0.0, hn = 0.0;
    for (int l = 0; l <= L_; ++l) {
        const double hp = std::pow(std::pow(3.0, -l), p_);
        mx = std::max(mx, D.hNorm[2 * l]);
        eu += D.hNorm[2 * l + 1];
        hn += hp * D.hNorm[2 * l + 1];
    }
    SweepStats st;
    st.maxNorm = std::sqrt(mx);
    st.euclidNorm = std::sqrt(eu);
    st.hNorm = std::sqrt(hn);
    st.updatedFineVertices = leafCount_;
    if (dyn_) {
        st.updatedFineVertices = lastCounts_.updatedFineVertices;
        st.refinedCells = lastCounts_.refinedCells;
        st.erasedCells = lastCounts_.erasedCells;
    }
    return st;
}

namespace {
double2* afield(const adev::ALvl& v, const std::string& f) {
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

long long full_flat(int p, int m, const int* g) {
    long long f = 0, s = 1;
    for (int d = 0; d < p; ++d) {
        f += static_cast<long long>(g[d]) * s;
        s *= m + 1;
    }
    return f;
}
}  // namespace

void AmrTree::get_field(int level, const std::string& name, double* host) const {
    if (level < 0 || level > L_) throw ConfigError("get_field: level out of range");
    // "<field>@all": hanging vertices included (the harness's refd_field_all)
    const bool all = name.size() > 4 && name.compare(name.size() - 4, 4, "@all") == 0;
    const std::string field = all ? name.substr(0, name.size() - 4) : name;
    const amr::HostLevel& h = host_[level];
    long long full = 1;
    for (int d = 0; d < p_; ++d) full *= h.m + 1;
    std::fill(host, host + 2 * full, 0.0);
    const double2* ptr = afield(dev_->lv[level], field);
    if (!ptr) {
        static const char* known[] = {"sf", "si", "sinext", "r"};
        for (const char* k : known)
            if (field == k) return;
        throw ConfigError("get_field: unknown field '" + field + "'");
    }
    std::vector<double2> box(static_cast<size_t>(h.n));
    AMR_CUDA(cudaMemcpyAsync(box.data(), ptr, box.size() * sizeof(double2), cudaMemcpyDeviceToHost, stream_));
    AMR_CUDA(cudaStreamSynchronize(stream_));
    int g[3] = {0, 0, 0};
    for (long long f = 0; f < h.n; ++f) {
        const unsigned char v = h.vflag[f];
        if (!(v & amr::kExists) || ((v & amr::kHanging) && !all)) continue;
        amr::box_unflat(h, p_, f, g);
        const long long ff = full_flat(p_, h.m, g);
        host[2 * ff] = box[f].x;
        host[2 * ff + 1] = box[f].y;
    }
}

void AmrTree::get_flags(int level, unsigned char* flags, signed char* succ, unsigned char* cells) const {
    if (level < 0 || level > L_) throw ConfigError("get_flags: level out of range");
    const amr::HostLevel& h = host_[level];
    long long full = 1;
    for (int d = 0; d < p_; ++d) full *= h.m + 1;
    if (flags) std::fill(flags, flags + full, 0);
    if (succ) std::fill(succ, succ + full, static_cast<signed char>(-1));
    if (cells) std::fill(cells, cells + full, 0);
    int g[3] = {0, 0, 0};
    for (long long f = 0; f < h.n; ++f) {
        if (!(h.vflag[f] & amr::kExists) && !h.cflag[f]) continue;
        amr::box_unflat(h, p_, f, g);
        const long long ff = full_flat(p_, h.m, g);
        if (cells) cells[ff] = h.cflag[f];
        if (!(h.vflag[f] & amr::kExists)) continue;
        if (flags) flags[ff] = h.vflag[f] & 31;  // classification bits only
        if (succ) succ[ff] = h.succ[f];
    }
}

std::uint64_t AmrTree::field_hash(int level, const std::string& field) const {
    // FNV-1a over the full-lattice layout of get_field, streamed plane by plane
    if (level < 0 || level > L_) throw ConfigError("field_hash: level out of range");
    const amr::HostLevel& h = host_[level];
    const double2* ptr = afield(dev_->lv[level], field);
    std::vector<double2> box(static_cast<size_t>(h.n), make_double2(0.0, 0.0));
    if (ptr) {
        AMR_CUDA(cudaMemcpyAsync(box.data(), ptr, box.size() * sizeof(double2), cudaMemcpyDeviceToHost, stream_));
        AMR_CUDA(cudaStreamSynchronize(stream_));
    }
    std::uint64_t hs = 1469598103934665603ull;
    auto feed = [&](double x) {
        const double y = x + 0.0;
        std::uint64_t bits;
        std::memcpy(&bits, &y, 8);
        for (int b = 0; b < 8; ++b) {
            hs ^= (bits >> (8 * b)) & 0xffu;
            hs *= 1099511628211ull;
        }
    };
    const int n1 = h.m + 1;
    long long full = 1;
    for (int d = 0; d < p_; ++d) full *= n1;
    int g[3] = {0, 0, 0};
    for (long long f = 0; f < full; ++f) {
        long long ff = f;
        for (int d = 0; d < p_; ++d) {
            g[d] = static_cast<int>(ff % n1);
            ff /= n1;
        }
        const long long bf = amr::box_flat(h, p_, g);
        double2 v = make_double2(0.0, 0.0);
        if (bf >= 0 && (h.vflag[bf] & amr::kExists) && !(h.vflag[bf] & amr::kHanging)) v = box[bf];
        feed(v.x);
        feed(v.y);
    }
    return hs;
}

void AmrTree::set_random_initial_guess(std::uint64_t seed) {
    Dev& D = *dev_;
    for (int l = L_; l >= 0; --l) {
        const int nb = blocks_for_n(D.lv[l].n, smCount_);
        if (p_ == 1) adev::k_amr_random<1><<<nb, 256, 0, stream_>>>(D.lv[l], seed);
        else if (p_ == 2) adev::k_amr_random<2><<<nb, 256, 0, stream_>>>(D.lv[l], seed);
        else adev::k_amr_random<3><<<nb, 256, 0, stream_>>>(D.lv[l], seed);
        if (l < L_) {
            if (p_ == 1) adev::k_amr_inject<1><<<nb, 256, 0, stream_>>>(D.lv[l], D.lv[l + 1]);
            else if (p_ == 2) adev::k_amr_inject<2><<<nb, 256, 0, stream_>>>(D.lv[l], D.lv[l + 1]);
            else adev::k_amr_inject<3><<<nb, 256, 0, stream_>>>(D.lv[l], D.lv[l + 1]);
        }
    }
    // reset_pipeline_state, cycles.cpp:843-853
    for (int l = 0; l <= L_; ++l) {
        const adev::ALvl& v = D.lv[l];
        for (double2* ptr : {v.sc, v.sf, v.si, v.sinext, v.uhat})
            if (ptr) AMR_CUDA(cudaMemsetAsync(ptr, 0, static_cast<size_t>(v.n) * sizeof(double2), stream_));
    }
    AMR_CUDA(cudaGetLastError());
    AMR_CUDA(cudaStreamSynchronize(stream_));
}

void AmrTree::time_cycles(const Policy& pol, int n0, int count, double* out4) {
    Dev& D = *dev_;
    double totalMs = 0.0;
    D.backToBack = true;
    struct Reset {
        bool& b;
        ~Reset() { b = false; }
    } reset{D.backToBack};
    for (int i = 0; i < count; ++i) {
        AMR_CUDA(cudaEventRecord(D.ev0, stream_));
        if (p_ == 1) run_cycle<1>(pol, n0 + i);
        else if (p_ == 2) run_cycle<2>(pol, n0 + i);
        else run_cycle<3>(pol, n0 + i);
        AMR_CUDA(cudaEventRecord(D.ev1, stream_));
        AMR_CUDA(cudaEventSynchronize(D.ev1));
        float ms = 0.f;
        AMR_CUDA(cudaEventElapsedTime(&ms, D.ev0, D.ev1));
        totalMs += ms;
    }
    out4[0] = totalMs;
    out4[1] = 0.0;
    out4[2] = 0.0;
    out4[3] = static_cast<double>(3 * (L_ + 1));  // top-down L+1, chi L (finest precomputed), residual L+1, norm
}

}  // namespace tmg
