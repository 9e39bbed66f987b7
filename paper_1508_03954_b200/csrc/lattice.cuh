// Lattice geometry shared by the exact and fast kernels: one array per field
// per level over the (3^l+1)^d vertex lattice, axis 0 fastest, complex128
// as double2.
#pragma once

#include <cuda_runtime.h>

#include "exact_ops.cuh"

#include <algorithm>
#include <cstdlib>
#include <utility>

namespace tmg {
namespace dev {

// Programmatic dependent launch: kernels launched with launch_k may be
// dispatched while their predecessor in the stream drains; each such kernel
// starts with griddep_wait(), which returns once the predecessor grid has
// completed and its memory is visible (a no-op for ordinary launches).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Developer A/B switches (environment), snapshotted when a
// hierarchy is constructed (refresh_switches) instead of being read on the
// launch path.  Every switch selects an older, bit-identical implementation.
struct Switches {
    bool pdl = true;        // TMG_PDL=0: ordinary launches
    bool triCoarse = true;  // TMG_TRI_COARSE=0: one thread per point for big coarse top-downs
    bool up = true;         // TMG_UP=0: restrict / smooth launches + cluster chain
    bool pyr = true;        // TMG_PYR=0: per-level top-down launches
    int gridCap = 32;       // TMG_GRID_CAP: blocks per SM of grid-stride launches
    int zchunks = 0;        // TMG_ZCHUNKS: z-chunk count of the 3D fused pass (0: automatic)
    bool graph = true;      // TMG_GRAPH=0: launch the fast cycle's kernels one by one (no CUDA graph)
};
inline Switches& switches() {
    static Switches s;
    return s;
}
inline void refresh_switches() {
    auto on = [](const char* name) {
        const char* e = std::getenv(name);
        return !(e && e[0] == '0');
    };
    Switches& s = switches();
    s.pdl = on("TMG_PDL");
    s.triCoarse = on("TMG_TRI_COARSE");
    s.up = on("TMG_UP");
    s.pyr = on("TMG_PYR");
    const char* cap = std::getenv("TMG_GRID_CAP");
    s.gridCap = cap ? std::max(1, std::atoi(cap)) : 32;
    const char* zc = std::getenv("TMG_ZCHUNKS");
    s.zchunks = zc ? std::max(1, std::atoi(zc)) : 0;
    s.graph = on("TMG_GRAPH");
}

inline bool pdl_enabled() { return switches().pdl; }

template <class... KArgs, class... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    if (!pdl_enabled()) {
        kernel<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
        return;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

struct Lvl {
    double2* u;
    double2* sc;
    double2* sf;
    double2* si;
    double2* sinext;
    double2* chi;
    double2* uhat;
    double2* rhat;
    double2* r;  // optional debug copy of the residual
    double2* scOut;  // coarse top-down output (null: in place into sc; the fused passes' level L-1)
    unsigned m;   // 3^l
    unsigned n1;  // 3^l + 1
    unsigned n;   // (3^l+1)^p
    int level;
};

template <int P>
__device__ __forceinline__ void unflat(unsigned f, unsigned n1, int* idx) {
#pragma unroll
    for (int d = 0; d < P; ++d) {
        idx[d] = static_cast<int>(f % n1);
        f /= n1;
    }
}

template <int P>
__device__ __forceinline__ unsigned flat(const int* idx, unsigned n1) {
    unsigned f = 0, s = 1;
#pragma unroll
    for (int d = 0; d < P; ++d) {
        f += static_cast<unsigned>(idx[d]) * s;
        s *= n1;
    }
    return f;
}

template <int P>
__device__ __forceinline__ bool on_boundary(const int* idx, int m) {
    bool b = false;
#pragma unroll
    for (int d = 0; d < P; ++d) b |= (idx[d] == 0) | (idx[d] == m);
    return b;
}

template <int P>
__device__ __forceinline__ bool is_cpoint(const int* idx) {
    bool c = true;
#pragma unroll
    for (int d = 0; d < P; ++d) c &= (idx[d] % 3 == 0);
    return c;
}

// proj/src/transfer.cpp:20-40, one axis fold: exact copies at rel 0 / 3.
// Branch-free (rel varies across the lanes of a warp): the blend is formed
// always and the exact copies selected, so the result is the same bits.
__device__ __forceinline__ double2 lerp_rel(double2 c0, double2 c1, int rel) {
    const double w0 = rel == 1 ? (2.0 / 3.0) : (1.0 / 3.0);
    const double w1 = rel == 1 ? (1.0 / 3.0) : (2.0 / 3.0);
    const double2 r = xadd(xscale(w0, c0), xscale(w1, c1));
    return rel == 0 ? c0 : rel == 3 ? c1 : r;
}

template <int P>
__device__ __forceinline__ double2 prolong(double2 (&v)[1 << P], const int* rel) {
    int n = 1 << P;
#pragma unroll
    for (int d = 0; d < P; ++d) {
        n >>= 1;
#pragma unroll
        for (int i = 0; i < (1 << (P - 1 - d)); ++i) v[i] = lerp_rel(v[2 * i], v[2 * i + 1], rel[d]);
    }
    return v[0];
}


// Block-level (max |r|^2, sum |r|^2) -> partials[2*blockIdx.x + {0,1}];
// fixed shuffle/shared-memory tree, so the result is deterministic.
__device__ __forceinline__ void block_norms(double mx, double sm, double* partials) {
    __shared__ double smax[32], ssum[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        sm += __shfl_xor_sync(0xffffffffu, sm, o);
    }
    const int nthreads = blockDim.x * blockDim.y;
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    const int w = tid >> 5, l = tid & 31;
    if (l == 0) {
        smax[w] = mx;
        ssum[w] = sm;
    }
    __syncthreads();
    if (w == 0) {
        const int nw = nthreads >> 5;
        mx = l < nw ? smax[l] : 0.0;
        sm = l < nw ? ssum[l] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            sm += __shfl_xor_sync(0xffffffffu, sm, o);
        }
        if (l == 0) {
            const unsigned b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
            partials[2 * b] = mx;
            partials[2 * b + 1] = sm;
        }
    }
}

}  // namespace dev
}  // namespace tmg
