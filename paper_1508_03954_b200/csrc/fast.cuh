// Fast-precision cycle kernels (precision = fast).
//
// Same cycle as the exact path evaluated the way a GPU
// wants it, mathematically identical and different only by rounding:
//  * the fine operator is applied as its assembled 3^d-point stencil with one
//    complex coefficient per neighbour class (centre / face / edge / corner:
//    2^(d-k) A_k for a neighbour differing on k axes), with FMA;
//  * the coarse levels run in correction form: on a regular grid with uniform
//    theta and constant phi the FAS coarse residual chi_l - H_l u_l equals
//    R r_{l+1} exactly (Lemma 2 + Galerkin, proj/tests/test_cycles.cpp:233-259
//    and Lemma 1 :217-231), so coarse levels carry only sc, the restricted
//    residual and the BPX si -- no coarse matvec, no u-hat;
//  * the Jacobi division uses the level's precomputed 1/diag.
#pragma once

#include <cuda_runtime.h>

#include "lattice.cuh"

namespace tmg {
namespace fast {

struct LevelCoef {
    double2 c[4];     // stencil coefficient per neighbour class (popcount of the offset)
    double2 invDiag;  // 1 / diag of an interior vertex
    double2 wRaw;     // omega_unmasked(pol, L - l, n)
};

struct ResArgs {
    dev::Lvl lv;   // the level being smoothed
    dev::Lvl par;  // level l-1: BPX si injection target
    LevelCoef k;
    int ellMin;
    int bpx;
    int hb;
    double* partials;
};

// Fine level: u += sc + P sc_{L-1} (- P si_{L-1} at non-cPoints, BPX).
void correct_fine(int P, const dev::Lvl& f, const dev::Lvl& pr, int bpx, int blocks, cudaStream_t s);
// Coarse level l < L: sc_l += P sc_{l-1} (- P si_{l-1}, BPX).
// (za, zb): plane range of the last axis, za < 0 for the whole level.
void topdown_coarse(int P, const dev::Lvl& c, const dev::Lvl& pr, int bpx, int blocks, cudaStream_t s, int za = -1,
                    int zb = -1);
// Load vector b = massScale (M x..x M) f on the interior of the finest level
// (planes [za, zb) of the last axis in 3D; za < 0: all).
void load_vector(int P, const dev::Lvl& F, const double2* f, double2 ms, int blocks, cudaStream_t s, int za = -1,
                 int zb = -1);
// Fine residual r = b - H u, norms, sc = omega r / diag, BPX injection; r to lv.rhat.
// Returns the number of blocks that wrote norm partials.
int residual_fine(int P, const ResArgs& a, int smCount, cudaStream_t s);
int residual_fine_blocks(int P, const dev::Lvl& f, int smCount);
// r_{l-1} = R r_l on interior coarse vertices (rhat arrays).
// smooth != nullptr: also the coarse level's smoothing (smooth_coarse) on the
// interior points, on the value just formed.
void restrict_level(int P, const dev::Lvl& fine, const dev::Lvl& coarse, const double* weights, int blocks,
                    cudaStream_t s, int za = -1, int zb = -1, const ResArgs* smooth = nullptr);
// Coarse chains (one cooperative launch per phase, grid barrier between levels):
//   chain_down: top-down of levels 1..top;
//   chain_up:   [restrict fine -> top,] then for l = top..1 smoothing of l and
//               restriction l -> l-1, then the final norm reduction.
constexpr int kChainThreads = 512;
constexpr int kMaxChainLevels = 10;
struct ChainArgs {
    dev::Lvl lv[kMaxChainLevels];
    LevelCoef k[kMaxChainLevels];
    dev::Lvl fine;
    int top;            // highest coarse level in the chain (L - 1)
    int firstRestrict;  // restrict fine.rhat into lv[top] first (unfused fine pass)
    int ellMin, bpx, hb;
    unsigned* bar;      // grid barrier state: arrivals, generation
    const double* normPartials;
    int normBlocks;
    double* normOut;    // nullptr: no norm reduction
    int cluster;        // 1: launched as one thread-block cluster (hardware cluster barriers)
};
int chain_grid(int P, int smCount);
int chain_cluster_size();
void chain_down(int P, const ChainArgs& a, int grid, cudaStream_t s);
void chain_up(int P, const ChainArgs& a, int grid, cudaStream_t s);
// The whole bottom-up below the level a.fine (its r complete and smoothed):
// for l = top .. 1 restriction into l fused with the smoothing of l, grid
// barriers between big steps, the small steps on the last CTA (cooperative
// launch, up to two CTAs per SM; count: zeroed counter, re-armed by the kernel).
size_t up_coop_smem(int P, const ChainArgs& a);
void up_coop(int P, const ChainArgs& a, unsigned* count, int smCount, cudaStream_t s);

// Every coarse top-down of one cycle in one launch without a grid-wide
// barrier ("pyramid"): each CTA owns a box of level T and rebuilds in shared
// memory the ancestor boxes (levels T-1 .. 0) its prolongation needs, each
// from the one above it; only level T is written (the intermediate levels'
// top-down values are transients: the bottom-up overwrites their sc).  Same
// arithmetic as chain_down + topdown_coarse, bit for bit.  P = 2, 3.
constexpr int kPyrMaxLevels = 16;
struct PyrLevel {
    const double2* sc;
    const double2* si;
    int m, n1;
};
struct PyrArgs {
    PyrLevel lv[kPyrMaxLevels];
    double2* scT;         // level T top-down output (== scTin: in place)
    const double2* scTin; // level T staged sc
    int T, bpx;
    int bz;               // points per thread (tile extent along the last axis / rows / 8)
    int nbx, nby;         // tiles along axes 0, 1
    int off[kPyrMaxLevels];  // shared-memory offset (double2) of level l's box (td, then si)
    int cap[kPyrMaxLevels];  // box capacity (points) of level l
};
// Builds the launch geometry for level T of the given levels (sc / si / m / n1
// of levels 0..T); returns the dynamic shared memory bytes.
size_t pyramid_setup(int P, PyrArgs& a, int T);
void topdown_pyramid(int P, const PyrArgs& a, size_t smem, cudaStream_t s);

// Coarse smoothing: sc_l = omega r_l / diag, si commit, BPX injection into l-1.
void smooth_coarse(int P, const ResArgs& a, int blocks, cudaStream_t s, int za = -1, int zb = -1);

}  // namespace fast
}  // namespace tmg
