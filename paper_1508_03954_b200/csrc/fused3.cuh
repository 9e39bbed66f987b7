// Fused fine pass for 3D, precision = fast (K2F in DESIGN.md §3).
//
// One kernel does, per fine vertex, everything the cycle needs on the finest
// level: the top-down correction, the residual r = b - H u of the corrected
// iterate, the norm partials, the Jacobi staging sc = omega r / diag, the
// BPX injection into si_{L-1} and the restriction R r into the coarse
// residual.
//
// Fine state ("v-form"): the finest level keeps v = u + sc, the iterate with
// its staged Jacobi correction already applied, plus sc itself for the
// field API (u = v - sc on request).  The reference applies the staged sc at
// the next touch-first (u += sc + P sc_{L-1}, cycles.cpp:119-122); applying it
// when it is formed is the same update in a different rounding order, and
// the next cycle then needs only v:  u' = v + P sc_{L-1} (- P si_{L-1}).
// HBM traffic per fine vertex: v and b read, v and sc written = 64 B
// (80 B with the (u, sc) pair).  v is double-buffered so halo reads never
// race with the owner's writes; sc is write-only.
//
// Structure: 2D tiles (32 x 8 columns) marching in z over a chunk of planes.
// The halo'd (34 x 10) v planes arrive by TMA (cp.async.bulk.tensor.3d) into
// a 4-stage mbarrier ring; the block forms the corrected plane in shared
// memory, every column keeps its centre / edge / corner plane sums in
// registers (z-marching), and the restriction is evaluated separably (x,
// then y, then z accumulators) into per-tile partial sums that a small
// combine kernel adds in a fixed order, so the coarse residual is
// deterministic without atomics.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "fast.cuh"
#include "lattice.cuh"

namespace tmg {
namespace fused3 {

// Tiles of 32 x TY points.  Two kernel shapes over the same tiles (fused3.cu
// Cfg<R>): R = 2 rows per thread on TY / 2 thread rows (128 threads, 4 blocks
// per SM, b tiles by TMA) and R = 1 (256 threads, 3 blocks per SM).  Measured
// at 729^3: complex128 R = 2 -4 % fine-pass time against R = 1 (243^3 -3 %);
// complex64 R = 2 -7 % against R = 1 since session 4 of round 2 (its b tiles
// start at the even column x0 - 1: a TMA box must start 16-byte aligned);
// TMG_F3_ROWS / TMG_F3_ROWS_C64 override.
#ifndef TMG_FUSED_TY
#define TMG_FUSED_TY 8
#endif
#ifndef TMG_F3_ROWS
#define TMG_F3_ROWS 2
#endif
#ifndef TMG_F3_ROWS_C64
#define TMG_F3_ROWS_C64 2
#endif
constexpr int TX = 32, TY = TMG_FUSED_TY;
constexpr int HX = TX + 2, HY = TY + 2;
constexpr int SX = TX / 3 + 3, SY = TY / 3 + 3;  // restriction slots per tile (upper bounds)
// coarse tile feeding the prolongation: parents floor((o-1)/3) .. floor((o+T)/3) + 1 of a tile
// [o, o+T) plus halo, for any tile origin o (T = TX or TY; 13 x 5 for 32 x 8, 13 x 8 for 32 x 16)
constexpr int CX = (TX + 3) / 3 + 2, CY = (TY + 3) / 3 + 2;

struct Geometry {
    int m;      // fine cells per axis (3^L)
    int mc;     // coarse cells per axis
    int nbx, nby, nbz;
    int zc;     // planes per z-chunk (multiple of 3)
    int sz;     // z slots per chunk
};

// Fine-level arrays are double2 (complex128) or float2 (precision =
// fast-complex64, the kernel instantiated with S = float): untyped here.
struct Args {
    void* uNew;
    void* scNew;
    const void* b;
    const double2* scC;   // coarse sc (after the coarse top-down)
    const double2* siC;   // coarse si (BPX)
    double2* sinextC;     // coarse si next (BPX injection)
    double2* partial;     // restriction partials
    double* norms;        // 2 doubles per block
    unsigned n1, n1c;
    Geometry g;
    fast::LevelCoef k;
    int bpx, hb, ellMin, level;
    int chunkBase;        // first global z-chunk of this launch
    int c64;              // fine level in complex64 (float2) storage and arithmetic
    int tmaZ0, tmaZ0c;    // first plane of the fine / coarse tensor maps (z-slab members; else 0)
    int writeSc;          // store the fine sc (else it is re-derived on demand: derive_u)
};

// Tile / z-chunk geometry; the chunk count is a multiple of `parts` (z-slabs:
// every rank gets the same number of chunks) where the lattice allows it.
Geometry geometry(int m, int mc, int parts = 1, int resident = 4 * 148);
int resident_blocks(int smCount);  // co-resident k_fused3 blocks on the device
size_t partial_count(const Geometry& g);
size_t smem_bytes(bool bpx, bool c64 = false);
int blocks(const Geometry& g);

// TMA descriptor for one lattice array (double2 viewed as float64 pairs, or
// float2 as float32 pairs when c64).
// kind 0: fine u / sc halo'd tile, 1: fine b tile, 2: two coarse planes.
// nz > 0: the map covers nz planes from `base` (a z-slab's allocated range)
bool encode_map(CUtensorMap* map, const void* base, unsigned n1, int kind, bool c64 = false, int nz = 0);

// The corrected fine iterate u = v_old + P sc_td(L-1) (- P si(L-1) off the
// cPoints, td-bpx) of the last fused pass, re-derived with the kernel's own
// arithmetic (y, z, then x interpolation of the complex128 coarse values;
// complex64 when c64) on the fine flat indices [fa, fb); boundary points get
// 0.  vOld: the fine state the pass read, scTD / siTD: the level L-1 values it
// prolonged (siTD null: td-add).  The fused pass then need not store the
// write-only fine sc (16 of its 64 B per vertex): sc = v - u.
void derive_u(const void* vOld, const double2* scTD, const double2* siTD, unsigned n1, unsigned n1c, unsigned fa,
              unsigned fb, double2* uOut, bool c64, cudaStream_t s);

// nchunks <= 0: all z-chunks (chunkBase must be 0)
void launch(const Args& a, const CUtensorMap& mapU, const CUtensorMap& mapC, const CUtensorMap& mapI,
            const CUtensorMap& mapB, cudaStream_t s, int nchunks = 0);
// r_{L-1}(W) = sum of the tile partials covering W, fixed order; coarse
// planes [za, zb) (za < 0: all).
// smooth != nullptr: also the level L-1 smoothing of fast::smooth_coarse on the
// interior points (boundary sc / si stay zero), saving its re-read of r.
void combine(const Args& a, double2* rCoarse, int blocks, cudaStream_t s, int za = -1, int zb = -1,
             const fast::ResArgs* smooth = nullptr);

}  // namespace fused3
}  // namespace tmg
