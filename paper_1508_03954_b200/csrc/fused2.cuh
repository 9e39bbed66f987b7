// Fused fine pass for 2D (fast precision): the 2D counterpart of fused3.
//
// One block owns a strip of TX columns and a y-chunk of rows and marches
// the rows once: correction u + sc + P sc_{L-1} (- P si, BPX) of the row into
// shared memory, the 9-point operator as two running row accumulators, the
// residual, norms, Jacobi staging, BPX injection, and the restriction --
// accumulated along y per column, reduced in x one step later on the next
// row barrier -- into per-strip partials summed in fixed order by k_combine2.
// The finest level keeps v = u + sc (the "v-form" of fused3.cuh): v and b
// are read once, v and sc written once -- 64 B per fine vertex instead of the
// 128 B of the unfused correct / residual / restrict kernels.
#pragma once

#include <cuda_runtime.h>

#include "fast.cuh"

namespace tmg {
namespace fused2 {

#ifndef TMG_F2_TX
#define TMG_F2_TX 256
#endif
constexpr int TX = TMG_F2_TX;  // strip width (threads per block)
constexpr int SXP = TX / 3 + 3;        // restriction slots per strip (upper bound)
constexpr int CXW = (TX + 1) / 3 + 3;  // coarse columns feeding the strip's prolongation
constexpr int kMaxYc = 48;             // rows per chunk cap (the chunk's coarse rows are staged in shared memory)

struct Geometry {
    int m, mc;    // fine / coarse cells per axis
    int nbx, nby; // strips in x, row chunks in y
    int yc;       // rows per chunk (multiple of 3)
    int sy;       // coarse-row slots per chunk
};

struct Args {
    double2* uNew;        // next state v
    double2* scNew;       // staged correction (write-only, field API)
    const double2* u;     // state v
    const double2* sc;    // unused (kept for layout symmetry)
    const double2* b;
    const double2* scC;
    const double2* siC;
    double2* sinextC;
    double2* partial;
    double* norms;
    unsigned n1, n1c;
    Geometry g;
    fast::LevelCoef k;
    int bpx, hb, ellMin, level;
    int writeSc;          // store the fine sc (else re-derived on demand: derive_u)
    int c64;              // u / uNew / scNew / b hold complex64 (float2) behind the double2 pointers
};

Geometry geometry(int m, int mc, int smCount);
// fused3::derive_u for the 2D pass (its phase B: y, then x interpolation)
void derive_u(const double2* vOld, const double2* scTD, const double2* siTD, unsigned n1, unsigned n1c, unsigned fa,
              unsigned fb, double2* uOut, bool c64, cudaStream_t s);
size_t partial_count(const Geometry& g);
int blocks(const Geometry& g);
void launch(const Args& a, cudaStream_t s);
// smooth != nullptr: also the level L-1 smoothing (fast::smooth_coarse) on the
// interior points, as fused3::combine
void combine(const Args& a, double2* rCoarse, cudaStream_t s, const fast::ResArgs* smooth = nullptr);

}  // namespace fused2
}  // namespace tmg
