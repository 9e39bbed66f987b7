// Verification cycles (bu_fas, textbook_add, evaluate_residual_norms) on the
// device hierarchy's exact storage; see vcycles.cu.
#pragma once

#include <cuda_runtime.h>

#include "fast.cuh"
#include "lattice.cuh"

namespace tmg {
namespace vc {

struct Ctx {
    const dev::Lvl* lv;          // levels 0..L (exact storage: u, sc, sf, si, sinext, chi, uhat)
    int L, ellMin;
    const fast::LevelCoef* fc;   // assembled stencil + 1/diag per level
    double2* const* r;           // per-level residual scratch
    double* partials;            // norm block partials
    double* dNorm;               // 2 doubles
    cudaStream_t stream;
    int smCount;
};

// textbook_add (cycles.cpp:605-714): Jacobi on the residual, correction scheme,
// u_l += omegaCG P u_{l-1} on the way up.
void textbook_add(int P, const Ctx& x, double2 omegaS, double2 omegaCG);
// bu_fas (cycles.cpp:374-603) on a regular tree; wNonCp / wCp: omega_of per level
// for non-C-points / C-points.
void bu_fas(int P, const Ctx& x, const double2* wNonCp, const double2* wCp, int bpx);
// evaluate_residual_norms (cycles.cpp:716-786): (max |r|^2, sum |r|^2) of the
// finest level's interior into out2 (host).
void residual_norms(int P, const Ctx& x, double* out2);

}  // namespace vc
}  // namespace tmg
