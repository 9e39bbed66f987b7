// Static adaptive spacetree (BASELINE cfg4) on the device.
//
// The reference stores an adaptive tree as per-level hash maps and fires
// createHangingVertex / destroyHangingVertex instead of touch-first / -last
// for vertices whose adjacent cells do not all exist (spacetree.cpp:367-392,
// cycles.cpp:143-171, 305-321).  Here each level is a dense box of the level
// lattice that bounds its existing cells, with per-vertex and per-cell flag
// bytes (the "patch lists with hanging-vertex tables"):
//   vertex: exists, hanging, refined, boundary, cPoint, succ, finish corner;
//   cell:   exists, refined.
// The cycle runs as level passes like the regular exact path, with every
// floating-point sum in the traversal's order, so iterates are bit-identical
// to the reference:
//   * residual / diag: existing cells around a vertex in base-3 Morton order;
//   * chi: leaf-cell loads and restricted fine residuals interleave in
//     traversal time -- the cells around W in Morton order; a leaf cell adds
//     its load when entered, a refined one the restriction of the fine
//     vertices that are touched last inside it, in their finish order (fine
//     cell in child order, then corner index of the vertex in that cell).
//     A fine vertex finishes in the latest existing cell around it, which is
//     precomputed per vertex ("finish corner", estar).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "dyn.hpp"
#include "hierarchy.hpp"

namespace tmg {

namespace dev {
struct LevelConst;  // exact_ops.cuh
}

namespace amr {

enum : unsigned char { kExists = 1, kHanging = 2, kRefined = 4, kBoundary = 8, kCPoint = 16, kRegularChi = 32,
                       kParentsAll = 64 /* static trees only (dynamic trees: dyn::kSCreated) */ };
enum : unsigned char { kCellExists = 1, kCellRefined = 2 };

// One level: a box of the (3^l+1)^p lattice, axis 0 fastest.
struct HostLevel {
    int level = 0;
    int m = 1;  // 3^l
    int lo[3] = {0, 0, 0};
    int n1[3] = {1, 1, 1};
    long long n = 0;
    std::vector<unsigned char> cflag;  // indexed by the cell's lower corner
    std::vector<unsigned char> vflag;
    std::vector<unsigned char> estar;  // corner of the vertex in the cell it finishes in (0xFF: none)
    std::vector<signed char> succ;
};

// Structure of the tree: levels 0..base regular, levels base+1..L refined
// where the parent cell's centre lies in the ball |x - 1/2|^2 < 0.04 (the
// reference harness's refine_all_leaves(level, sphereOnly), applied to
// levels base .. L-1 in turn; oracle/refdriver.cpp).
std::vector<HostLevel> build_sphere_tree(int p, int base, int L);

// kRegularChi: every cell around the vertex is refined and every interior
// fine vertex within two fine steps is touched last as the lower corner of
// its own cell (finish corner 0), so chi is the plain restriction in the
// regular tree's order (no loads, no finish-corner lookups).
void mark_regular_chi(std::vector<HostLevel>& lv, int p);
// kParentsAll: all 2^p corners of the vertex's parent cell (parent_stencil) exist,
// so the top-down prolongation needs no existence look-ups (static trees)
void mark_parents_all(std::vector<HostLevel>& lv, int p);

}  // namespace amr

class AmrTree {
  public:
    AmrTree(const Problem& prob, const std::vector<dev::LevelConst>& kc, const std::vector<Cplx>& diagInterior,
            cudaStream_t stream, int smCount);
    ~AmrTree();

    SweepStats cycle(const Policy& pol, int n);
    // dynamic adaptivity (prob.dynStart > 0): MarkStats of amr.cpp:61-222 on the device
    AmrMarkStats mark();
    bool dynamic() const { return dyn_ != nullptr; }
    // cumulative wall-clock ms of the dynamic phases: host replay, table upload, device sweep,
    // final-classification upload, mark (device + mark download); [5] kernels launched
    const double* phase_ms() const { return phaseMs_; }
    // overwrite the pending cell marks of `level` (4 refineMark, 8 eraseMark per lattice cell)
    void set_cell_marks(int level, const unsigned char* cells);
    int levels() const { return L_; }
    long long leaf_vertices() const { return leafCount_; }
    long long existing_vertices() const { return existingCount_; }
    long long hanging_vertices() const { return hangingCount_; }

    // Full-lattice layout ((3^l+1)^p), zero where the vertex is absent or
    // hanging -- the layout of the reference harness's field dumps.
    void get_field(int level, const std::string& field, double* host) const;
    // flags byte (amr::k*) and succ per lattice point, -1 succ where absent.
    // cells (optional): amr::kCell* per cell, indexed by its lower corner.
    void get_flags(int level, unsigned char* flags, signed char* succ, unsigned char* cells = nullptr) const;
    std::uint64_t field_hash(int level, const std::string& field) const;
    void set_random_initial_guess(std::uint64_t seed);
    void time_cycles(const Policy& pol, int n0, int count, double* out4);

    struct Dev;

  private:
    template <int P>
    void run_cycle(const Policy& pol, int n);
    template <int P>
    void run_cycle_launches(const Policy& pol, int n);
    template <int P>
    void run_cycle_dyn(const Policy& pol, int n);
    template <int P>
    AmrMarkStats mark_dyn();
    void init_dynamic();
    void upload_weights();
    void upload_sweep_tables();
    void upload_final_flags();
    void upload_final_flags_full();
    void refresh_counts();
    template <int P>
    void build_rhs();
    template <int P>
    void build_chi_lists();
    template <int P>
    const unsigned char* chi_order_table();

    Problem prob_;
    bool chiDirect_ = true;  // TMG_CHI_DIRECT=0: stored term lists for every vertex (developer A/B, same bits)
    int p_ = 3, L_ = 1, base_ = 0;
    cudaStream_t stream_;
    int smCount_;
    std::vector<amr::HostLevel> host_;
    std::unique_ptr<dyn::DynTree> dyn_;  // dynamic adaptivity: the structure, replayed per sweep
    dyn::SweepCounts lastCounts_;
    double phaseMs_[6] = {0, 0, 0, 0, 0, 0};  // + [5]: kernels launched
    std::unique_ptr<Dev> dev_;  // device arrays + the per-level exact constants
    std::vector<Cplx> diag_;
    long long leafCount_ = 0, existingCount_ = 0, hangingCount_ = 0;
};

}  // namespace tmg
