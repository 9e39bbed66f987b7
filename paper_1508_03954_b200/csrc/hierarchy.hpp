// Device-resident multilevel hierarchy of a regular 3^d spacetree: the B200
// replacement of the reference's hash-per-level Spacetree storage
// (proj/src/spacetree.cpp) plus the td_add / td_bpx cycle
// (proj/src/cycles.cpp:57-354) as level passes of sm_100a kernels.
//
// Storage: one lattice array per field per level, (3^l+1)^d vertices, axis 0
// fastest, complex128 as interleaved double2 (16-byte vector loads/stores).
#pragma once

#include <array>
#include <complex>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace tmg {

using Cplx = std::complex<double>;

// Error classes mirror proj/include/treemg/types.hpp:18-38 so that the C-ABI
// maps them to the same status codes (proj/src/capi.cpp:28-43).
struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct UnsupportedConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CapacityError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct SingularDiagonalError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

enum class OmegaKind { JacobiOnly = 0, UndampedCG = 1, LGrid = 2, Exponential = 3, Transition = 4 };

struct Policy {  // OmegaPolicy, proj/include/treemg/cycles.hpp:17-24
    OmegaKind kind = OmegaKind::Exponential;
    Cplx omegaS = Cplx(0.8, 0.0);
    int lGrid = 2;
    bool hbMask = false;
    bool bpx = false;
    bool twoPhase = false;
};

enum class ChiKind { Zero = 0, SinProduct = 1, BallIndicator = 2, Seeded = 3, Gaussian = 4 };

struct Problem {
    int dim = 2;
    int levels = 1;
    int ellMin = 1;
    double theta = 0.0;
    Cplx phi = Cplx(0.0);
    ChiKind chi = ChiKind::SinProduct;
    std::uint64_t rhsSeed = 12345;
    bool rhsSphere = false;
    int rhsLattice = -1;  // level the seeded rhs is keyed on (-1: levels)
    bool fast = false;    // precision = fast
    bool c64 = false;     // precision = fast-complex64: fine level in complex64 storage / arithmetic (2D / 3D fused passes)
    bool hostNorms = false;  // norms = host: reference-order sums of |r| on the host (exact mode)
    int zParts = 1;          // fused fine pass: z-chunks come in multiples of this (z-slabs)
    bool gaussian = false;   // 2D gaussian scenario: per-cell phi and absorbing-layer theta (exact only)
    int channels = 1;        // unknowns per vertex (kernels.cpp:33-66; exact precision for > 1)
    Cplx coupling = Cplx(0.0);  // A_ij for i != j (runner.cpp:152-157)
    int sphereLevels = 0;    // static adaptive tree: levels-sphereLevels regular, refined inside |x-1/2|^2<0.04
    // dynamic adaptivity (h_max / h_min runs, runner.cpp:206-366): dynStart > 0 builds the regular
    // tree of that depth; levels is the reference level (level_for_h(h_min)), the deepest refinement
    int dynStart = 0;
    double hMax = 0.0, hMin = 0.0;
    std::size_t maxVertices = 8u * 1024u * 1024u;
    int device = 0;
    // z-slab member (SlabGroup): the fine-level planes [slabLo, slabHi)
    // are owned; levels L and L-1 are allocated only over the planes the slab
    // reads / writes (owned + halos), behind global-index base pointers
    int slabLo = -1, slabHi = -1;
};

struct SweepStats {  // SweepStats, cycles.hpp:37-45
    double maxNorm = 0.0, euclidNorm = 0.0, hNorm = 0.0;  // aggregated over channels (runner.cpp:68-77)
    long long updatedFineVertices = 0;
    int refinedCells = 0, erasedCells = 0;  // dynamic adaptivity: structural edits of the sweep
    std::vector<double> chMax, chEuclid, chH;  // per channel (channels > 1)
};

struct AmrMarkStats {  // MarkStats, amr.hpp:19-27
    long long refineVertices = 0, eraseVertices = 0, refineCells = 0, eraseCells = 0;
    long long vetoConvergence = 0, vetoHMin = 0, vetoHMax = 0;
};

// Makes `device` current for its lifetime and restores the caller's device:
// a handle's kernels run on its own device whatever is current on the calling
// thread (treemg.h: a handle may move between threads).
struct DeviceScope {
    int prev = -1, want;
    explicit DeviceScope(int device);
    ~DeviceScope();
    DeviceScope(const DeviceScope&) = delete;
    DeviceScope& operator=(const DeviceScope&) = delete;
};

// omega_unmasked, proj/src/cycles.cpp:11-31 (host, same libstdc++ arithmetic)
Cplx omega_unmasked(const Policy& pol, int succ, int n);

class Hierarchy {
  public:
    explicit Hierarchy(const Problem& prob);
    ~Hierarchy();
    Hierarchy(const Hierarchy&) = delete;
    Hierarchy& operator=(const Hierarchy&) = delete;

    // One cycle.  bpx selects td_bpx (hb mask forced off, cycles.cpp:345-354).
    SweepStats cycle(const Policy& pol, int n);
    // Verification cycles of a regular tree in exact storage (precision = exact),
    // each followed by evaluate_residual_norms: bu_fas (cycles.cpp:374-603) and
    // textbook_add (cycles.cpp:605-714).
    SweepStats bu_fas(const Policy& pol, int n);
    SweepStats textbook_add(Cplx omegaS, Cplx omegaCG);

    // Dynamic adaptivity: mark (amr.cpp:61-222) on the device after a sweep; the
    // marks take effect in the next cycle (refine on descent, erase on backtracking).
    AmrMarkStats mark();
    // overwrite the pending cell marks of a dynamically adaptive tree (4 refine, 8 erase per lattice cell)
    void set_cell_marks(int level, const unsigned char* cells);
    // dynamic adaptivity: cumulative ms of host replay, table upload, device sweep, final upload, mark;
    // out6[5]: kernels launched
    void dyn_phase_ms(double* out6) const;
    long long existing_vertices() const;  // adaptive trees: stored vertices (hanging included)

    int dim() const;
    int levels() const;  // current depth (grows under dynamic adaptivity)
    long long lattice_size(int level) const;
    long long interior_fine_vertices() const;
    // adaptive trees: flags byte / succ per lattice point (amr.hpp); false if regular
    bool get_flags(int level, unsigned char* flags, signed char* succ, unsigned char* cells = nullptr) const;
    long long hanging_vertices() const;

    void get_field(int level, const std::string& field, double* host) const;
    void set_field(int level, const std::string& field, const double* host);
    void set_fine_interior_u(const double* host);
    void set_random_initial_guess(std::uint64_t seed);
    void set_fine_rhs(const double* hostNodalChi);
    std::uint64_t field_hash(int level, const std::string& field) const;

    // Adds one uniformly refined level on top (FMG unfolding through
    // refine_cell of every leaf + classify()): the new
    // level's u is p-linearly prolonged, its other payload zero.
    // toComplex64: the new finest level in complex64 (FMG's last unfolding of a precision = fast-complex64 run;
    // the stages below it run in complex128)
    void unfold(bool toComplex64 = false);

    // Timing helpers (CUDA events on the hierarchy stream).
    void time_cycles(const Policy& pol, int n0, int count, bool flushL2, double* out4);
    void e2e_step(const Policy& pol, int n, const double* hostChi, double* out3);

    struct Impl;
    Impl* raw() { return impl_.get(); }

  private:
    std::unique_ptr<Impl> impl_;
};

// z-slab decomposition of a 3D fast-precision hierarchy: the
// fine level and level L-1 are sharded in z, levels <= L-2 are replicated.
// Either K "virtual" slabs in one process on one device (transfers are
// device copies -- the test mode) or one slab per process/GPU over NCCL.
class SlabGroup {
  public:
    // ncclId == nullptr: `local` slabs in this process (rank 0, world = local),
    // spread round-robin over `devices` GPUs from prob.device (transfers are
    // device / peer copies); else one slab for `rank` of `world` over NCCL.
    SlabGroup(const Problem& prob, int local, int rank, int world, const void* ncclId, int devices = 1);
    ~SlabGroup();
    SlabGroup(const SlabGroup&) = delete;
    SlabGroup& operator=(const SlabGroup&) = delete;

    SweepStats cycle(const Policy& pol, int n);
    // Fine-level u of the planes owned by the local slabs, full-lattice layout
    // (other planes left untouched in `host`).
    void get_fine_u(double* host);
    // Whole-lattice u / sc of any level gathered from the local slabs (all slabs
    // local: ncclId == nullptr), bitwise what one GPU's Hierarchy::get_field gives.
    void get_field(int level, const std::string& field, double* host);
    std::uint64_t field_hash(int level, const std::string& field);
    int levels() const;
    long long interior_fine_vertices() const;
    // FMG's last unfolding onto slabs: a group one level deeper than `coarse`
    // (a single-GPU hierarchy at the previous FMG stage, consumed), with that
    // stage's state and the new finest level p-linearly prolonged on every
    // slab's planes -- Hierarchy::unfold restricted to the slab ranges.
    static std::unique_ptr<SlabGroup> unfold_from(Hierarchy& coarse, int local, int devices);
    void time_cycles(const Policy& pol, int n0, int count, double* out4);
    void e2e_step(const Policy& pol, int n, const double* hostChi, double* out3, long long* h2dBytes);
    int owned_planes(int* z0, int* z1) const;  // of the first local slab

    struct State;

  private:
    std::unique_ptr<State> st_;
};

std::vector<std::array<int, 8>> slab_plan(int levels, int world, int resident = 4 * 148);
// co-resident blocks of the 3D fused fine pass on the current device (the chunking input of slab_plan)
int fused3_resident_blocks(int smCount);

// 128-byte NCCL unique id (dlopen'd libnccl); false if NCCL is unavailable.
bool nccl_unique_id(void* out128);

// Test hook: x / y elementwise on the device with the kernels' __divdc3
// restatement (per-element divisor constants); host buffers.
void test_divdc3(const double* x, const double* y, double* out, long long n);
// |x + iy| on the device as the host libm's hypot computes it (dynamic adaptivity's mark features)
void test_hypot(const double* x, const double* y, double* out, long long n);

}  // namespace tmg
