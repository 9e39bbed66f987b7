/* Extensions of the treemg C interface served by libtreemg_b200.so.
 *
 * 1. Run-result history accessor ("add an extension accessor
 *    without changing existing signatures") -- the per-sweep rows the
 *    reference only writes to <out>.csv (proj/src/runner.cpp:318-329).
 *
 * 2. The device-resident multilevel hierarchy: the drop-in for the C++ cycle
 *    API  td_add / td_bpx (proj/include/treemg/cycles.hpp:56-62,
 *    proj/src/cycles.cpp:336-354) acting on a Spacetree.  The spacetree's
 *    hash-per-level storage (proj/src/spacetree.cpp) is replaced by per-level
 *    lattice arrays in HBM; the handle owns them plus one CUDA stream.  Field
 *    import/export (full level lattice, axis 0 fastest, interleaved re/im
 *    doubles) lets the reference's cycle tests run against it.
 *
 * Extension configuration keys accepted by treemg_config_set (on top of the
 * reference's keys, runner.cpp:81-106):
 *   rhs = analytic | seeded     seeded: f = unit_rand complex, keyed on the
 *                               final-lattice position
 *   rhs_seed = <u64>            default 12345
 *   rhs_mask = none | sphere    f zero outside |x - 1/2|^2 < 0.04
 *   precision = exact | fast | fast-complex64
 *                               exact: bit-identical iterates to the reference
 *                               fast: FMA, correction-form coarse levels
 *                               fast-complex64: fast with the finest level stored
 *                               and computed in complex64 (2D / 3D; coarse levels and
 *                               norm sums complex128 / double)
 *   max_vertices = <n>          vertex cap (reference default 8388608)
 *   hb_sweeps = <k>             hierarchical-basis mask for sweeps 1..k, then off
 *   fmg_from = <level>          FMG unfolding from <level> up to `level` (fast-complex64: the
 *                               stages below `level` run in complex128)
 *   fmg_stage_cap = <n>         sweeps per FMG stage (default max_sweeps)
 *   sphere_levels = <k>         static adaptive tree (BASELINE cfg4): `level` regular,
 *                               then k levels refined where the parent cell's centre
 *                               lies in |x - 1/2|^2 < 0.04; hanging vertices; precision
 *                               exact (bit-identical) or fast (regular vertices' residual
 *                               as the assembled stencil), not fast-complex64
 *   norms = device | host       host (exact precision only): |r| downloaded and
 *                               summed on the host in the reference's traversal
 *                               order, so CSV/log bytes match the reference
 *   fingerprint = 0 | 1         hash the final fine u / sc (treemg_result_fingerprint)
 *   device = <ordinal>          CUDA device
 *   gpus = <n>                  n > 1: the finest level as n z-slabs over the GPUs
 *                               device .. device+n-1 of this process (3D, fast;
 *                               with fmg_from: at the last unfolding); bitwise
 *                               identical iterates to gpus = 1
 */

#ifndef TREEMG_B200_H
#define TREEMG_B200_H

#include "treemg.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- 1. history ---------------------------------------------------------- */
int treemg_result_history_rows(const treemg_result* res);
/* row i: sweep, workUnits, vertexCount, maxNorm, euclid, hNorm */
treemg_status treemg_result_history_row(const treemg_result* res, int i, double* out6);
/* wall time of the run's cycle loop in milliseconds */
double treemg_result_device_ms(const treemg_result* res);
/* FNV-1a of the final finest-level field ("u" or "sc") bit patterns; needs
 * config key fingerprint = 1, else 0; which = "u#<c>" reads channel c's u */
unsigned long long treemg_result_fingerprint(const treemg_result* res, const char* which);

/* ---- 2. device hierarchy ------------------------------------------------- */
typedef struct tmg_hierarchy tmg_hierarchy;

typedef struct tmg_problem {
    int dim;                       /* 1..3 */
    int levels;                    /* finest level L (regular grid, 3^L cells per axis) */
    int ell_min;                   /* coarsest smoothed level (spacetree.hpp Config::ellMin) */
    double theta;                  /* cell rotation, radians (ProblemSpec::thetaGlobal) */
    double phi_re, phi_im;         /* constant Helmholtz shift phi */
    int chi_kind;                  /* 0 zero, 1 sin product, 2 ball indicator, 3 seeded, 4 gaussian scenario
                                      (2D; cell-varying phi and absorbing-layer theta, problems.cpp:20-24,
                                      78-90; exact precision) */
    unsigned long long rhs_seed;
    int rhs_sphere;
    int precision;                 /* 0 exact, 1 fast, 2 fast-complex64 (2D / 3D: complex64 fine level) */
    long long max_vertices;        /* 0: reference default 8388608 */
    int device;                    /* CUDA device ordinal */
    int sphere_levels;             /* static adaptive tree: `levels` regular, then this many levels refined
                                      where the parent cell's centre lies in |x - 1/2|^2 < 0.04 (BASELINE cfg4;
                                      the cycle then runs the hanging-vertex events cycles.cpp:143-171, 305-321) */
    int channels;                  /* unknowns per vertex, 0 or 1: one (RunConfig::channels, runner.cpp:152;
                                      > 1 runs in exact precision on regular trees) */
    double coupling_re, coupling_im; /* A_ij for i != j, mass-weighted (runner.cpp:153-157, kernels.cpp:52-53) */
    double h_max, h_min;           /* both > 0: dynamic adaptivity (the runner's h_max / h_min, runner.cpp:206-366):
                                      `levels` is ignored, the tree starts regular at max(ell_min,
                                      level_for_h(h_max)) and tmg_mark after a sweep marks cells that the next
                                      sweep refines / erases; exact precision */
} tmg_problem;

typedef struct tmg_policy {        /* OmegaPolicy, proj/include/treemg/cycles.hpp:17-24 */
    int kind;                      /* 0 jacobi-only, 1 undamped, 2 lgrid, 3 exponential, 4 transition */
    double omega_re, omega_im;
    int lgrid;
    int hb;
    int bpx;
    int two_phase;
} tmg_policy;

typedef struct tmg_sweep_stats {   /* SweepStats, cycles.hpp:37-45 (channel 0) */
    double max_norm, euclid_norm, h_norm;
    long long updated_fine_vertices;
} tmg_sweep_stats;

treemg_status tmg_hierarchy_create(const tmg_problem* prob, tmg_hierarchy** out);
void tmg_hierarchy_destroy(tmg_hierarchy* h);

/* One cycle; n is the 1-based sweep counter (cycles.cpp:336-354). */
treemg_status tmg_td_add(tmg_hierarchy* h, const tmg_policy* pol, int n, tmg_sweep_stats* out);
treemg_status tmg_td_bpx(tmg_hierarchy* h, const tmg_policy* pol, int n, tmg_sweep_stats* out);
/* Per-channel norms of the last td_add / td_bpx sweep (SweepStats::maxNorm[c] etc.,
   cycles.hpp:27-31): writes min(channels, cap) entries of each non-null array and
   returns the channel count (0 for a one-channel hierarchy), -1 on a null handle. */
int tmg_channel_norms(tmg_hierarchy* h, double* max_norm, double* euclid, double* h_norm, int cap);
/* Dynamic adaptivity: mark (amr.cpp:61-222) on the device after a td_add / td_bpx.
 * out9: refinedCells, erasedCells of the last sweep, then MarkStats (amr.hpp:19-27)
 * refineVertices, eraseVertices, refineCells, eraseCells, vetoConvergence, vetoHMin, vetoHMax. */
treemg_status tmg_mark(tmg_hierarchy* h, long long* out9);
/* current depth of the tree (grows under dynamic adaptivity) */
int tmg_levels(const tmg_hierarchy* h);
/* overwrite the pending marks of every existing cell of `level` (full lattice,
 * lower corner: 4 refineMark, 8 eraseMark), e.g. to replay externally chosen marks */
treemg_status tmg_set_cell_marks(tmg_hierarchy* h, int level, const unsigned char* cells);
/* dynamic adaptivity: cumulative wall-clock ms of the host traversal replay, the sweep-table
 * upload, the device sweep, the final-classification upload and mark (all sweeps so far);
 * out6[5]: kernels launched */
treemg_status tmg_dyn_phase_ms(const tmg_hierarchy* h, double* out6);
/* adaptive trees: stored vertices, hanging ones included */
long long tmg_existing_vertices(const tmg_hierarchy* h);

/* Verification cycles of a regular tree held in exact storage (precision 0),
 * each followed by evaluate_residual_norms (cycles.cpp:716-786) into *out:
 * bu_fas(tree, spec, pol, n) (cycles.cpp:374-603) and
 * textbook_add(tree, spec, omegaS, omegaCG) (cycles.cpp:605-714).  The
 * reference sums these in hash-map order, so parity is a tolerance, not
 * bit-identity. */
treemg_status tmg_bu_fas(tmg_hierarchy* h, const tmg_policy* pol, int n, tmg_sweep_stats* out);
treemg_status tmg_textbook_add(tmg_hierarchy* h, double omega_s_re, double omega_s_im, double omega_cg_re,
                               double omega_cg_im, tmg_sweep_stats* out);
long long tmg_lattice_size(const tmg_hierarchy* h, int level);
/* field: u chi r rhat uhat diag sc sf si sinext; out: 2*lattice_size doubles */
treemg_status tmg_get_field(tmg_hierarchy* h, int level, const char* field, double* out);
treemg_status tmg_set_field(tmg_hierarchy* h, int level, const char* field, const double* in);
/* proj/tests/test_util.hpp:48-65 semantics: interior values of the finest
 * level (interior lattice order), injected upward, pipeline state reset */
treemg_status tmg_set_fine_interior_u(tmg_hierarchy* h, const double* u);
/* proj/src/cycles.cpp:812-840 */
treemg_status tmg_set_random_initial_guess(tmg_hierarchy* h, unsigned long long seed);
/* nodal right-hand side chi at the finest lattice (host buffer, 2*lattice
 * doubles); rebuilds the consistent-mass load vector on the device */
treemg_status tmg_set_fine_rhs(tmg_hierarchy* h, const double* chi_nodal);
/* FNV-1a over (re+0.0, im+0.0) bit patterns of a level field, lattice order */
unsigned long long tmg_field_hash(tmg_hierarchy* h, int level, const char* field);
/* adaptive trees: per lattice point of `level` the classification byte
 * (1 exists, 2 hanging, 4 refined, 8 boundary, 16 cPoint; spacetree.cpp:438-489),
 * succ (-1 absent) and per cell (lower corner) 1 exists | 2 refined; any
 * pointer may be NULL.  TREEMG_E_CONFIG on a regular tree. */
treemg_status tmg_get_flags(tmg_hierarchy* h, int level, unsigned char* flags, signed char* succ,
                            unsigned char* cells);
long long tmg_hanging_vertices(const tmg_hierarchy* h);
/* Host-only (no GPU): the static sphere tree's structure as tmg_get_flags
 * reports it, plus per vertex the corner index it has in the cell it is
 * touched last in (0xFF absent) -- the restriction-order table of amr.hpp. */
treemg_status tmg_sphere_tree(int dim, int base, int sphere_levels, int level, unsigned char* flags,
                              signed char* succ, unsigned char* cells, unsigned char* finish_corner);
/* Host-only (no GPU): the structural replay of dynamic adaptivity (dyn.hpp).
 * A tree built as build_regular(start) (spacetree.cpp:48-76); cell marks
 * (full-lattice, lower corner; 4 refineMark, 8 eraseMark) are applied by
 * tmg_dyn_sweep exactly as one td_add / td_bpx traversal with applyMarks does
 * (refine on descent cycles.cpp:174-180, erase on backtracking :222-241),
 * followed by classify().  out4: refinedCells, erasedCells, touch-last
 * updates of unrefined interior vertices, vertices with a special pattern. */
typedef struct tmg_dyn tmg_dyn;
treemg_status tmg_dyn_create(int dim, int start, int max_level, int ell_min, double h_min, long long max_vertices,
                             tmg_dyn** out);
void tmg_dyn_destroy(tmg_dyn* h);
int tmg_dyn_depth(const tmg_dyn* h);
long long tmg_dyn_interior_count(const tmg_dyn* h);
treemg_status tmg_dyn_set_cell_marks(tmg_dyn* h, int level, const unsigned char* cells);
treemg_status tmg_dyn_sweep(tmg_dyn* h, long long* out4);
/* flags: 1 exists | 2 hanging | 4 refined | 8 boundary | 16 cPoint; succ (-1 absent);
 * cells: 1 exists | 2 refined | 4 refineMark | 8 eraseMark (full lattices) */
treemg_status tmg_dyn_flags(tmg_dyn* h, int level, unsigned char* flags, signed char* succ, unsigned char* cells);
/* The per-vertex tables of the last sweep: role (dyn.hpp kS*), first finish
 * corner, finish / skipped cells as bit masks over cell = v - 1 + bits(e),
 * succ at the touch-last finish, and the cells visited (1) / refined on entry (2). */
treemg_status tmg_dyn_sweep_tables(tmg_dyn* h, int level, unsigned char* role, unsigned char* finish_corner,
                                   unsigned char* finish_cells, unsigned char* skip_cells, signed char* succ,
                                   unsigned char* cells);
/* Spacetree::interior_fine_vertex_count (spacetree.cpp:225-231): non-hanging,
 * non-refined, interior vertices over all levels */
long long tmg_leaf_vertices(const tmg_hierarchy* h);

/* Timing: runs `count` cycles starting at sweep counter n0 with CUDA events on
 * the hierarchy's stream; out[0] = total ms, out[1] = ms in the fine-level
 * residual kernel (average per cycle), out[2] = ms in the fine-level
 * correction kernel (average per cycle), out[3] = kernel launches per cycle. */
treemg_status tmg_time_cycles(tmg_hierarchy* h, const tmg_policy* pol, int n0, int count, int flush_l2,
                              double* out4);

/* e2e step through the boundary: host chi (pinned or pageable) -> device load
 * vector -> one cycle -> host norms.  out3 = max, euclid, h. */
treemg_status tmg_e2e_step(tmg_hierarchy* h, const tmg_policy* pol, int n, const double* chi_nodal,
                           double* out3);

const char* tmg_last_error(void);

/* ---- 3. z-slab multi-GPU cycle ---------------------------
 * The fine level and level L-1 are split into z-slabs (whole z-chunks of the
 * fused fine pass), coarser levels are replicated; halos, restriction
 * partials and the replicated level's residual move over NCCL (dlopen'd
 * libnccl.so.2), one slab per process/GPU.  With nccl_id == NULL, `local`
 * slabs run in this process with device-copy transfers: on one device (the
 * single-GPU test mode of the same code path), or with
 * tmg_slabs_create_local spread over `devices` GPUs with peer copies over
 * NVLink (what treemg_run's `gpus` key drives).  Each slab allocates only
 * its planes (+ halos) of levels L and L-1.  3D, fast precision; iterates
 * are bitwise identical for every slab count. */
typedef struct tmg_slabs tmg_slabs;
treemg_status tmg_nccl_unique_id(unsigned char* out128);
treemg_status tmg_slabs_create(const tmg_problem* prob, int local, int rank, int world,
                               const unsigned char* nccl_id, tmg_slabs** out);
treemg_status tmg_slabs_create_local(const tmg_problem* prob, int slabs, int devices, tmg_slabs** out);
void tmg_slabs_destroy(tmg_slabs* h);
/* whole-lattice u or sc of any level gathered from the slabs of this process
 * (bitwise what one GPU's tmg_get_field returns) */
treemg_status tmg_slabs_get_field(tmg_slabs* h, int level, const char* field, double* out);
treemg_status tmg_slabs_cycle(tmg_slabs* h, const tmg_policy* pol, int n, tmg_sweep_stats* out);
/* owned fine planes of the local slabs into a full-lattice host buffer */
treemg_status tmg_slabs_get_fine_u(tmg_slabs* h, double* out);
treemg_status tmg_slabs_time_cycles(tmg_slabs* h, const tmg_policy* pol, int n0, int count, double* out4);
int tmg_slabs_owned_planes(tmg_slabs* h, int* z0, int* z1);
/* e2e step: owned (+halo) planes of a full-lattice host rhs -> device load
 * vector -> one cycle -> host norms (out3); *h2d_bytes = bytes uploaded */
treemg_status tmg_slabs_e2e_step(tmg_slabs* h, const tmg_policy* pol, int n, const double* chi, double* out3,
                                 long long* h2d_bytes);
/* host-only slab plan: per slab {cb, ce, z0, z1, Zs, Ze, Ws, We} (fused
 * z-chunks, fine planes, level L-1 planes, level L-2 planes); out: 8*world */
treemg_status tmg_slab_plan(int levels, int world, int* out8);

/* Test hook: out = x / y elementwise (interleaved complex, host buffers) on
 * the device with the kernels' restatement of libgcc __divdc3. */
treemg_status tmg_test_divdc3(const double* x, const double* y, double* out, long long n);
/* Test hook: the device's restatement of the host libm hypot (glibc, Borges' algorithm with
 * the non-FMA correction) that the dynamic-adaptivity features use for std::abs(complex). */
treemg_status tmg_test_hypot(const double* x, const double* y, double* out, long long n);

#ifdef __cplusplus
}
#endif

#endif /* TREEMG_B200_H */
