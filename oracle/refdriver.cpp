// Oracle harness around the UNMODIFIED reference library (built by
// oracle/Makefile from /root/reference/proj/src into oracle/_ref/).
//
// TEST INFRASTRUCTURE ONLY. Nothing in the product links or loads this file;
// only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg do.
//
// What it adds on top of the reference's public C++ API, and nothing else:
//   * the seeded complex right-hand side of BASELINE.json:
//     accumulate_cell_rhs below restates proj/src/kernels.cpp:69-87 with a
//     complex chi; for every non-seeded problem it forwards to the reference
//     function itself (renamed at compile time, see oracle/Makefile), so the
//     reference's own problems run the reference code bit-for-bit;
//   * the runner's sweep loop (proj/src/runner.cpp:206-381) restated so the
//     BASELINE configurations the reference cannot express through run()
//     become runnable: raised vertex cap (cfg3), static sphere refinement
//     through Spacetree::refine_cell (cfg4), hb-then-additive schedule (cfg4),
//     FMG unfolding through whole-level refine_cell + classify() (cfg5);
//   * per-sweep std::chrono timing of td_add/td_bpx (the CPU baseline);
//   * field dumps and bit-pattern hashes of the tree state for parity tests.
// The reference's own C-ABI (proj/src/capi.cpp) is also exported from the
// same shared object, unmodified, for byte-identical CSV comparisons.

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "treemg/amr.hpp"
#include "treemg/cycles.hpp"
#include "treemg/elemops.hpp"
#include "treemg/kernels.hpp"
#include "treemg/problems.hpp"
#include "treemg/runner.hpp"
#include "treemg/spacetree.hpp"
#include "treemg/transfer.hpp"

namespace treemg {
// The reference definition from proj/src/kernels.cpp:69-87 (renamed by the
// Makefile so that the harness can supply accumulate_cell_rhs itself).
void accumulate_cell_rhs_reference(const CellKernel& k, const ProblemSpec& spec, int level,
                                   const Index& cellIndex, std::span<Cplx> dB);
}  // namespace treemg

namespace {

using namespace treemg;

struct SeededRhs {
    bool on = false;
    std::uint64_t seed = 12345;
    int lmax = 0;        // lattice the seed is keyed on (final level)
    bool sphere = false; // f masked to |x - 1/2|^2 < 0.04
};

SeededRhs g_rhs;

// splitmix64 finaliser -> uniform [-1,1); restates proj/src/cycles.cpp:802-808.
double unit_rand(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    x = x ^ (x >> 31);
    return 2.0 * static_cast<double>(x >> 11) / 9007199254740992.0 - 1.0;
}

// |x - 1/2|^2 < 0.04 for x = idx / m, evaluated exactly in integers:
// sum_d (2 idx_d - m)^2 / (4 m^2) < 1/25.
bool vertex_in_sphere(int p, std::int64_t m, const Index& idx) {
    std::int64_t s = 0;
    for (int d = 0; d < p; ++d) {
        const std::int64_t t = 2 * static_cast<std::int64_t>(idx[d]) - m;
        s += t * t;
    }
    return 25 * s < 4 * m * m;
}

// Cell centre (idx + 1/2) / m inside the same ball.
bool cell_centre_in_sphere(int p, std::int64_t m, const Index& idx) {
    std::int64_t s = 0;
    for (int d = 0; d < p; ++d) {
        const std::int64_t t = 2 * static_cast<std::int64_t>(idx[d]) + 1 - m;
        s += t * t;
    }
    return 25 * s < 4 * m * m;
}

// Seeded nodal field, keyed on the final-lattice position.
Cplx seeded_f(int p, int level, const Index& v, int c) {
    Index fi = zero_index();
    const int scale = pow3(g_rhs.lmax - level);
    for (int d = 0; d < p; ++d) fi[d] = v[d] * scale;
    if (g_rhs.sphere && !vertex_in_sphere(p, pow3(g_rhs.lmax), fi)) return Cplx(0.0);
    const std::uint64_t s = g_rhs.seed ^ (static_cast<std::uint64_t>(c) << 48) ^ pack_index(p, fi);
    return Cplx(unit_rand(s), unit_rand(s ^ 0x5bf03635ull));
}

}  // namespace

namespace treemg {

// proj/src/kernels.cpp:69-87 with a complex chi (the SURVEY §8c extension).
// For real chi, double*Cplx(chi,0) reproduces the real-only accumulation
// bit-for-bit, but non-seeded problems do not even get here: they run the
// reference function itself.
void accumulate_cell_rhs(const CellKernel& k, const ProblemSpec& spec, int level,
                         const Index& cellIndex, std::span<Cplx> dB) {
    if (!g_rhs.on) {
        accumulate_cell_rhs_reference(k, spec, level, cellIndex, dB);
        return;
    }
    const int n = k.ref->n;
    const int nc = k.channels;
    Cplx chiCorner[1 << kMaxDim];
    for (int c = 0; c < nc; ++c) {
        for (int b = 0; b < n; ++b) {
            Index x = cellIndex;
            for (int d = 0; d < spec.dim; ++d) x[d] += (b >> d) & 1;
            chiCorner[b] = seeded_f(spec.dim, level, x, c);
        }
        for (int a = 0; a < n; ++a) {
            Cplx acc(0.0);
            for (int b = 0; b < n; ++b) acc += k.ref->mas(a, b) * chiCorner[b];
            dB[a * nc + c] += k.massScale * acc;
        }
    }
}

}  // namespace treemg

namespace {

std::string trim(const std::string& s) {
    std::size_t a = s.find_first_not_of(" \t\r\n");
    if (a == std::string::npos) return "";
    std::size_t b = s.find_last_not_of(" \t\r\n");
    return s.substr(a, b - a + 1);
}

struct Row {
    int sweep = 0;
    double workUnits = 0.0;
    std::size_t vertexCount = 0;
    double maxNorm = 0.0, euclid = 0.0, hNorm = 0.0;
    std::vector<double> chMax, chEuclid, chH;
};

struct Session {
    RunConfig cfg;
    ProblemSpec spec;
    OmegaPolicy pol;
    std::unique_ptr<Spacetree> tree;
    SeededRhs rhs;
    std::size_t maxVertices = 8u * 1024u * 1024u;
    int sphereLevels = 0;
    int hbSweeps = -1;
    int fmgFrom = 0;
    int fmgStageCap = 0;
    bool checkLemma1 = false;
    int finalLevel = 0;
    // dynamic adaptivity (h_max / h_min, runner.cpp:206-366): marks after every sweep
    bool adaptive = false;
    AmrConfig amr;
    MarkStats lastMark;
    int lastRefined = 0, lastErased = 0;

    // run results
    int status = 0;  // 0 ok, 1 usage, 2 capacity, 3 runtime
    std::string message;
    int outcome = 1;  // 0 converged, 1 budget exhausted, 2 diverged
    int sweeps = 0;
    double firstNorm = 0.0, finalNorm = 0.0, workUnits = 0.0;
    std::size_t vertexCount = 0;
    std::vector<Row> history;
    std::vector<double> sweepSeconds;
    std::vector<int> sweepLevel;
    std::string csv, log;
    SweepStats last;
};

double aggregate_max(const std::vector<double>& v) {
    double m = 0.0;
    for (double x : v) m = std::max(m, x);
    return m;
}
double aggregate_l2(const std::vector<double>& v) {
    double s = 0.0;
    for (double x : v) s += x * x;
    return std::sqrt(s);
}

Cplx default_omega(const RunConfig& cfg) {  // proj/src/runner.cpp:176-179
    if (cfg.omegaS) return *cfg.omegaS;
    return cfg.problem == "gaussian" ? Cplx(0.4, 0.0) : Cplx(0.8, 0.0);
}

void refine_all_leaves(Spacetree& tree, int level, bool sphereOnly) {
    std::vector<Key> keys;
    const int p = tree.dim();
    tree.for_each_cell_at(level, [&](const Index& idx, Cell& c) {
        if (c.refined) return;
        if (sphereOnly && !cell_centre_in_sphere(p, pow3(level), idx)) return;
        keys.push_back(pack_index(p, idx));
    });
    std::sort(keys.begin(), keys.end());
    for (Key k : keys) tree.refine_cell(level, unpack_index(p, k));
}

void setup(Session& s, const std::string& text) {
    std::istringstream in(text);
    std::string line;
    while (std::getline(in, line)) {
        const std::size_t hash = line.find('#');
        if (hash != std::string::npos) line = line.substr(0, hash);
        line = trim(line);
        if (line.empty()) continue;
        const std::size_t eq = line.find('=');
        if (eq == std::string::npos) throw ConfigError("malformed config line: " + line);
        const std::string key = trim(line.substr(0, eq)), value = trim(line.substr(eq + 1));
        if (key == "rhs") s.rhs.on = (value == "seeded");
        else if (key == "rhs_seed") s.rhs.seed = std::stoull(value);
        else if (key == "rhs_mask") s.rhs.sphere = (value == "sphere");
        else if (key == "max_vertices") s.maxVertices = std::stoull(value);
        else if (key == "sphere_levels") s.sphereLevels = std::stoi(value);
        else if (key == "hb_sweeps") s.hbSweeps = std::stoi(value);
        else if (key == "fmg_from") s.fmgFrom = std::stoi(value);
        else if (key == "fmg_stage_cap") s.fmgStageCap = std::stoi(value);
        else if (key == "check_lemma1") s.checkLemma1 = (value == "1");
        else if (key == "precision" || key == "gpus") {}  // GPU-side keys, no CPU meaning
        else apply_override(s.cfg, key, value);
    }
    s.cfg.validate();
    s.spec = problem_of(s.cfg);
    s.adaptive = s.cfg.fixedLevel == 0;
    if (s.adaptive && (s.sphereLevels > 0 || s.fmgFrom > 0))
        throw UnsupportedConfigError("oracle driver: h_max/h_min runs take no sphere_levels / fmg_from");
    s.finalLevel = s.adaptive ? reference_level_of(s.cfg) : s.cfg.fixedLevel + s.sphereLevels;
    const int start = s.adaptive ? start_level_of(s.cfg) : s.fmgFrom > 0 ? s.fmgFrom : s.cfg.fixedLevel;
    s.amr.hMax = s.cfg.hMax;  // runner.cpp:228-230
    s.amr.hMin = s.cfg.hMin;
    s.rhs.lmax = s.finalLevel;
    g_rhs = s.rhs;
    Spacetree::Config tcfg;
    tcfg.dim = s.cfg.dim;
    tcfg.channels = s.cfg.channels;
    tcfg.ellMin = s.cfg.ellMin;
    tcfg.maxVertices = s.maxVertices;
    s.tree = std::make_unique<Spacetree>(Spacetree::build_regular(s.cfg.dim, start, tcfg));
    const ProblemSpec* sp = &s.spec;
    s.tree->set_theta_assigner([sp](int level, const Index& idx) { return cell_theta(*sp, level, idx); });
    for (int k = 0; k < s.sphereLevels; ++k) refine_all_leaves(*s.tree, s.cfg.fixedLevel + k, true);
    if (s.sphereLevels > 0) {
        s.tree->classify();
        s.tree->clear_structure_dirty();
    }
    if (s.cfg.randomInitialGuess) set_random_initial_guess(*s.tree, s.cfg.seed);
    s.pol.kind = s.cfg.omegaKind;
    s.pol.omegaS = default_omega(s.cfg);
    s.pol.lGrid = s.cfg.lGrid;
    s.pol.hbMask = s.cfg.hbMask;
    s.pol.twoPhase = s.cfg.twoPhase;
}

SweepStats one_sweep(Session& s, int n) {
    g_rhs = s.rhs;
    OmegaPolicy pol = s.pol;
    if (s.hbSweeps >= 0) pol.hbMask = n <= s.hbSweeps;
    SweepOptions opt;
    opt.checkLemma1 = s.checkLemma1;
    opt.applyMarks = s.adaptive;  // runner.cpp:256-258
    opt.hMinRefine = s.cfg.hMin;
    switch (s.cfg.cycle) {
        case CycleKind::TdAdd: return td_add(*s.tree, s.spec, pol, n, opt);
        case CycleKind::TdBPX: return td_bpx(*s.tree, s.spec, pol, n, opt);
        case CycleKind::BuFAS:
            bu_fas(*s.tree, s.spec, pol, n);
            return evaluate_residual_norms(*s.tree, s.spec);
        case CycleKind::TextbookAdd: {
            const Cplx wcg = s.cfg.omegaCG != 0.0 ? Cplx(s.cfg.omegaCG, 0.0) : pol.omegaS;
            textbook_add(*s.tree, s.spec, pol.omegaS, wcg);
            return evaluate_residual_norms(*s.tree, s.spec);
        }
    }
    return {};
}

// The sweep loop of proj/src/runner.cpp:259-366, plus FMG stages.
void run_loop(Session& s) {
    const RunConfig& cfg = s.cfg;
    double referenceCost = 1.0;
    {
        double n = 1.0;
        for (int d = 0; d < cfg.dim; ++d) n *= static_cast<double>(pow3(s.finalLevel) - 1);
        referenceCost = std::max(1.0, n);
    }
    char buf[256];
    std::ostringstream csv, log;
    csv << "sweep,workUnits,vertexCount,maxNorm,euclid,hNorm";
    if (cfg.channels > 1)
        for (int c = 0; c < cfg.channels; ++c) csv << ",maxNorm" << c << ",euclid" << c << ",hNorm" << c;
    csv << "\n";
    double cumulativeUpdates = 0.0, minNorm = 0.0, stageFirst = 0.0;
    bool haveMin = false;
    int stageSweep = 0;
    const int stageCap = s.fmgStageCap > 0 ? s.fmgStageCap : cfg.maxSweeps;
    const bool fmg = s.fmgFrom > 0 && s.fmgFrom < cfg.fixedLevel;
    int n = 0;
    for (;;) {
        ++n;
        ++stageSweep;
        SweepStats stats;
        std::string failure;
        const auto t0 = std::chrono::steady_clock::now();
        try {
            stats = one_sweep(s, n);
        } catch (const SingularDiagonalError& e) {
            failure = e.what();
        }
        const auto t1 = std::chrono::steady_clock::now();
        s.sweepSeconds.push_back(std::chrono::duration<double>(t1 - t0).count());
        s.sweepLevel.push_back(s.tree->depth());
        s.sweeps = n;
        if (!failure.empty()) {
            s.outcome = 2;
            s.message = failure;
            log << "sweep " << n << ": " << failure << "\n";
            break;
        }
        cumulativeUpdates += static_cast<double>(stats.updatedFineVertices);
        Row rec;
        rec.sweep = n;
        rec.workUnits = cumulativeUpdates / referenceCost;
        rec.vertexCount = s.tree->interior_fine_vertex_count();
        rec.maxNorm = aggregate_max(stats.maxNorm);
        rec.euclid = aggregate_l2(stats.euclidNorm);
        rec.hNorm = aggregate_l2(stats.hNorm);
        rec.chMax = stats.maxNorm;
        rec.chEuclid = stats.euclidNorm;
        rec.chH = stats.hNorm;
        const double current = cfg.norm == NormKind::Max      ? rec.maxNorm
                               : cfg.norm == NormKind::Euclid ? rec.euclid
                                                              : rec.hNorm;
        if (n == 1) s.firstNorm = current;
        if (stageSweep == 1) stageFirst = current;
        s.finalNorm = current;
        s.workUnits = rec.workUnits;
        s.vertexCount = rec.vertexCount;
        std::snprintf(buf, sizeof buf, "%d,%.17g,%zu,%.17g,%.17g,%.17g", n, rec.workUnits, rec.vertexCount,
                      rec.maxNorm, rec.euclid, rec.hNorm);
        csv << buf;
        if (cfg.channels > 1)
            for (int c = 0; c < cfg.channels; ++c) {
                std::snprintf(buf, sizeof buf, ",%.17g,%.17g,%.17g", rec.chMax[c], rec.chEuclid[c], rec.chH[c]);
                csv << buf;
            }
        csv << "\n";
        s.last = stats;
        s.history.push_back(rec);
        if (!std::isfinite(current)) {
            s.outcome = 2;
            s.message = "non-finite residual";
            break;
        }
        if (!haveMin || current < minNorm) {
            minNorm = current;
            haveMin = true;
        }
        if (current > minNorm * 1e6 && stageSweep > 1) {
            s.outcome = 2;
            s.message = "residual grew six orders over its minimum";
            break;
        }
        const bool converged = stageFirst < 1e-300 || current <= cfg.targetResidualDrop * stageFirst;
        if (s.adaptive) {  // runner.cpp:350-358
            s.lastMark = mark(*s.tree, s.amr);
            const MarkStats& m = s.lastMark;
            log << "sweep " << n << ": refined=" << stats.refinedCells << " erased=" << stats.erasedCells
                << " marks(refine=" << m.refineCells << ", erase=" << m.eraseCells << ", veto_conv=" << m.vetoConvergence
                << ", veto_hmin=" << m.vetoHMin << ", veto_hmax=" << m.vetoHMax << ")\n";
        }
        const bool lastStage = !fmg || s.tree->depth() >= cfg.fixedLevel;
        if (lastStage) {
            if (converged) {
                s.outcome = 0;
                break;
            }
            if (stageSweep >= stageCap) {
                s.outcome = 1;
                break;
            }
        } else if (converged || stageSweep >= stageCap) {
            log << "unfold after sweep " << n << " to level " << s.tree->depth() + 1 << "\n";
            refine_all_leaves(*s.tree, s.tree->depth(), false);
            s.tree->classify();
            s.tree->clear_structure_dirty();
            stageSweep = 0;
            haveMin = false;
        }
    }
    const char* name = s.outcome == 0 ? "converged" : s.outcome == 2 ? "diverged" : "budget-exhausted";
    log << "status=" << name << " sweeps=" << s.sweeps << " workUnits=" << s.workUnits
        << " vertices=" << s.vertexCount << " firstNorm=" << s.firstNorm << " finalNorm=" << s.finalNorm << "\n";
    s.csv = csv.str();
    s.log = log.str();
}

template <class Fn>
int guarded(Session* s, Fn&& fn) {
    try {
        fn();
        s->status = 0;
    } catch (const ConfigError& e) {
        s->status = 1;
        s->message = e.what();
    } catch (const UnsupportedConfigError& e) {
        s->status = 1;
        s->message = e.what();
    } catch (const CapacityError& e) {
        s->status = 2;
        s->message = e.what();
    } catch (const std::exception& e) {
        s->status = 3;
        s->message = e.what();
    }
    return s->status;
}

Cplx field_of(const ChannelState& ch, const char* f) {
    if (!std::strcmp(f, "u")) return ch.u;
    if (!std::strcmp(f, "chi")) return ch.chi;
    if (!std::strcmp(f, "r")) return ch.r;
    if (!std::strcmp(f, "rhat")) return ch.rHat;
    if (!std::strcmp(f, "uhat")) return ch.uHat;
    if (!std::strcmp(f, "diag")) return ch.diag;
    if (!std::strcmp(f, "sc")) return ch.sc;
    if (!std::strcmp(f, "sf")) return ch.sf;
    if (!std::strcmp(f, "si")) return ch.si;
    if (!std::strcmp(f, "sinext")) return ch.siNext;
    if (!std::strcmp(f, "s")) return Cplx(ch.s, 0.0);
    return Cplx(std::nan(""), std::nan(""));
}

std::size_t lattice_size(int p, int level) {
    std::size_t n = 1;
    for (int d = 0; d < p; ++d) n *= static_cast<std::size_t>(pow3(level) + 1);
    return n;
}

std::size_t lattice_flat(int p, int level, const Index& idx) {
    const std::size_t m = static_cast<std::size_t>(pow3(level) + 1);
    std::size_t flat = 0, stride = 1;
    for (int d = 0; d < p; ++d) {
        flat += static_cast<std::size_t>(idx[d]) * stride;
        stride *= m;
    }
    return flat;
}

}  // namespace

extern "C" {

void* refd_new(const char* text) {
    auto* s = new Session();
    guarded(s, [&] { setup(*s, text ? text : ""); });
    return s;
}

void refd_free(void* h) { delete static_cast<Session*>(h); }
int refd_status(void* h) { return static_cast<Session*>(h)->status; }
const char* refd_message(void* h) { return static_cast<Session*>(h)->message.c_str(); }
int refd_depth(void* h) { return static_cast<Session*>(h)->tree ? static_cast<Session*>(h)->tree->depth() : -1; }

int refd_run(void* h) {
    auto* s = static_cast<Session*>(h);
    if (s->status != 0) return s->status;
    return guarded(s, [&] { run_loop(*s); });
}

int refd_outcome(void* h) { return static_cast<Session*>(h)->outcome; }
int refd_sweeps(void* h) { return static_cast<Session*>(h)->sweeps; }
double refd_first_norm(void* h) { return static_cast<Session*>(h)->firstNorm; }
double refd_final_norm(void* h) { return static_cast<Session*>(h)->finalNorm; }
const char* refd_csv(void* h) { return static_cast<Session*>(h)->csv.c_str(); }
const char* refd_log(void* h) { return static_cast<Session*>(h)->log.c_str(); }
int refd_history_rows(void* h) { return static_cast<int>(static_cast<Session*>(h)->history.size()); }

// Row i: sweep, workUnits, vertexCount, maxNorm, euclid, hNorm.
void refd_history_row(void* h, int i, double* out) {
    const Row& r = static_cast<Session*>(h)->history.at(static_cast<std::size_t>(i));
    out[0] = r.sweep;
    out[1] = r.workUnits;
    out[2] = static_cast<double>(r.vertexCount);
    out[3] = r.maxNorm;
    out[4] = r.euclid;
    out[5] = r.hNorm;
}

int refd_timed_sweeps(void* h) { return static_cast<int>(static_cast<Session*>(h)->sweepSeconds.size()); }
double refd_sweep_seconds(void* h, int i) { return static_cast<Session*>(h)->sweepSeconds.at(static_cast<std::size_t>(i)); }

// One cycle with the session's policy; out: max, euclid, h (aggregated),
// updatedFineVertices, lemma1MaxError.
int refd_sweep(void* h, int n, double* out) {
    auto* s = static_cast<Session*>(h);
    if (s->status != 0) return s->status;
    return guarded(s, [&] {
        const auto t0 = std::chrono::steady_clock::now();
        const SweepStats st = one_sweep(*s, n);
        const auto t1 = std::chrono::steady_clock::now();
        s->sweepSeconds.push_back(std::chrono::duration<double>(t1 - t0).count());
        if (out) {
            out[0] = aggregate_max(st.maxNorm);
            out[1] = aggregate_l2(st.euclidNorm);
            out[2] = aggregate_l2(st.hNorm);
            out[3] = static_cast<double>(st.updatedFineVertices);
            out[4] = st.lemma1MaxError;
        }
        if (s->adaptive) {
            s->lastRefined = st.refinedCells;
            s->lastErased = st.erasedCells;
            s->lastMark = mark(*s->tree, s->amr);
        }
    });
}

long long refd_lattice_size(void* h, int level) {
    auto* s = static_cast<Session*>(h);
    return static_cast<long long>(lattice_size(s->tree->dim(), level));
}

// Full-lattice dump (axis 0 fastest, (3^l+1)^p entries, interleaved re/im);
// absent or hanging vertices read 0 and get mask 0.
void refd_field(void* h, int level, const char* field, int channel, double* out, unsigned char* mask) {
    auto* s = static_cast<Session*>(h);
    const int p = s->tree->dim();
    const std::size_t n = lattice_size(p, level);
    std::fill(out, out + 2 * n, 0.0);
    if (mask) std::fill(mask, mask + n, 0);
    s->tree->for_each_vertex_at(level, [&](const Index& idx, Vertex& v) {
        if (v.hanging) return;
        const std::size_t f = lattice_flat(p, level, idx);
        const Cplx z = field_of(v.ch[channel], field);
        out[2 * f] = z.real();
        out[2 * f + 1] = z.imag();
        if (mask) mask[f] = 1;
    });
}

// As refd_field, hanging vertices included: mask 1 = regular, 2 = hanging.
void refd_field_all(void* h, int level, const char* field, int channel, double* out, unsigned char* mask) {
    auto* s = static_cast<Session*>(h);
    const int p = s->tree->dim();
    const std::size_t n = lattice_size(p, level);
    std::fill(out, out + 2 * n, 0.0);
    std::fill(mask, mask + n, 0);
    s->tree->for_each_vertex_at(level, [&](const Index& idx, Vertex& v) {
        const std::size_t f = lattice_flat(p, level, idx);
        const Cplx z = field_of(v.ch[channel], field);
        out[2 * f] = z.real();
        out[2 * f + 1] = z.imag();
        mask[f] = v.hanging ? 2 : 1;
    });
}

// Classification per lattice point (1 exists, 2 hanging, 4 refined,
// 8 boundary, 16 cPoint), succ (-1 absent) and per cell (lower corner)
// 1 exists | 2 refined -- the encoding of tmg_get_flags.
void refd_flags(void* h, int level, unsigned char* flags, signed char* succ, unsigned char* cells) {
    auto* s = static_cast<Session*>(h);
    const int p = s->tree->dim();
    const std::size_t n = lattice_size(p, level);
    std::fill(flags, flags + n, 0);
    std::fill(succ, succ + n, static_cast<signed char>(-1));
    std::fill(cells, cells + n, 0);
    s->tree->for_each_vertex_at(level, [&](const Index& idx, Vertex& v) {
        const std::size_t f = lattice_flat(p, level, idx);
        flags[f] = static_cast<unsigned char>(1 | (v.hanging ? 2 : 0) | (v.refined ? 4 : 0) |
                                              (v.onBoundary ? 8 : 0) | (v.cPoint ? 16 : 0));
        succ[f] = static_cast<signed char>(v.succ);
    });
    s->tree->for_each_cell_at(level, [&](const Index& idx, Cell& c) {
        cells[lattice_flat(p, level, idx)] = static_cast<unsigned char>(1 | (c.refined ? 2 : 0));
    });
}

long long refd_interior_count(void* h) {
    return static_cast<long long>(static_cast<Session*>(h)->tree->interior_fine_vertex_count());
}

// Mirrors proj/tests/test_util.hpp:48-65 (set_fine_interior_u): interior
// lattice order of the finest level, re-injected upward, pipeline reset.
void refd_set_fine_interior_u(void* h, const double* u) {
    auto* s = static_cast<Session*>(h);
    Spacetree& tree = *s->tree;
    const int p = tree.dim();
    const int L = tree.depth();
    const int m = pow3(L) - 1;
    tree.for_each_vertex_at(L, [&](const Index& idx, Vertex& v) {
        if (v.onBoundary || v.hanging) return;
        std::size_t flat = 0, stride = 1;
        for (int d = 0; d < p; ++d) {
            flat += static_cast<std::size_t>(idx[d] - 1) * stride;
            stride *= static_cast<std::size_t>(m);
        }
        v.ch[0].u = Cplx(u[2 * flat], u[2 * flat + 1]);
    });
    for (int l = L - 1; l >= 0; --l) {
        tree.for_each_vertex_at(l, [&](const Index& idx, Vertex& v) {
            if (v.onBoundary || v.hanging || !v.refined) return;
            Index fi = idx;
            for (int d = 0; d < p; ++d) fi[d] *= 3;
            const Vertex* fv = tree.find_vertex(l + 1, fi);
            if (fv) v.ch[0].u = fv->ch[0].u;
        });
    }
    reset_pipeline_state(tree);
}

// FNV-1a over the bit patterns of (re + 0.0, im + 0.0) of a level field in
// lattice order (the +0.0 folds -0 into +0).
unsigned long long refd_field_hash(void* h, int level, const char* field, int channel) {
    auto* s = static_cast<Session*>(h);
    const int p = s->tree->dim();
    const std::size_t n = lattice_size(p, level);
    std::vector<double> buf(2 * n);
    refd_field(h, level, field, channel, buf.data(), nullptr);
    std::uint64_t hsh = 1469598103934665603ull;
    for (double x : buf) {
        const double y = x + 0.0;
        std::uint64_t bits;
        std::memcpy(&bits, &y, 8);
        for (int b = 0; b < 8; ++b) {
            hsh ^= (bits >> (8 * b)) & 0xffu;
            hsh *= 1099511628211ull;
        }
    }
    return hsh;
}

// Dynamic adaptivity: refinedCells, erasedCells of the last refd_sweep and the
// MarkStats of the mark() that followed it (amr.hpp:19-27).
void refd_mark_stats(void* h, long long* out9) {
    auto* s = static_cast<Session*>(h);
    const MarkStats& m = s->lastMark;
    const long long v[9] = {s->lastRefined, s->lastErased,
                            static_cast<long long>(m.refineVertices), static_cast<long long>(m.eraseVertices),
                            static_cast<long long>(m.refineCells), static_cast<long long>(m.eraseCells),
                            static_cast<long long>(m.vetoConvergence), static_cast<long long>(m.vetoHMin),
                            static_cast<long long>(m.vetoHMax)};
    std::copy(v, v + 9, out9);
}

// Per cell (lower corner, full lattice): 1 exists | 2 refined | 4 refineMark | 8 eraseMark.
void refd_cell_marks(void* h, int level, unsigned char* cells) {
    auto* s = static_cast<Session*>(h);
    const int p = s->tree->dim();
    std::fill(cells, cells + lattice_size(p, level), 0);
    if (level > s->tree->depth()) return;
    s->tree->for_each_cell_at(level, [&](const Index& idx, Cell& c) {
        cells[lattice_flat(p, level, idx)] = static_cast<unsigned char>(1 | (c.refined ? 2 : 0) |
                                                                        (c.refineMark ? 4 : 0) | (c.eraseMark ? 8 : 0));
    });
}

// Overwrites the pending marks of every existing cell (4 refineMark, 8 eraseMark).
void refd_set_cell_marks(void* h, int level, const unsigned char* cells) {
    auto* s = static_cast<Session*>(h);
    const int p = s->tree->dim();
    s->tree->for_each_cell_at(level, [&](const Index& idx, Cell& c) {
        const unsigned char m = cells[lattice_flat(p, level, idx)];
        c.refineMark = (m & 4) != 0;
        c.eraseMark = (m & 8) != 0;
    });
}

// Regular-grid classification summary used to pin the per-level omega tables.
int refd_vertex_succ(void* h, int level, const int* idx) {
    auto* s = static_cast<Session*>(h);
    Index i = zero_index();
    for (int d = 0; d < s->tree->dim(); ++d) i[d] = idx[d];
    const Vertex* v = s->tree->find_vertex(level, i);
    return v ? v->succ : -1;
}

// omega_unmasked / omega_of straight from the reference (cycles.cpp:17-36).
void refd_omega(int kind, double wr, double wi, int lgrid, int hb, int bpx, int twoPhase, int succ, int cpoint,
                int n, int masked, double* out) {
    OmegaPolicy pol;
    pol.kind = static_cast<OmegaKind>(kind);
    pol.omegaS = Cplx(wr, wi);
    pol.lGrid = lgrid;
    pol.hbMask = hb != 0;
    pol.bpx = bpx != 0;
    pol.twoPhase = twoPhase != 0;
    const Cplx w = masked ? omega_of(pol, succ, cpoint != 0, n) : omega_unmasked(pol, succ, n);
    out[0] = w.real();
    out[1] = w.imag();
}

}  // extern "C"
