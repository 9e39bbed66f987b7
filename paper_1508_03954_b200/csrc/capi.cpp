// The treemg C-ABI (include/treemg.h) plus the B200 extensions
// (include/treemg_b200.h).  Mirrors proj/src/capi.cpp: opaque handles,
// thread-local last error, exception -> status mapping; exceptions never
// cross the boundary.

#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <string>

#include "../../include/treemg.h"
#include "../../include/treemg_b200.h"
#include "amr.hpp"
#include "dyn.hpp"
#include "runner.hpp"

using namespace tmg;

struct treemg_config {
    RunConfig cfg;
};

struct treemg_result {
    RunResult res;
    int channels = 1;
};

struct tmg_hierarchy {
    std::unique_ptr<Hierarchy> h;
    int device = 0;
    SweepStats last;  // per-channel norms of the last sweep (tmg_channel_norms)
};

struct tmg_slabs {
    std::unique_ptr<SlabGroup> g;
    int device = 0;
};

namespace {

thread_local std::string g_lastError;


treemg_status fail(treemg_status code, const char* what) {
    g_lastError = what ? what : "unknown error";
    return code;
}

template <class Fn>
treemg_status guarded(Fn&& fn) {  // capi.cpp:28-43
    try {
        fn();
        g_lastError.clear();
        return TREEMG_OK;
    } catch (const ConfigError& e) {
        return fail(TREEMG_E_USAGE, e.what());
    } catch (const UnsupportedConfigError& e) {
        return fail(TREEMG_E_USAGE, e.what());
    } catch (const CapacityError& e) {
        return fail(TREEMG_E_CAPACITY, e.what());
    } catch (const std::exception& e) {
        return fail(TREEMG_E_RUNTIME, e.what());
    }
}

Policy policy_from(const tmg_policy* p) {
    Policy pol;
    pol.kind = static_cast<OmegaKind>(p->kind);
    pol.omegaS = Cplx(p->omega_re, p->omega_im);
    pol.lGrid = p->lgrid;
    pol.hbMask = p->hb != 0;
    pol.bpx = p->bpx != 0;
    pol.twoPhase = p->two_phase != 0;
    return pol;
}

void fill_stats(const SweepStats& st, tmg_sweep_stats* out) {
    if (!out) return;
    out->max_norm = st.maxNorm;
    out->euclid_norm = st.euclidNorm;
    out->h_norm = st.hNorm;
    out->updated_fine_vertices = st.updatedFineVertices;
}

}  // namespace

extern "C" {

unsigned treemg_version(void) { return 100; }

const char* treemg_last_error(void) { return g_lastError.c_str(); }

const char* tmg_last_error(void) { return g_lastError.c_str(); }

treemg_config* treemg_config_new(void) { return new treemg_config(); }

void treemg_config_free(treemg_config* cfg) { delete cfg; }

treemg_status treemg_config_load_file(treemg_config* cfg, const char* path) {
    if (!cfg || !path) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] { cfg->cfg = parse_config_file(path); });
}

treemg_status treemg_config_set(treemg_config* cfg, const char* key, const char* value) {
    if (!cfg || !key || !value) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] { apply_override(cfg->cfg, key, value); });
}

treemg_status treemg_run(const treemg_config* cfg, treemg_result** out) {
    if (!cfg || !out) return fail(TREEMG_E_USAGE, "null argument");
    *out = nullptr;
    auto* res = new treemg_result();
    const treemg_status st = guarded([&] {
        res->res = run(cfg->cfg);
        res->channels = cfg->cfg.channels;
    });
    if (st != TREEMG_OK) {
        delete res;
        return st;
    }
    *out = res;
    return TREEMG_OK;
}

void treemg_result_free(treemg_result* res) { delete res; }

treemg_outcome treemg_result_outcome(const treemg_result* res) {
    switch (res->res.outcome) {
        case RunOutcome::Converged: return TREEMG_RUN_CONVERGED;
        case RunOutcome::BudgetExhausted: return TREEMG_RUN_BUDGET_EXHAUSTED;
        case RunOutcome::Diverged: return TREEMG_RUN_DIVERGED;
    }
    return TREEMG_RUN_DIVERGED;
}

int treemg_result_sweeps(const treemg_result* res) { return res->res.sweeps; }

double treemg_result_work_units(const treemg_result* res) { return res->res.workUnits; }

long long treemg_result_vertex_count(const treemg_result* res) {
    return static_cast<long long>(res->res.vertexCount);
}

double treemg_result_final_norm(const treemg_result* res, const char* which, int channel) {  // capi.cpp:102-112
    if (res->res.history.empty()) return 0.0;
    const SweepRecord& rec = res->res.history.back();
    const bool agg = channel < 0;
    if (!agg && channel >= res->channels) return -1.0;
    const bool one = agg || rec.perChannelMax.empty();  // a single channel is its own aggregate
    const auto c = static_cast<std::size_t>(channel);
    if (std::strcmp(which, "max") == 0) return one ? rec.maxNorm : rec.perChannelMax[c];
    if (std::strcmp(which, "euclid") == 0) return one ? rec.euclidNorm : rec.perChannelEuclid[c];
    if (std::strcmp(which, "h") == 0) return one ? rec.hNorm : rec.perChannelH[c];
    return -1.0;
}

double treemg_result_first_norm(const treemg_result* res) { return res->res.firstNorm; }

// ---- extensions --------------------------------------------------------------

int treemg_result_history_rows(const treemg_result* res) { return static_cast<int>(res->res.history.size()); }

treemg_status treemg_result_history_row(const treemg_result* res, int i, double* out6) {
    if (!res || !out6 || i < 0 || i >= static_cast<int>(res->res.history.size()))
        return fail(TREEMG_E_USAGE, "history row out of range");
    const SweepRecord& r = res->res.history[static_cast<std::size_t>(i)];
    out6[0] = r.sweep;
    out6[1] = r.workUnits;
    out6[2] = static_cast<double>(r.vertexCount);
    out6[3] = r.maxNorm;
    out6[4] = r.euclidNorm;
    out6[5] = r.hNorm;
    return TREEMG_OK;
}

double treemg_result_device_ms(const treemg_result* res) { return res->res.deviceMs; }

unsigned long long treemg_result_fingerprint(const treemg_result* res, const char* which) {
    if (!res || !which) return 0;
    if (std::strcmp(which, "u") == 0) return res->res.uHash;
    if (std::strcmp(which, "sc") == 0) return res->res.scHash;
    if (std::strncmp(which, "u#", 2) == 0) {  // "u#<c>": channel c's u
        const int c = std::atoi(which + 2);
        if (c == 0) return res->res.uHash;
        if (c >= 1 && static_cast<std::size_t>(c) <= res->res.channelUHash.size())
            return res->res.channelUHash[static_cast<std::size_t>(c) - 1];
    }
    return 0;
}

treemg_status tmg_test_hypot(const double* x, const double* y, double* out, long long n) {
    if (!x || !y || !out || n < 0) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] { test_hypot(x, y, out, n); });
}

treemg_status tmg_test_divdc3(const double* x, const double* y, double* out, long long n) {
    if (!x || !y || !out || n < 0) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] { test_divdc3(x, y, out, n); });
}

namespace {
Problem problem_from(const tmg_problem* prob) {
    Problem p;
    p.dim = prob->dim;
    p.levels = prob->levels;
    p.ellMin = prob->ell_min;
    p.theta = prob->theta;
    p.phi = Cplx(prob->phi_re, prob->phi_im);
    p.chi = static_cast<ChiKind>(prob->chi_kind);
    p.gaussian = prob->chi_kind == 4;
    p.rhsSeed = prob->rhs_seed;
    p.rhsSphere = prob->rhs_sphere != 0;
    p.fast = prob->precision == 1 || prob->precision == 2;
    p.c64 = prob->precision == 2;
    if (prob->max_vertices > 0) p.maxVertices = static_cast<std::size_t>(prob->max_vertices);
    p.device = prob->device;
    p.sphereLevels = prob->sphere_levels;
    p.levels += p.sphereLevels;
    p.channels = prob->channels > 0 ? prob->channels : 1;
    p.coupling = Cplx(prob->coupling_re, prob->coupling_im);
    if (prob->h_max > 0.0 || prob->h_min > 0.0) {  // dynamic adaptivity: levels from h_max / h_min
        RunConfig rc;
        rc.fixedLevel = 0;
        rc.hMax = prob->h_max;
        rc.hMin = prob->h_min;
        rc.ellMin = prob->ell_min;
        if (!(rc.hMax > 0.0 && rc.hMin > 0.0 && rc.hMin <= rc.hMax))
            throw ConfigError("adaptive runs need 0 < h_min <= h_max");
        p.dynStart = start_level_of(rc);
        p.levels = std::max(p.dynStart, std::min(reference_level_of(rc), 9));
        p.hMax = rc.hMax;
        p.hMin = rc.hMin;
        p.rhsLattice = reference_level_of(rc);
    }
    if (p.ellMin < 1) throw ConfigError("ellMin must be >= 1");
    return p;
}
}  // namespace

treemg_status tmg_nccl_unique_id(unsigned char* out128) {
    if (!out128) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        if (!nccl_unique_id(out128)) throw CudaError("NCCL unavailable");
    });
}

treemg_status tmg_slabs_create(const tmg_problem* prob, int local, int rank, int world,
                               const unsigned char* nccl_id, tmg_slabs** out) {
    if (!prob || !out) return fail(TREEMG_E_USAGE, "null argument");
    *out = nullptr;
    auto* h = new tmg_slabs();
    const treemg_status st = guarded([&] {
        const Problem p = problem_from(prob);
        h->device = p.device;
        const DeviceScope ds(h->device);
        h->g = std::make_unique<SlabGroup>(p, local, rank, world, nccl_id);
    });
    if (st != TREEMG_OK) {
        delete h;
        return st;
    }
    *out = h;
    return TREEMG_OK;
}

treemg_status tmg_slabs_create_local(const tmg_problem* prob, int slabs, int devices, tmg_slabs** out) {
    if (!prob || !out) return fail(TREEMG_E_USAGE, "null argument");
    *out = nullptr;
    auto* h = new tmg_slabs();
    const treemg_status st = guarded([&] {
        const Problem p = problem_from(prob);
        h->device = p.device;
        const DeviceScope ds(h->device);
        h->g = std::make_unique<SlabGroup>(p, slabs, 0, slabs, nullptr, devices);
    });
    if (st != TREEMG_OK) {
        delete h;
        return st;
    }
    *out = h;
    return TREEMG_OK;
}

treemg_status tmg_slabs_get_field(tmg_slabs* h, int level, const char* field, double* out) {
    if (!h || !field || !out) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        const DeviceScope ds(h->device);
        h->g->get_field(level, field, out);
    });
}

void tmg_slabs_destroy(tmg_slabs* h) {
    if (!h) return;
    const DeviceScope ds(h->device);
    delete h;
}

treemg_status tmg_slabs_cycle(tmg_slabs* h, const tmg_policy* pol, int n, tmg_sweep_stats* out) {
    if (!h || !pol) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        const DeviceScope ds(h->device);
        Policy p = policy_from(pol);
        if (n < 1) throw ConfigError("sweep counter starts at 1");
        if (p.bpx) p.hbMask = false;
        fill_stats(h->g->cycle(p, n), out);
    });
}

treemg_status tmg_slabs_get_fine_u(tmg_slabs* h, double* out) {
    if (!h || !out) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        const DeviceScope ds(h->device); h->g->get_fine_u(out); });
}

treemg_status tmg_slabs_time_cycles(tmg_slabs* h, const tmg_policy* pol, int n0, int count, double* out4) {
    if (!h || !pol || !out4) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        const DeviceScope ds(h->device);
        Policy p = policy_from(pol);
        if (p.bpx) p.hbMask = false;
        h->g->time_cycles(p, n0, count, out4);
    });
}

treemg_status tmg_slabs_e2e_step(tmg_slabs* h, const tmg_policy* pol, int n, const double* chi, double* out3,
                                 long long* h2d_bytes) {
    if (!h || !pol || !chi || !out3) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        const DeviceScope ds(h->device);
        Policy p = policy_from(pol);
        if (p.bpx) p.hbMask = false;
        h->g->e2e_step(p, n, chi, out3, h2d_bytes);
    });
}

treemg_status tmg_slab_plan(int levels, int world, int* out8) {
    if (!out8) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        // the chunking the live device runs (co-resident fused blocks); 4 x 148 without a GPU
        int ndev = 0, resident = 4 * 148;
        if (cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0) {
            int dev = 0, sms = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            resident = fused3_resident_blocks(sms);
        } else {
            cudaGetLastError();
        }
        const auto plan = slab_plan(levels, world, resident);
        for (size_t r = 0; r < plan.size(); ++r)
            for (int k = 0; k < 8; ++k) out8[8 * r + static_cast<size_t>(k)] = plan[r][static_cast<size_t>(k)];
    });
}

int tmg_slabs_owned_planes(tmg_slabs* h, int* z0, int* z1) {
    if (!h || !z0 || !z1) return 0;
    return h->g->owned_planes(z0, z1);
}

treemg_status tmg_hierarchy_create(const tmg_problem* prob, tmg_hierarchy** out) {
    if (!prob || !out) return fail(TREEMG_E_USAGE, "null argument");
    *out = nullptr;
    auto* h = new tmg_hierarchy();
    const treemg_status st = guarded([&] {
        const Problem p = problem_from(prob);
        h->device = p.device;
        const DeviceScope ds(h->device);
        h->h = std::make_unique<Hierarchy>(p);
    });
    if (st != TREEMG_OK) {
        delete h;
        return st;
    }
    *out = h;
    return TREEMG_OK;
}

void tmg_hierarchy_destroy(tmg_hierarchy* h) {
    if (!h) return;
    const DeviceScope ds(h->device);
    delete h;
}

treemg_status tmg_td_add(tmg_hierarchy* h, const tmg_policy* pol, int n, tmg_sweep_stats* out) {
    if (!h || !pol) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        const DeviceScope ds(h->device);
        Policy p = policy_from(pol);
        if (p.bpx) throw ConfigError("td_add: policy has bpx set, use td_bpx");  // cycles.cpp:338
        if (n < 1) throw ConfigError("sweep counter starts at 1");
        fill_stats(h->last = h->h->cycle(p, n), out);
    });
}

treemg_status tmg_td_bpx(tmg_hierarchy* h, const tmg_policy* pol, int n, tmg_sweep_stats* out) {
    if (!h || !pol) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        const DeviceScope ds(h->device);
        Policy p = policy_from(pol);
        if (n < 1) throw ConfigError("sweep counter starts at 1");
        p.bpx = true;  // cycles.cpp:349-351
        p.hbMask = false;
        fill_stats(h->last = h->h->cycle(p, n), out);
    });
}

treemg_status tmg_bu_fas(tmg_hierarchy* h, const tmg_policy* pol, int n, tmg_sweep_stats* out) {
    if (!h || !pol) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        const DeviceScope ds(h->device);
        if (n < 1) throw ConfigError("sweep counter starts at 1");
        fill_stats(h->h->bu_fas(policy_from(pol), n), out);
    });
}

treemg_status tmg_textbook_add(tmg_hierarchy* h, double omega_s_re, double omega_s_im, double omega_cg_re,
                               double omega_cg_im, tmg_sweep_stats* out) {
    if (!h) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        const DeviceScope ds(h->device);
        fill_stats(h->h->textbook_add(Cplx(omega_s_re, omega_s_im), Cplx(omega_cg_re, omega_cg_im)), out);
    });
}

long long tmg_lattice_size(const tmg_hierarchy* h, int level) { return h ? h->h->lattice_size(level) : 0; }

treemg_status tmg_get_field(tmg_hierarchy* h, int level, const char* field, double* out) {
    if (!h || !field || !out) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        const DeviceScope ds(h->device); h->h->get_field(level, field, out); });
}

treemg_status tmg_set_field(tmg_hierarchy* h, int level, const char* field, const double* in) {
    if (!h || !field || !in) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        const DeviceScope ds(h->device); h->h->set_field(level, field, in); });
}

treemg_status tmg_set_fine_interior_u(tmg_hierarchy* h, const double* u) {
    if (!h || !u) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        const DeviceScope ds(h->device); h->h->set_fine_interior_u(u); });
}

treemg_status tmg_set_random_initial_guess(tmg_hierarchy* h, unsigned long long seed) {
    if (!h) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        const DeviceScope ds(h->device); h->h->set_random_initial_guess(seed); });
}

treemg_status tmg_set_fine_rhs(tmg_hierarchy* h, const double* chi) {
    if (!h || !chi) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        const DeviceScope ds(h->device); h->h->set_fine_rhs(chi); });
}

treemg_status tmg_get_flags(tmg_hierarchy* h, int level, unsigned char* flags, signed char* succ,
                            unsigned char* cells) {
    if (!h) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        const DeviceScope ds(h->device);
        if (!h->h->get_flags(level, flags, succ, cells)) throw ConfigError("get_flags: the tree is regular");
    });
}

treemg_status tmg_sphere_tree(int dim, int base, int sphere_levels, int level, unsigned char* flags,
                              signed char* succ, unsigned char* cells, unsigned char* finish_corner) {
    return guarded([&] {
        if (dim < 1 || dim > 3 || base < 1 || sphere_levels < 1 || base + sphere_levels > 9)
            throw ConfigError("tmg_sphere_tree: bad arguments");
        const int L = base + sphere_levels;
        if (level < 0 || level > L) throw ConfigError("tmg_sphere_tree: level out of range");
        const std::vector<amr::HostLevel> lv = amr::build_sphere_tree(dim, base, L);
        const amr::HostLevel& h = lv[static_cast<size_t>(level)];
        long long full = 1;
        for (int d = 0; d < dim; ++d) full *= h.m + 1;
        if (flags) std::fill(flags, flags + full, 0);
        if (succ) std::fill(succ, succ + full, static_cast<signed char>(-1));
        if (cells) std::fill(cells, cells + full, 0);
        if (finish_corner) std::fill(finish_corner, finish_corner + full, 0xFF);
        for (long long f = 0; f < h.n; ++f) {
            long long ff = f, gf = 0, s = 1;
            for (int d = 0; d < dim; ++d) {
                gf += (h.lo[d] + ff % h.n1[d]) * s;
                ff /= h.n1[d];
                s *= h.m + 1;
            }
            if (cells) cells[gf] = h.cflag[f];
            if (!(h.vflag[f] & amr::kExists)) continue;
            if (flags) flags[gf] = h.vflag[f];
            if (succ) succ[gf] = h.succ[f];
            if (finish_corner) finish_corner[gf] = h.estar[f];
        }
    });
}

struct tmg_dyn {
    std::unique_ptr<dyn::DynTree> t;
};

treemg_status tmg_dyn_create(int dim, int start, int max_level, int ell_min, double h_min, long long max_vertices,
                             tmg_dyn** out) {
    if (!out) return fail(TREEMG_E_USAGE, "null argument");
    *out = nullptr;
    auto* h = new tmg_dyn();
    const treemg_status st = guarded([&] {
        h->t = std::make_unique<dyn::DynTree>(dim, start, max_level, ell_min, h_min,
                                              static_cast<std::size_t>(max_vertices > 0 ? max_vertices : 8388608));
    });
    if (st != TREEMG_OK) {
        delete h;
        return st;
    }
    *out = h;
    return TREEMG_OK;
}

void tmg_dyn_destroy(tmg_dyn* h) { delete h; }

int tmg_dyn_depth(const tmg_dyn* h) { return h ? h->t->depth() : -1; }

long long tmg_dyn_interior_count(const tmg_dyn* h) { return h ? h->t->interior_fine_vertex_count() : -1; }

treemg_status tmg_dyn_set_cell_marks(tmg_dyn* h, int level, const unsigned char* cells) {
    if (!h || !cells) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        if (level < 0 || level > h->t->max_level()) throw ConfigError("tmg_dyn_set_cell_marks: level out of range");
        dyn::Level& L = h->t->level(level);
        const unsigned char mk = dyn::kRM | dyn::kEM;
        for (long long f = 0; f < L.n; ++f)
            L.cell[f] = static_cast<unsigned char>((L.cell[f] & ~mk) | ((L.cell[f] & dyn::kCE) ? (cells[f] & mk) : 0));
    });
}

treemg_status tmg_dyn_sweep(tmg_dyn* h, long long* out4) {
    if (!h) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        const dyn::SweepCounts c = h->t->sweep();
        h->t->clear_notes();
        if (out4) {
            out4[0] = c.refinedCells;
            out4[1] = c.erasedCells;
            out4[2] = c.updatedFineVertices;
            out4[3] = c.specialVertices;
        }
    });
}

treemg_status tmg_dyn_flags(tmg_dyn* h, int level, unsigned char* flags, signed char* succ, unsigned char* cells) {
    if (!h) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        if (level < 0 || level > h->t->max_level()) throw ConfigError("tmg_dyn_flags: level out of range");
        const dyn::Level& L = h->t->level(level);
        for (long long f = 0; f < L.n; ++f) {
            const bool ex = level <= h->t->depth() && (L.vtx[f] & dyn::kVE);
            if (flags) flags[f] = ex ? L.vtx[f] : 0;
            if (succ) succ[f] = ex ? L.succ[f] : static_cast<signed char>(-1);
            if (cells) cells[f] = level <= h->t->depth() ? L.cell[f] : 0;
        }
    });
}

treemg_status tmg_dyn_sweep_tables(tmg_dyn* h, int level, unsigned char* role, unsigned char* finish_corner,
                                   unsigned char* finish_cells, unsigned char* skip_cells, signed char* succ,
                                   unsigned char* cells) {
    if (!h) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        if (level < 0 || level > h->t->max_level()) throw ConfigError("tmg_dyn_sweep_tables: level out of range");
        const dyn::Level& L = h->t->level(level);
        const size_t n = static_cast<size_t>(L.n);
        if (role) std::copy(L.sflag.begin(), L.sflag.end(), role);
        if (finish_corner) std::copy(L.sestar.begin(), L.sestar.end(), finish_corner);
        if (finish_cells) std::copy(L.sfmask.begin(), L.sfmask.end(), finish_cells);
        if (skip_cells) std::copy(L.sskip.begin(), L.sskip.end(), skip_cells);
        if (succ) std::copy(L.ssucc.begin(), L.ssucc.end(), succ);
        if (cells) std::copy(L.scell.begin(), L.scell.begin() + static_cast<long long>(n), cells);
    });
}

long long tmg_hanging_vertices(const tmg_hierarchy* h) { return h ? h->h->hanging_vertices() : 0; }

long long tmg_leaf_vertices(const tmg_hierarchy* h) { return h ? h->h->interior_fine_vertices() : 0; }

unsigned long long tmg_field_hash(tmg_hierarchy* h, int level, const char* field) {
    unsigned long long v = 0;
    if (!h || !field) return 0;
    guarded([&] { v = h->h->field_hash(level, field); });
    return v;
}

treemg_status tmg_time_cycles(tmg_hierarchy* h, const tmg_policy* pol, int n0, int count, int flush_l2,
                              double* out4) {
    if (!h || !pol || !out4) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        const DeviceScope ds(h->device); h->h->time_cycles(policy_from(pol), n0, count, flush_l2 != 0, out4); });
}

treemg_status tmg_e2e_step(tmg_hierarchy* h, const tmg_policy* pol, int n, const double* chi, double* out3) {
    if (!h || !pol || !chi || !out3) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        const DeviceScope ds(h->device); h->h->e2e_step(policy_from(pol), n, chi, out3); });
}

treemg_status tmg_mark(tmg_hierarchy* h, long long* out9) {
    if (!h) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        const DeviceScope ds(h->device);
        const AmrMarkStats m = h->h->mark();
        if (out9) {
            const long long v[9] = {h->last.refinedCells, h->last.erasedCells, m.refineVertices, m.eraseVertices,
                                    m.refineCells, m.eraseCells, m.vetoConvergence, m.vetoHMin, m.vetoHMax};
            std::copy(v, v + 9, out9);
        }
    });
}

int tmg_levels(const tmg_hierarchy* h) { return h ? h->h->levels() : -1; }

treemg_status tmg_dyn_phase_ms(const tmg_hierarchy* h, double* out6) {
    if (!h || !out6) return fail(TREEMG_E_USAGE, "null argument");
    h->h->dyn_phase_ms(out6);
    return TREEMG_OK;
}

long long tmg_existing_vertices(const tmg_hierarchy* h) { return h ? h->h->existing_vertices() : 0; }

treemg_status tmg_set_cell_marks(tmg_hierarchy* h, int level, const unsigned char* cells) {
    if (!h || !cells) return fail(TREEMG_E_USAGE, "null argument");
    return guarded([&] {
        const DeviceScope ds(h->device); h->h->set_cell_marks(level, cells); });
}

int tmg_channel_norms(tmg_hierarchy* h, double* maxNorm, double* euclid, double* hNorm, int cap) {
    if (!h) return -1;
    const SweepStats& st = h->last;
    const int n = static_cast<int>(st.chMax.size());
    for (int c = 0; c < n && c < cap; ++c) {
        if (maxNorm) maxNorm[c] = st.chMax[c];
        if (euclid) euclid[c] = st.chEuclid[c];
        if (hNorm) hNorm[c] = st.chH[c];
    }
    return n;
}

}  // extern "C"
