// DynTree: see dyn.hpp.  Every rule below restates the reference's traversal
// bookkeeping; the file:line of each is given where it is used.
#include "dyn.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <climits>
#include <cmath>
#include <string>

#include "hierarchy.hpp"

namespace tmg {
namespace dyn {

namespace {
constexpr int kMaxLevel = 9;  // spacetree.cpp:12

int pow3i(int l) {
    int r = 1;
    for (int i = 0; i < l; ++i) r *= 3;
    return r;
}

bool bit(int x, int d) { return (x >> d) & 1; }
}  // namespace

DynTree::DynTree(int dim, int start, int maxLevel, int ellMin, double hMinRefine, std::size_t maxVertices)
    : p_(dim), ellMin_(ellMin), depth_(start), hMin_(hMinRefine), maxVertices_(maxVertices) {
    if (dim < 1 || dim > 3) throw ConfigError("dynamic adaptivity: dimension out of range");
    if (start < 1 || start > maxLevel) throw ConfigError("dynamic adaptivity: bad start level");
    lv_.resize(static_cast<size_t>(maxLevel) + 1);
    for (int l = 0; l <= maxLevel; ++l) {
        Level& L = lv_[l];
        L.m = pow3i(l);
        L.n1 = L.m + 1;
        L.n = 1;
        for (int d = 0; d < p_; ++d) {
            L.stride[d] = L.n;
            L.n *= L.n1;
        }
        for (int e = 0; e < (1 << p_); ++e) {
            L.off[e] = 0;
            for (int d = 0; d < p_; ++d) L.off[e] += bit(e, d) ? L.stride[d] : 0;
        }
        if (L.n >= (1LL << 31)) throw CapacityError("dynamic adaptivity: level lattice exceeds 2^31 points");
        const size_t n = static_cast<size_t>(L.n);
        L.cell.assign(n, 0);
        L.vtx.assign(n, 0);
        L.succ.assign(n, 0);
        L.epoch.assign(n, 0);
        L.entered.assign(n, 0);
        L.done.assign(n, 0);
        L.expected.assign(n, 0);
        L.stale.assign(n, 0);
        L.vtxOld.assign(n, 0);
        L.noted.assign(n, 0);
        L.sflag.assign(n, 0);
        L.scell.assign(n, 0);
        L.sestar.assign(n, 0xFF);
        L.sfmask.assign(n, 0);
        L.sskip.assign(n, 0);
        L.ssucc.assign(n, 0);
    }
    // build_regular(start): every cell of levels 0..start, refined below start
    int g[3] = {0, 0, 0};
    for (int l = 0; l <= start; ++l) {
        Level& L = lv_[l];
        for (long long f = 0; f < L.n; ++f) {
            unflat(l, f, g);
            bool inDomain = true, bnd = false, cp = l > 0;
            for (int d = 0; d < p_; ++d) {
                inDomain &= g[d] <= L.m - 1;
                bnd |= g[d] == 0 || g[d] == L.m;
                cp &= g[d] % 3 == 0;
            }
            if (inDomain) L.cell[f] = static_cast<unsigned char>(kCE | (l < start ? kCR : 0));
            L.vtx[f] = static_cast<unsigned char>(kVE | (bnd ? kVB : 0) | (cp ? kVC : 0));
            ++total_;
        }
    }
    classify();
}

long long DynTree::flat(int l, const int* g) const {
    const Level& L = lv_[l];
    long long f = 0, s = 1;
    for (int d = 0; d < p_; ++d) {
        if (g[d] < 0 || g[d] > L.m) return -1;
        f += static_cast<long long>(g[d]) * s;
        s *= L.n1;
    }
    return f;
}

void DynTree::unflat(int l, long long f, int* g) const {
    const Level& L = lv_[l];
    for (int d = 0; d < p_; ++d) {
        g[d] = static_cast<int>(f % L.n1);
        f /= L.n1;
    }
}

bool DynTree::has_cell(int l, const int* c) const {
    if (l < 0 || l > depth_) return false;
    const Level& L = lv_[l];
    for (int d = 0; d < p_; ++d)
        if (c[d] < 0 || c[d] > L.m - 1) return false;
    return L.cell[static_cast<size_t>(flat(l, c))] & kCE;
}

int DynTree::existing_adjacent(int l, const int* v) const {  // spacetree.cpp:145-162
    int have = 0;
    for (int e = 0; e < (1 << p_); ++e) {
        int c[3] = {0, 0, 0};
        for (int d = 0; d < p_; ++d) c[d] = v[d] - bit(e, d);
        if (has_cell(l, c)) ++have;
    }
    return have;
}

int DynTree::indomain_adjacent(int l, const int* v) const {  // spacetree.cpp:133-143
    const int m = lv_[l].m;
    int n = 1;
    for (int d = 0; d < p_; ++d) n *= (v[d] - 1 >= 0 ? 1 : 0) + (v[d] <= m - 1 ? 1 : 0);
    return n;
}

void DynTree::check_capacity(std::size_t add) const {  // spacetree.cpp:240-243
    if (total_ + add > maxVertices_)
        throw CapacityError("vertex capacity exceeded (" + std::to_string(maxVertices_) + ")");
}

void DynTree::ensure_level(int l) {
    if (l >= static_cast<int>(lv_.size()))
        throw CapacityError("dynamic adaptivity: refinement below the allocated reference level");
    depth_ = std::max(depth_, l);
}

// existing cells around lattice point v (cells v - bits(e)), and how many of them are refined
int DynTree::adjacent_cells(int l, long long f, const int* v, int* refinedAdj) const {
    const Level& L = lv_[l];
    int low = 0;  // axes on which v has no lower neighbour cell
    for (int d = 0; d < p_; ++d) low |= (v[d] == 0) << d;
    int have = 0, ref = 0;
    for (int e = 0; e < (1 << p_); ++e) {
        if (e & low) continue;
        const unsigned char c = L.cell[static_cast<size_t>(f - L.off[e])];  // upper-rim cells are never set
        if (c & kCE) {
            ++have;
            ref += (c & kCR) ? 1 : 0;
        }
    }
    if (refinedAdj) *refinedAdj = ref;
    return have;
}

void DynTree::note_vtx(Level& L, long long f) {
    if (L.noted[f] & 1) return;
    L.noted[f] |= 1;
    L.vtxOld[f] = L.vtx[f];
    L.vtxNoted.push_back(f);
}

void DynTree::note_cell(Level& L, long long f) {
    if (L.noted[f] & 2) return;
    L.noted[f] |= 2;
    L.cellNoted.push_back(f);
}

void DynTree::clear_notes() {
    for (Level& L : lv_) {
        for (long long f : L.vtxNoted) L.noted[f] &= static_cast<unsigned char>(~1);
        for (long long f : L.cellNoted) L.noted[f] &= static_cast<unsigned char>(~2);
        L.vtxNoted.clear();
        L.cellNoted.clear();
    }
}

void DynTree::mark_stale(int l, const int* v) {
    Level& L = lv_[l];
    long long f = 0;
    for (int d = 0; d < p_; ++d) {
        if (v[d] < 0 || v[d] > L.m) return;
        f += v[d] * L.stride[d];
    }
    if (!L.stale[f]) {
        L.stale[f] = 1;
        L.staleList.push_back(f);
    }
}

void DynTree::stale_parents(int l, const int* v) {
    if (l < 1) return;
    const Level& C = lv_[l - 1];
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int d = 0; d < p_; ++d) {  // W with |3 W - v| <= 3 on every axis
        lo[d] = std::max(0, (v[d] - 1) / 3);
        hi[d] = std::min(C.m, (v[d] + 3) / 3);
    }
    int w[3] = {0, 0, 0};
    for (w[2] = lo[2]; w[2] <= hi[2]; ++w[2])
        for (w[1] = lo[1]; w[1] <= hi[1]; ++w[1])
            for (w[0] = lo[0]; w[0] <= hi[0]; ++w[0]) mark_stale(l - 1, w);
}

// refresh_classification, spacetree.cpp:438-489
bool DynTree::refresh(int l, const int* v) {
    Level& L = lv_[l];
    long long f = 0;
    bool bnd = false, cp = l > 0;
    for (int d = 0; d < p_; ++d) {
        f += v[d] * L.stride[d];
        bnd |= v[d] == 0 || v[d] == L.m;
        cp &= v[d] % 3 == 0;
    }
    L.stale[f] = 0;
    note_vtx(L, f);
    const unsigned char oldFl = L.vtx[f];
    const signed char oldSucc = L.succ[f];
    unsigned char fl = L.vtx[f] & kVE;
    if (bnd) fl |= kVB;
    if (cp) fl |= kVC;
    const int total = indomain_adjacent(l, v);
    int refinedAdj = 0;
    const int have = l <= depth_ ? adjacent_cells(l, f, v, &refinedAdj) : 0;
    const bool hanging = have < total;
    const bool refined = !hanging && refinedAdj == have;
    if (hanging) fl |= kVH;
    if (refined) fl |= kVR;
    L.vtx[f] = fl;
    if (!refined) {
        L.succ[f] = 0;
        if (fl != oldFl || oldSucc != 0) stale_parents(l, v);
        return fl != oldFl || oldSucc != 0;
    }
    int minSucc = INT_MAX;
    if (l + 1 <= depth_) {
        const Level& F = lv_[l + 1];
        int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
        for (int d = 0; d < p_; ++d) {
            lo[d] = std::max(0, 3 * v[d] - 3);
            hi[d] = std::min(F.m, 3 * v[d] + 3);
        }
        for (int z = p_ > 2 ? lo[2] : 0; z <= (p_ > 2 ? hi[2] : 0); ++z)
            for (int y = p_ > 1 ? lo[1] : 0; y <= (p_ > 1 ? hi[1] : 0); ++y) {
                const long long row = z * F.stride[2] + y * F.stride[1];
                for (int x = lo[0]; x <= hi[0]; ++x) {
                    const long long wf = row + x;
                    const unsigned char fv = F.vtx[static_cast<size_t>(wf)];
                    if (!(fv & kVE)) continue;
                    minSucc = std::min(minSucc, (fv & kVH) ? 0 : static_cast<int>(F.succ[static_cast<size_t>(wf)]));
                }
            }
    }
    L.succ[f] = static_cast<signed char>(minSucc == INT_MAX ? 0 : 1 + minSucc);
    const bool changed = fl != oldFl || L.succ[f] != oldSucc;
    if (changed) stale_parents(l, v);
    return changed;
}

// classify() restricted to the vertices whose inputs changed, finest level
// first so that succ changes propagate upwards (same result as classify())
void DynTree::classify_stale() {
    int g[3] = {0, 0, 0};
    for (int l = static_cast<int>(lv_.size()) - 1; l >= 0; --l) {
        Level& L = lv_[l];
        for (size_t i = 0; i < L.staleList.size(); ++i) {
            const long long f = L.staleList[i];
            if (!L.stale[f]) continue;
            if (!(L.vtx[f] & kVE) || l > depth_) {
                L.stale[f] = 0;
                continue;
            }
            unflat(l, f, g);
            refresh(l, g);
        }
        L.staleList.clear();
    }
}

void DynTree::classify() {
    for (int l = depth_; l >= 0; --l) {
        Level& L = lv_[l];
        int g[3] = {0, 0, 0};
        for (long long f = 0; f < L.n; ++f) {
            if (!(L.vtx[f] & kVE)) continue;
            unflat(l, f, g);
            refresh(l, g);
        }
    }
}

void DynTree::clear_marks() {
    for (Level& L : lv_)
        for (unsigned char& c : L.cell) c &= static_cast<unsigned char>(~(kRM | kEM));
}

long long DynTree::interior_fine_vertex_count() const {
    long long n = 0;
    for (int l = 0; l <= depth_; ++l)
        for (unsigned char v : lv_[l].vtx)
            if ((v & kVE) && !(v & (kVH | kVR | kVB))) ++n;
    return n;
}

// touch_vertex, spacetree.cpp:367-380
void DynTree::touch(int l, long long f, const int* v) {
    Level& L = lv_[l];
    if (L.epoch[f] == epoch_) return;
    L.epoch[f] = epoch_;
    L.sweepList.push_back(f);
    L.done[f] = 0;
    L.expected[f] = static_cast<unsigned char>(adjacent_cells(l, f, v, nullptr));
    const bool hangNow = L.expected[f] < indomain_adjacent(l, v);
    L.sflag[f] = static_cast<unsigned char>(kSE | (hangNow ? kSH : 0) | (L.vtx[f] & (kVB | kVC)));
}

// finish_vertex_visit, spacetree.cpp:382-392, and the classification refresh
// of touch_last (cycles.cpp:245) for the touch-last role; v is corner `corner`
// of the cell being left
void DynTree::finish(int l, long long f, const int* v, int corner) {
    Level& L = lv_[l];
    ++L.done[f];
    if (L.done[f] != L.expected[f]) return;
    const int ce = (~corner) & ((1 << p_) - 1);  // cell convention of exact_ops.cuh: cell = v - 1 + bits(ce)
    if (L.sfmask[f] == 0) L.sestar[f] = static_cast<unsigned char>(corner);
    else L.sflag[f] |= kSSpecial;  // finishes more than once
    L.sfmask[f] |= static_cast<unsigned char>(1u << ce);
    if (L.sflag[f] & kSH) return;  // destroy_hanging
    if (dirty_ && L.stale[f]) refresh(l, v);  // unchanged inputs: the stored classification is current
    const unsigned char vf = L.vtx[f];
    if (vf & kVR) L.sflag[f] |= kSR;
    L.ssucc[f] = L.succ[f];
    if (!(vf & kVR) && !(vf & kVB)) ++counts_.updatedFineVertices;  // cycles.cpp:247-249
}

// refine_cell inside the traversal, spacetree.cpp:272-329
void DynTree::refine(int l, const int* c) {
    if (l + 1 > kMaxLevel) throw CapacityError("refine_cell: maximum depth reached");
    ensure_level(l + 1);
    Level& P = lv_[l];
    Level& F = lv_[l + 1];
    int blockCells = 1, blockVerts = 1;
    for (int d = 0; d < p_; ++d) {
        blockCells *= 3;
        blockVerts *= 4;
    }
    check_capacity(static_cast<std::size_t>(blockVerts));
    note_cell(P, flat(l, c));
    P.cell[static_cast<size_t>(flat(l, c))] |= kCR;
    for (int e = 0; e < (1 << p_); ++e) {  // the cell's corners see one more refined cell
        int w[3] = {0, 0, 0};
        for (int d = 0; d < p_; ++d) w[d] = c[d] + bit(e, d);
        mark_stale(l, w);
    }
    for (int t = 0; t < blockCells; ++t) {
        int ci[3] = {0, 0, 0}, tt = t;
        for (int d = 0; d < p_; ++d) {
            ci[d] = 3 * c[d] + tt % 3;
            tt /= 3;
        }
        note_cell(F, flat(l + 1, ci));
        F.cell[static_cast<size_t>(flat(l + 1, ci))] = kCE;
    }
    for (int t = 0; t < blockVerts; ++t) {
        int vi[3] = {0, 0, 0}, rel[3] = {0, 0, 0}, tt = t;
        for (int d = 0; d < p_; ++d) {
            rel[d] = tt % 4;
            vi[d] = 3 * c[d] + rel[d];
            tt /= 4;
        }
        const long long f = flat(l + 1, vi);
        mark_stale(l + 1, vi);  // new adjacent cells
        if (!(F.vtx[f] & kVE)) {  // create_vertex_if_missing, spacetree.cpp:245-270
            if (F.epoch[f] == epoch_)
                // it lived earlier in this traversal (touched, then deleted by an erase): two
                // vertices would share one lattice slot of the level passes
                throw UnsupportedConfigError(
                    "B200 path: a vertex erased and re-created within one traversal (an erase next to a later "
                    "refinement) is not supported");
            check_capacity(1);
            note_vtx(F, f);
            F.vtx[f] = kVE;
            F.succ[f] = 0;
            ++total_;
            F.epoch[f] = epoch_;
            F.sweepList.push_back(f);
            F.done[f] = 0;
            F.expected[f] = static_cast<unsigned char>(existing_adjacent(l + 1, vi));
            const bool hangNow = F.expected[f] < indomain_adjacent(l + 1, vi);
            refresh(l + 1, vi);
            stale_parents(l + 1, vi);  // a new vertex in the coarser vertices' succ scans
            F.sflag[f] = static_cast<unsigned char>(kSE | kSCreated | (hangNow ? kSH : 0) | (F.vtx[f] & (kVB | kVC)));
            // adjacent cells already entered in this traversal never reach it
            unsigned char skip = 0;
            for (int e = 0; e < (1 << p_); ++e) {
                int cc[3] = {0, 0, 0};
                for (int d = 0; d < p_; ++d) cc[d] = vi[d] - 1 + bit(e, d);
                if (has_cell(l + 1, cc) && F.entered[static_cast<size_t>(flat(l + 1, cc))] == epoch_)
                    skip |= static_cast<unsigned char>(1u << e);
            }
            F.sskip[f] = skip;
            if (skip) F.sflag[f] |= kSSpecial;
        } else if (F.epoch[f] == epoch_) {
            int added = 1;
            for (int d = 0; d < p_; ++d) added *= (rel[d] == 1 || rel[d] == 2) ? 2 : 1;
            F.expected[f] = static_cast<unsigned char>(F.expected[f] + added);
        }
    }
    dirty_ = true;
}

// erase_subtree, spacetree.cpp:331-365
void DynTree::erase(int l, const int* c) {
    Level& F = lv_[l + 1];
    int blockCells = 1, blockVerts = 1;
    for (int d = 0; d < p_; ++d) {
        blockCells *= 3;
        blockVerts *= 4;
    }
    for (int t = 0; t < blockCells; ++t) {
        int ci[3] = {0, 0, 0}, tt = t;
        for (int d = 0; d < p_; ++d) {
            ci[d] = 3 * c[d] + tt % 3;
            tt /= 3;
        }
        const size_t cf = static_cast<size_t>(flat(l + 1, ci));
        if (F.cell[cf] & kCR) erase(l + 1, ci);
        note_cell(F, static_cast<long long>(cf));
        F.cell[cf] = 0;
    }
    note_cell(lv_[l], flat(l, c));
    lv_[l].cell[static_cast<size_t>(flat(l, c))] &= static_cast<unsigned char>(~kCR);
    for (int e = 0; e < (1 << p_); ++e) {
        int w[3] = {0, 0, 0};
        for (int d = 0; d < p_; ++d) w[d] = c[d] + bit(e, d);
        mark_stale(l, w);
    }
    for (int t = 0; t < blockVerts; ++t) {
        int vi[3] = {0, 0, 0}, tt = t;
        for (int d = 0; d < p_; ++d) {
            vi[d] = 3 * c[d] + tt % 4;
            tt /= 4;
        }
        const size_t f = static_cast<size_t>(flat(l + 1, vi));
        mark_stale(l + 1, vi);
        if (existing_adjacent(l + 1, vi) == 0 && (F.vtx[f] & kVE)) {
            note_vtx(F, static_cast<long long>(f));
            F.vtx[f] = 0;
            --total_;
            stale_parents(l + 1, vi);
        }
    }
    dirty_ = true;
}

// visit_cell, spacetree.cpp:394-424, with the structural hooks of TdSweep:
// enter_cell's refine mark (cycles.cpp:174-180), leave_cell's erase (:222-241)
void DynTree::visit(int l, const int* c) {
    const int nc = 1 << p_;
    Level& L = lv_[l];
    long long cfl = 0;
    for (int d = 0; d < p_; ++d) cfl += c[d] * L.stride[d];
    const size_t cf = static_cast<size_t>(cfl);
    L.cellList.push_back(cfl);
    int v[3] = {0, 0, 0};
    for (int e = 0; e < nc; ++e) {  // touch_vertex: only a vertex's first touch in this sweep does work
        const long long f = cfl + L.off[e];
        if (L.epoch[static_cast<size_t>(f)] == epoch_) continue;
        for (int d = 0; d < p_; ++d) v[d] = c[d] + bit(e, d);
        touch(l, f, v);
    }
    L.entered[cf] = epoch_;
    if (L.cell[cf] & kRM) {
        L.cell[cf] &= static_cast<unsigned char>(~kRM);
        if (!(L.cell[cf] & kCR) && std::pow(3.0, -l) > hMin_) {
            refine(l, c);
            ++counts_.refinedCells;
        }
    }
    const bool refined = L.cell[cf] & kCR;
    L.scell[cf] = static_cast<unsigned char>(kCE | (refined ? kCR : 0));
    if (refined) {
        int blockCells = 1;
        for (int d = 0; d < p_; ++d) blockCells *= 3;
        for (int t = 0; t < blockCells; ++t) {
            int ci[3] = {0, 0, 0}, tt = t;
            for (int d = 0; d < p_; ++d) {
                ci[d] = 3 * c[d] + tt % 3;
                tt /= 3;
            }
            visit(l + 1, ci);
        }
    }
    if (L.cell[cf] & kEM) {
        L.cell[cf] &= static_cast<unsigned char>(~kEM);
        if (L.cell[cf] & kCR) {
            bool flat = true;
            int blockCells = 1;
            for (int d = 0; d < p_; ++d) blockCells *= 3;
            for (int t = 0; t < blockCells && flat; ++t) {
                int ci[3] = {0, 0, 0}, tt = t;
                for (int d = 0; d < p_; ++d) {
                    ci[d] = 3 * c[d] + tt % 3;
                    tt /= 3;
                }
                const long long f = this->flat(l + 1, ci);
                if (lv_[l + 1].cell[static_cast<size_t>(f)] & kCR) flat = false;
            }
            if (flat) {
                erase(l, c);
                ++counts_.erasedCells;
            }
        }
    }
    for (int e = 0; e < nc; ++e) {  // finish_vertex_visit: only the last of the expected visits does work
        const long long f = cfl + L.off[e];
        if (static_cast<unsigned char>(L.done[static_cast<size_t>(f)] + 1) != L.expected[static_cast<size_t>(f)]) {
            ++L.done[static_cast<size_t>(f)];
            continue;
        }
        for (int d = 0; d < p_; ++d) v[d] = c[d] + bit(e, d);
        finish(l, f, v, e);
    }
}

SweepCounts DynTree::sweep() {
    static const bool prof = [] {
        const char* e = std::getenv("TMG_DYN_PROFILE");
        return e && e[0] == '1';
    }();
    auto t0 = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (!prof) return;
        const auto t1 = std::chrono::steady_clock::now();
        std::fprintf(stderr, " [%s %.1fms]", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
        t0 = t1;
    };
    ++epoch_;
    dirty_ = false;
    counts_ = SweepCounts{};
    for (Level& L : lv_) {  // reset the previous sweep's table entries
        for (long long f : L.sweepList) {
            L.sflag[f] = 0;
            L.sestar[f] = 0xFF;
            L.sfmask[f] = 0;
            L.sskip[f] = 0;
            L.ssucc[f] = 0;
        }
        for (long long f : L.cellList) L.scell[f] = 0;
        L.sweepList.clear();
        L.cellList.clear();
    }
    lap("reset");
    const int zero[3] = {0, 0, 0};
    visit(0, zero);
    lap("dfs");
    for (int l = 0; l <= depth_; ++l) {
        Level& L = lv_[l];
        for (long long f : L.sweepList) {
            unsigned char& s = L.sflag[f];
            if (L.sfmask[f] == 0) s |= kSSpecial;  // never finishes
            if (s & kSSpecial) ++counts_.specialVertices;
        }
    }
    lap("scan");
    if (dirty_) {  // TdSweep::run, cycles.cpp:89-92 (classify(), over the vertices it can change)
        classify_stale();
        dirty_ = false;
    }
    lap("classify");
    return counts_;
}

}  // namespace dyn
}  // namespace tmg
