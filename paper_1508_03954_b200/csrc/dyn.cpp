// DynTree: see dyn.hpp.  Every rule below restates the reference's traversal
// bookkeeping; the file:line of each is given where it is used.
#include "dyn.hpp"

#include <algorithm>
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
        for (int d = 0; d < p_; ++d) L.n *= L.n1;
        if (L.n >= (1LL << 31)) throw CapacityError("dynamic adaptivity: level lattice exceeds 2^31 points");
        const size_t n = static_cast<size_t>(L.n);
        L.cell.assign(n, 0);
        L.vtx.assign(n, 0);
        L.succ.assign(n, 0);
        L.epoch.assign(n, 0);
        L.entered.assign(n, 0);
        L.done.assign(n, 0);
        L.expected.assign(n, 0);
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

// refresh_classification, spacetree.cpp:438-489
void DynTree::refresh(int l, const int* v) {
    Level& L = lv_[l];
    const long long f = flat(l, v);
    unsigned char fl = L.vtx[f] & kVE;
    bool bnd = false, cp = l > 0;
    for (int d = 0; d < p_; ++d) {
        bnd |= v[d] == 0 || v[d] == L.m;
        cp &= v[d] % 3 == 0;
    }
    if (bnd) fl |= kVB;
    if (cp) fl |= kVC;
    const int total = indomain_adjacent(l, v);
    int have = 0, refinedAdj = 0;
    for (int e = 0; e < (1 << p_); ++e) {
        int c[3] = {0, 0, 0};
        for (int d = 0; d < p_; ++d) c[d] = v[d] - bit(e, d);
        if (!has_cell(l, c)) continue;
        ++have;
        if (L.cell[static_cast<size_t>(flat(l, c))] & kCR) ++refinedAdj;
    }
    const bool hanging = have < total;
    const bool refined = !hanging && refinedAdj == have;
    if (hanging) fl |= kVH;
    if (refined) fl |= kVR;
    L.vtx[f] = fl;
    if (!refined) {
        L.succ[f] = 0;
        return;
    }
    int minSucc = INT_MAX;
    if (l + 1 <= depth_) {
        const Level& F = lv_[l + 1];
        int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
        for (int d = 0; d < p_; ++d) {
            lo[d] = std::max(0, 3 * v[d] - 3);
            hi[d] = std::min(F.m, 3 * v[d] + 3);
        }
        int w[3] = {0, 0, 0};
        for (w[2] = p_ > 2 ? lo[2] : 0; w[2] <= (p_ > 2 ? hi[2] : 0); ++w[2])
            for (w[1] = p_ > 1 ? lo[1] : 0; w[1] <= (p_ > 1 ? hi[1] : 0); ++w[1])
                for (w[0] = lo[0]; w[0] <= hi[0]; ++w[0]) {
                    const long long wf = flat(l + 1, w);
                    const unsigned char fv = F.vtx[wf];
                    if (!(fv & kVE)) continue;
                    minSucc = std::min(minSucc, (fv & kVH) ? 0 : static_cast<int>(F.succ[wf]));
                }
    }
    L.succ[f] = static_cast<signed char>(minSucc == INT_MAX ? 0 : 1 + minSucc);
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
void DynTree::touch(int l, const int* v) {
    Level& L = lv_[l];
    const long long f = flat(l, v);
    if (L.epoch[f] == epoch_) return;
    L.epoch[f] = epoch_;
    L.done[f] = 0;
    L.expected[f] = static_cast<unsigned char>(existing_adjacent(l, v));
    const bool hangNow = L.expected[f] < indomain_adjacent(l, v);
    L.sflag[f] = static_cast<unsigned char>(kSE | (hangNow ? kSH : 0) | (L.vtx[f] & (kVB | kVC)));
}

// finish_vertex_visit, spacetree.cpp:382-392, and the classification refresh
// of touch_last (cycles.cpp:245) for the touch-last role
void DynTree::finish(int l, const int* v, int corner, const int* cell) {
    Level& L = lv_[l];
    const long long f = flat(l, v);
    ++L.done[f];
    if (L.done[f] != L.expected[f]) return;
    int ce = 0;  // cell convention of exact_ops.cuh: cell = v - 1 + bits(ce)
    for (int d = 0; d < p_; ++d) ce |= (cell[d] - v[d] + 1) << d;
    if (L.sfmask[f] == 0) L.sestar[f] = static_cast<unsigned char>(corner);
    else L.sflag[f] |= kSSpecial;  // finishes more than once
    L.sfmask[f] |= static_cast<unsigned char>(1u << ce);
    if (L.sflag[f] & kSH) return;  // destroy_hanging
    if (dirty_) refresh(l, v);
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
    P.cell[static_cast<size_t>(flat(l, c))] |= kCR;
    for (int t = 0; t < blockCells; ++t) {
        int ci[3] = {0, 0, 0}, tt = t;
        for (int d = 0; d < p_; ++d) {
            ci[d] = 3 * c[d] + tt % 3;
            tt /= 3;
        }
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
        if (!(F.vtx[f] & kVE)) {  // create_vertex_if_missing, spacetree.cpp:245-270
            if (F.epoch[f] == epoch_)
                // it lived earlier in this traversal (touched, then deleted by an erase): two
                // vertices would share one lattice slot of the level passes
                throw UnsupportedConfigError(
                    "B200 path: a vertex erased and re-created within one traversal (an erase next to a later "
                    "refinement) is not supported");
            check_capacity(1);
            F.vtx[f] = kVE;
            F.succ[f] = 0;
            ++total_;
            F.epoch[f] = epoch_;
            F.done[f] = 0;
            F.expected[f] = static_cast<unsigned char>(existing_adjacent(l + 1, vi));
            const bool hangNow = F.expected[f] < indomain_adjacent(l + 1, vi);
            refresh(l + 1, vi);
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
        F.cell[cf] = 0;
    }
    lv_[l].cell[static_cast<size_t>(flat(l, c))] &= static_cast<unsigned char>(~kCR);
    for (int t = 0; t < blockVerts; ++t) {
        int vi[3] = {0, 0, 0}, tt = t;
        for (int d = 0; d < p_; ++d) {
            vi[d] = 3 * c[d] + tt % 4;
            tt /= 4;
        }
        const size_t f = static_cast<size_t>(flat(l + 1, vi));
        if (existing_adjacent(l + 1, vi) == 0 && (F.vtx[f] & kVE)) {
            F.vtx[f] = 0;
            --total_;
        }
    }
    dirty_ = true;
}

// visit_cell, spacetree.cpp:394-424, with the structural hooks of TdSweep:
// enter_cell's refine mark (cycles.cpp:174-180), leave_cell's erase (:222-241)
void DynTree::visit(int l, const int* c) {
    const int nc = 1 << p_;
    int v[3] = {0, 0, 0};
    for (int e = 0; e < nc; ++e) {
        for (int d = 0; d < p_; ++d) v[d] = c[d] + bit(e, d);
        touch(l, v);
    }
    Level& L = lv_[l];
    const size_t cf = static_cast<size_t>(flat(l, c));
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
    for (int e = 0; e < nc; ++e) {
        for (int d = 0; d < p_; ++d) v[d] = c[d] + bit(e, d);
        finish(l, v, e, c);
    }
}

SweepCounts DynTree::sweep() {
    ++epoch_;
    dirty_ = false;
    counts_ = SweepCounts{};
    for (Level& L : lv_) {
        std::fill(L.sflag.begin(), L.sflag.end(), 0);
        std::fill(L.scell.begin(), L.scell.end(), 0);
        std::fill(L.sestar.begin(), L.sestar.end(), 0xFF);
        std::fill(L.sfmask.begin(), L.sfmask.end(), 0);
        std::fill(L.sskip.begin(), L.sskip.end(), 0);
        std::fill(L.ssucc.begin(), L.ssucc.end(), 0);
    }
    const int zero[3] = {0, 0, 0};
    visit(0, zero);
    for (int l = 0; l <= depth_; ++l) {
        Level& L = lv_[l];
        for (long long f = 0; f < L.n; ++f) {
            unsigned char& s = L.sflag[f];
            if (!(s & kSE)) continue;
            if (L.sfmask[f] == 0) s |= kSSpecial;  // never finishes
            if (s & kSSpecial) ++counts_.specialVertices;
        }
    }
    if (dirty_) {  // TdSweep::run, cycles.cpp:89-92
        classify();
        dirty_ = false;
    }
    return counts_;
}

}  // namespace dyn
}  // namespace tmg
