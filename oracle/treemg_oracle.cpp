// CPU restatement of the reference's single-sweep additive multilevel cycle
// (td_add / td_bpx) as two LEVEL PASSES over lattice arrays -- the oracle the
// parity tests check the CUDA path against.
//
// TEST INFRASTRUCTURE ONLY: loaded by tests/ (and smoke()) through ctypes,
// never by the product.  Pinned bit-for-bit against the reference itself
// (oracle/_ref, built from /root/reference) by tests/test_oracle_pin.py and
// against the committed golden fixtures under tests/golden/.
//
// Algorithm: SURVEY.md Appendix A, i.e. the dense transcription
// proj/src/oracle.cpp:465-509 with the per-vertex semantics of
// proj/src/cycles.cpp:102-303.  Arithmetic follows the reference expression
// by expression (std::complex<double>, compiled without FMA) so the result is
// bit-identical to the spacetree traversal, which requires reproducing two
// orders the traversal fixes:
//   * the 2^p cells around a vertex are entered in base-3 Morton (DFS) order
//     (proj/src/spacetree.cpp:394-424), which fixes the summation order of r,
//     r-hat, diag and the leaf load chi at every vertex;
//   * vertices are finished ("touched last") in Morton order of their
//     Morton-maximal adjacent cell, ties by corner index
//     (spacetree.cpp:419-423), which fixes the order in which restricted
//     r-hat values are summed into the coarse chi (cycles.cpp:292-301) and the
//     order of the norm sums (cycles.cpp:248-258).
// Regular grids, one channel, 1 <= p <= 3.

#include <algorithm>
#include <array>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

using Cplx = std::complex<double>;

int pow3(int l) {
    int r = 1;
    for (int i = 0; i < l; ++i) r *= 3;
    return r;
}

// proj/src/elemops.cpp:13-18
Cplx cplx_ipow(Cplx z, int e) {
    if (e < 0) return 1.0 / cplx_ipow(z, -e);
    Cplx r = 1.0;
    for (int i = 0; i < e; ++i) r *= z;
    return r;
}

// proj/src/elemops.cpp:29-55: tensor-product p-linear reference matrices,
// axis 0 = bit 0 of the corner index.
struct RefMat {
    int n = 0;
    double lap[8][8]{}, mas[8][8]{};
};

RefMat build_ref(int p) {
    static const double kLap1[2][2] = {{1.0, -1.0}, {-1.0, 1.0}};
    static const double kMass1[2][2] = {{1.0 / 3.0, 1.0 / 6.0}, {1.0 / 6.0, 1.0 / 3.0}};
    RefMat m;
    m.n = 1 << p;
    for (int a = 0; a < m.n; ++a)
        for (int b = 0; b < m.n; ++b) {
            double mass = 1.0;
            for (int d = 0; d < p; ++d) mass *= kMass1[(a >> d) & 1][(b >> d) & 1];
            m.mas[a][b] = mass;
            double lap = 0.0;
            for (int d = 0; d < p; ++d) {
                double t = kLap1[(a >> d) & 1][(b >> d) & 1];
                for (int i = 0; i < p; ++i)
                    if (i != d) t *= kMass1[(a >> i) & 1][(b >> i) & 1];
                lap += t;
            }
            m.lap[a][b] = lap;
        }
    return m;
}

// proj/src/transfer.cpp:7-8
const double kW0[4] = {1.0, 2.0 / 3.0, 1.0 / 3.0, 0.0};
const double kW1[4] = {0.0, 1.0 / 3.0, 2.0 / 3.0, 1.0};

// proj/src/transfer.cpp:20-40: fold axis 0 first, exact copies at rel 0/3.
Cplx prolong(const Cplx* corners, const int* rel, int p) {
    Cplx vals[8];
    const int nc = 1 << p;
    for (int i = 0; i < nc; ++i) vals[i] = corners[i];
    int n = nc;
    for (int d = 0; d < p; ++d) {
        const int r = rel[d];
        n >>= 1;
        for (int i = 0; i < n; ++i) {
            const Cplx c0 = vals[2 * i], c1 = vals[2 * i + 1];
            if (r == 0) vals[i] = c0;
            else if (r == 3) vals[i] = c1;
            else vals[i] = kW0[r] * c0 + kW1[r] * c1;
        }
    }
    return vals[0];
}

// proj/src/cycles.cpp:802-808
double unit_rand(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    x = x ^ (x >> 31);
    return 2.0 * static_cast<double>(x >> 11) / 9007199254740992.0 - 1.0;
}

// proj/src/spacetree.cpp:15-19
std::uint64_t pack_index(int p, const int* idx) {
    std::uint64_t k = 0;
    for (int d = 0; d < p; ++d) k |= static_cast<std::uint64_t>(static_cast<std::uint16_t>(idx[d])) << (16 * d);
    return k;
}

enum class Kind { JacobiOnly = 0, Undamped = 1, LGrid = 2, Exponential = 3, Transition = 4 };

struct Policy {
    Kind kind = Kind::Exponential;
    Cplx omegaS = Cplx(0.8, 0.0);
    int lGrid = 2;
    bool hb = false, bpx = false, twoPhase = false;
};

// proj/src/cycles.cpp:11-31
Cplx two_phase(int n) {
    const Cplx w1 = 0.01 * Cplx(std::sqrt(3.0), -1.0);
    return (n % 2 == 1) ? w1 : -std::conj(w1);
}

Cplx omega_unmasked(const Policy& pol, int succ, int n) {
    const Cplx ws = pol.twoPhase ? two_phase(n) : pol.omegaS;
    switch (pol.kind) {
        case Kind::JacobiOnly: return succ == 0 ? ws : Cplx(0.0);
        case Kind::Undamped: return ws;
        case Kind::LGrid: return succ <= pol.lGrid ? ws : Cplx(0.0);
        case Kind::Exponential: return cplx_ipow(ws, succ + 1);
        case Kind::Transition: {
            const double e = (1.0 - 1.0 / static_cast<double>(n)) * (succ + 1);
            if (e == 0.0) return Cplx(1.0);
            return std::pow(ws, e);
        }
    }
    return Cplx(0.0);
}

struct Level {
    int m = 0;          // 3^l cells per axis
    std::size_t n = 0;  // (m+1)^p lattice vertices
    std::vector<Cplx> u, sc, sf, si, siNext, chi, r, rHat, uHat, diag;
    std::vector<std::uint32_t> finishOrder;  // touch-last order
};

struct Stats {
    double maxN = 0.0, euclid = 0.0, hN = 0.0;
    std::size_t updated = 0;
};

class Oracle {
  public:
    int p = 2, L = 1, ellMin = 1;
    double theta = 0.0;
    Cplx phi = 0.0;
    int chiKind = 1;  // 0 zero, 1 sin product, 2 ball, 3 seeded
    std::uint64_t rhsSeed = 12345;
    bool rhsSphere = false;
    Policy pol;
    RefMat R;
    std::vector<Level> lv;
    std::vector<Cplx> fineChiNodal;  // chi at the finest-lattice vertices

    void init() {
        R = build_ref(p);
        lv.assign(L + 1, Level{});
        for (int l = 0; l <= L; ++l) {
            Level& V = lv[l];
            V.m = pow3(l);
            V.n = 1;
            for (int d = 0; d < p; ++d) V.n *= static_cast<std::size_t>(V.m + 1);
            for (auto* f : {&V.u, &V.sc, &V.sf, &V.si, &V.siNext, &V.chi, &V.r, &V.rHat, &V.uHat, &V.diag})
                f->assign(V.n, Cplx(0.0));
            build_finish_order(l);
        }
        // nodal chi at the finest level (the only leaf cells of a regular tree)
        Level& F = lv[L];
        fineChiNodal.assign(F.n, Cplx(0.0));
        const double h = std::pow(3.0, -L);
        for (std::size_t f = 0; f < F.n; ++f) {
            int idx[3];
            unflat(L, f, idx);
            fineChiNodal[f] = chi_at(idx, h);
        }
    }

    void unflat(int l, std::size_t f, int* idx) const {
        const std::size_t m1 = static_cast<std::size_t>(lv[l].m + 1);
        for (int d = 0; d < p; ++d) {
            idx[d] = static_cast<int>(f % m1);
            f /= m1;
        }
    }
    std::size_t flat(int l, const int* idx) const {
        const std::size_t m1 = static_cast<std::size_t>(lv[l].m + 1);
        std::size_t f = 0, s = 1;
        for (int d = 0; d < p; ++d) {
            f += static_cast<std::size_t>(idx[d]) * s;
            s *= m1;
        }
        return f;
    }
    bool boundary(int l, const int* idx) const {
        for (int d = 0; d < p; ++d)
            if (idx[d] == 0 || idx[d] == lv[l].m) return true;
        return false;
    }
    bool cpoint(int l, const int* idx) const {
        if (l == 0) return false;
        for (int d = 0; d < p; ++d)
            if (idx[d] % 3 != 0) return false;
        return true;
    }

    // DFS (base-3 Morton) key of a cell: per level from the coarsest, the child
    // slot t = sum_d digit_d 3^d (spacetree.cpp:408-416: axis 0 fastest).
    std::uint64_t morton(int l, const int* c) const {
        std::uint64_t key = 0;
        for (int k = l - 1; k >= 0; --k) {
            int slot = 0, mul = 1;
            for (int d = 0; d < p; ++d) {
                slot += ((c[d] / pow3(k)) % 3) * mul;
                mul *= 3;
            }
            key = key * static_cast<std::uint64_t>(pow3(p)) + static_cast<std::uint64_t>(slot);
        }
        return key;
    }

    void build_finish_order(int l) {
        Level& V = lv[l];
        std::vector<std::pair<std::uint64_t, std::uint32_t>> keys(V.n);
        for (std::size_t f = 0; f < V.n; ++f) {
            int idx[3], c[3];
            unflat(l, f, idx);
            int corner = 0;
            for (int d = 0; d < p; ++d) {
                c[d] = std::min(idx[d], V.m - 1);
                if (c[d] != idx[d]) corner |= 1 << d;
            }
            const std::uint64_t key = (l == 0 ? 0 : morton(l, c)) * 16u + static_cast<std::uint64_t>(corner);
            keys[f] = {key, static_cast<std::uint32_t>(f)};
        }
        std::sort(keys.begin(), keys.end());
        V.finishOrder.resize(V.n);
        for (std::size_t i = 0; i < V.n; ++i) V.finishOrder[i] = keys[i].second;
    }

    // Adjacent existing cells of a vertex in DFS (Morton) order, each with the
    // vertex's corner index inside it.
    int adjacent_cells(int l, const int* idx, int cells[][3], int* corners) const {
        struct C { std::uint64_t key; int c[3]; int a; };
        C tmp[8];
        int k = 0;
        for (int e = 0; e < (1 << p); ++e) {
            C x{};
            bool ok = true;
            for (int d = 0; d < p; ++d) {
                x.c[d] = idx[d] - 1 + ((e >> d) & 1);
                if (x.c[d] < 0 || x.c[d] > lv[l].m - 1) ok = false;
            }
            if (!ok) continue;
            int a = 0;
            for (int d = 0; d < p; ++d)
                if (idx[d] - x.c[d] == 1) a |= 1 << d;
            x.a = a;
            x.key = morton(l, x.c);
            tmp[k++] = x;
        }
        std::sort(tmp, tmp + k, [](const C& a, const C& b) { return a.key < b.key; });
        for (int i = 0; i < k; ++i) {
            for (int d = 0; d < p; ++d) cells[i][d] = tmp[i].c[d];
            corners[i] = tmp[i].a;
        }
        return k;
    }

    // proj/src/problems.cpp:55-68 (+ the seeded complex field)
    Cplx chi_at(const int* idx, double h) const {
        double x[3];
        for (int d = 0; d < p; ++d) x[d] = idx[d] * h;
        switch (chiKind) {
            case 0: return Cplx(0.0);
            case 1: {
                const double dd = static_cast<double>(p);
                double v = dd * M_PI * M_PI;
                for (int d = 0; d < p; ++d) v *= std::sin(M_PI * x[d]);
                return Cplx(v, 0.0);
            }
            case 2: {
                double r2 = 0.0;
                for (int d = 0; d < p; ++d) r2 += (x[d] - 0.5) * (x[d] - 0.5);
                return Cplx(r2 < 0.01 ? 1.0 : 0.0, 0.0);
            }
            default: {
                const std::int64_t m = pow3(L);
                if (rhsSphere) {
                    std::int64_t s = 0;
                    for (int d = 0; d < p; ++d) {
                        const std::int64_t t = 2 * static_cast<std::int64_t>(idx[d]) - m;
                        s += t * t;
                    }
                    if (!(25 * s < 4 * m * m)) return Cplx(0.0);
                }
                const std::uint64_t s = rhsSeed ^ pack_index(p, idx);
                return Cplx(unit_rand(s), unit_rand(s ^ 0x5bf03635ull));
            }
        }
    }

    // make_cell_kernel (kernels.cpp:7-23) for a constant-coefficient level
    void cell_scales(int l, Cplx& lapScale, Cplx& massScale) const {
        const double h = std::pow(3.0, -l);
        const Cplx hElem = h * Cplx(std::cos(theta), std::sin(theta));
        lapScale = cplx_ipow(hElem, p - 2);
        massScale = cplx_ipow(hElem, p);
    }

    // One td_add / td_bpx sweep; mirrors proj/src/cycles.cpp:102-303 level-wise.
    // Throws std::domain_error on a vanishing diagonal (kernels.cpp:102-106).
    Stats sweep(int n, bool hbMask) {
        Policy P = pol;
        P.hb = hbMask;
        if (P.bpx) P.hb = false;  // cycles.cpp:351
        // ---- top-down: touch_first (cycles.cpp:102-141), coarse to fine
        for (int l = 0; l <= L; ++l) {
            Level& V = lv[l];
            for (std::size_t f = 0; f < V.n; ++f) {
                int idx[3];
                unflat(l, f, idx);
                V.r[f] = V.rHat[f] = V.diag[f] = Cplx(0.0);
                V.chi[f] = Cplx(0.0);
                V.siNext[f] = Cplx(0.0);
                if (l > 0) {
                    int q[3], rel[3];
                    parent_stencil(l, idx, q, rel);
                    Cplx cu[8], csc[8], csi[8];
                    for (int e = 0; e < (1 << p); ++e) {
                        int pi[3];
                        for (int d = 0; d < p; ++d) pi[d] = q[d] + ((e >> d) & 1);
                        const std::size_t pf = flat(l - 1, pi);
                        cu[e] = lv[l - 1].u[pf];
                        csc[e] = lv[l - 1].sc[pf];
                        csi[e] = P.bpx ? lv[l - 1].si[pf] : Cplx(0.0);
                    }
                    V.sc[f] += prolong(csc, rel, p);
                    if (P.bpx && !cpoint(l, idx)) V.sc[f] -= prolong(csi, rel, p);
                    V.u[f] += V.sc[f] + V.sf[f];
                    V.sf[f] = Cplx(0.0);
                    V.uHat[f] = V.u[f] - prolong(cu, rel, p);
                } else {
                    V.u[f] += V.sc[f] + V.sf[f];
                    V.sf[f] = Cplx(0.0);
                    V.uHat[f] = Cplx(0.0);
                }
                if (boundary(l, idx)) {
                    V.u[f] = Cplx(0.0);
                    V.uHat[f] = Cplx(0.0);
                }
            }
        }
        // ---- bottom-up: enter_cell accumulation, then touch_last, fine to coarse
        Stats st;
        for (int l = L; l >= 0; --l) {
            Level& V = lv[l];
            Cplx lapScale, massScale;
            cell_scales(l, lapScale, massScale);
            Cplx A[8][8];
            for (int a = 0; a < R.n; ++a)
                for (int b = 0; b < R.n; ++b)
                    A[a][b] = lapScale * R.lap[a][b] - phi * massScale * R.mas[a][b];  // kernels.cpp:43-44
            // enter_cell contributions, gathered per vertex in DFS cell order
            for (std::size_t f = 0; f < V.n; ++f) {
                int idx[3], cells[8][3], corners[8];
                unflat(l, f, idx);
                const int k = adjacent_cells(l, idx, cells, corners);
                for (int i = 0; i < k; ++i) {
                    const int a = corners[i];
                    Cplx accR(0.0), accRhat(0.0);
                    for (int b = 0; b < R.n; ++b) {
                        int vb[3];
                        for (int d = 0; d < p; ++d) vb[d] = cells[i][d] + ((b >> d) & 1);
                        const std::size_t fb = flat(l, vb);
                        accR += A[a][b] * V.u[fb];
                        accRhat += A[a][b] * V.uHat[fb];
                    }
                    V.r[f] += -accR;
                    V.rHat[f] += -accRhat;
                    V.diag[f] += lapScale * R.lap[a][a] - phi * massScale * R.mas[a][a];
                    if (l == L) {  // leaf cell: consistent-mass load (kernels.cpp:69-87)
                        Cplx acc(0.0);
                        for (int b = 0; b < R.n; ++b) {
                            int vb[3];
                            for (int d = 0; d < p; ++d) vb[d] = cells[i][d] + ((b >> d) & 1);
                            acc += R.mas[a][b] * fineChiNodal[flat(l, vb)];
                        }
                        V.chi[f] += massScale * acc;
                    }
                }
            }
            // touch_last in DFS finishing order (cycles.cpp:243-303)
            const double hp = std::pow(std::pow(3.0, -l), p);
            const Cplx wRaw = omega_unmasked(P, L - l, n);
            for (std::uint32_t f : V.finishOrder) {
                int idx[3];
                unflat(l, f, idx);
                const bool bnd = boundary(l, idx), cp = cpoint(l, idx);
                if (bnd) {
                    V.u[f] = Cplx(0.0);
                    V.r[f] = Cplx(0.0);
                    V.rHat[f] = Cplx(0.0);
                } else {
                    V.r[f] = V.chi[f] + V.r[f];
                    V.rHat[f] = V.chi[f] + V.rHat[f];
                }
                V.si[f] = V.siNext[f];
                if (l == L && !bnd) {  // non-refined, non-boundary
                    ++st.updated;
                    const double mm = std::abs(V.r[f]);
                    st.maxN = std::max(st.maxN, mm);
                    st.euclid += mm * mm;
                    st.hN += hp * mm * mm;
                }
                if (l < ellMin) {
                    V.sc[f] = Cplx(0.0);
                    continue;
                }
                Cplx smooth(0.0);
                if (!bnd) {
                    if (std::abs(V.diag[f]) < 1e-300) throw std::domain_error("vanishing operator diagonal");
                    smooth = Cplx(1.0) * V.r[f] / V.diag[f];
                }
                if (P.bpx) {
                    V.sc[f] = cp ? Cplx(0.0) : wRaw * smooth;
                } else {
                    const Cplx w = (P.hb && cp) ? Cplx(0.0) : wRaw;
                    V.sc[f] = w == Cplx(0.0) ? Cplx(0.0) : w * smooth;
                }
                if (l > ellMin) {
                    if (cp) {
                        int wi[3];
                        for (int d = 0; d < p; ++d) wi[d] = idx[d] / 3;
                        const std::size_t wf = flat(l - 1, wi);
                        lv[l - 1].sf[wf] = V.sf[f] + V.sc[f];
                        if (P.bpx) lv[l - 1].siNext[wf] = wRaw * smooth;
                    }
                    int q[3], rel[3];
                    parent_stencil(l, idx, q, rel);
                    for (int e = 0; e < (1 << p); ++e) {
                        double wgt = 1.0;
                        for (int d = 0; d < p; ++d) wgt *= ((e >> d) & 1) ? kW1[rel[d]] : kW0[rel[d]];
                        if (wgt == 0.0) continue;
                        int pi[3];
                        for (int d = 0; d < p; ++d) pi[d] = q[d] + ((e >> d) & 1);
                        lv[l - 1].chi[flat(l - 1, pi)] += wgt * V.rHat[f];
                    }
                }
            }
        }
        st.euclid = std::sqrt(st.euclid);
        st.hN = std::sqrt(st.hN);
        return st;
    }

    // proj/src/spacetree.cpp:164-174
    void parent_stencil(int l, const int* idx, int* q, int* rel) const {
        const int mc = pow3(l - 1);
        for (int d = 0; d < p; ++d) {
            q[d] = std::min(idx[d] / 3, mc - 1);
            rel[d] = idx[d] - 3 * q[d];
        }
    }

    // proj/src/cycles.cpp:812-852 (set_random_initial_guess) on a regular tree
    void random_initial(std::uint64_t seed) {
        for (int l = L; l >= 0; --l) {
            Level& V = lv[l];
            for (std::size_t f = 0; f < V.n; ++f) {
                int idx[3];
                unflat(l, f, idx);
                if (boundary(l, idx)) {
                    V.u[f] = Cplx(0.0);
                } else if (l == L) {
                    const std::uint64_t base = seed ^ (static_cast<std::uint64_t>(l) << 56) ^ pack_index(p, idx);
                    V.u[f] = Cplx(unit_rand(base), unit_rand(base ^ 0x5bf03635ull));
                } else {
                    int fi[3];
                    for (int d = 0; d < p; ++d) fi[d] = idx[d] * 3;
                    V.u[f] = lv[l + 1].u[flat(l + 1, fi)];
                }
            }
        }
        reset_pipeline();
    }

    void reset_pipeline() {
        for (Level& V : lv)
            for (auto* fld : {&V.sc, &V.sf, &V.si, &V.siNext, &V.uHat}) std::fill(fld->begin(), fld->end(), Cplx(0.0));
    }
};

std::string trim(const std::string& s) {
    std::size_t a = s.find_first_not_of(" \t\r\n");
    if (a == std::string::npos) return "";
    std::size_t b = s.find_last_not_of(" \t\r\n");
    return s.substr(a, b - a + 1);
}

Cplx parse_cplx(const std::string& v) {  // runner.cpp:32-36
    const std::size_t comma = v.find(',');
    if (comma == std::string::npos) return Cplx(std::stod(v), 0.0);
    return Cplx(std::stod(v.substr(0, comma)), std::stod(v.substr(comma + 1)));
}

struct Session {
    Oracle o;
    std::string message;
    int status = 0;
    int maxSweeps = 100, hbSweeps = -1;
    double targetDrop = 1e-6;
    int normKind = 2;  // 0 max, 1 euclid, 2 h
    bool randomInit = false;
    std::uint64_t seed = 0;
    bool hbMask = false;
    // run results
    int outcome = 1, sweeps = 0;
    double firstNorm = 0.0, finalNorm = 0.0;
    std::vector<std::array<double, 6>> history;
};

void setup(Session& s, const std::string& text) {
    Oracle& o = s.o;
    std::string problem = "poisson-sin", cycle = "td-add", omega = "exponential";
    bool havePhi = false, haveOmega = false, seeded = false;
    Cplx phiVal;
    std::istringstream in(text);
    std::string line;
    while (std::getline(in, line)) {
        const std::size_t hash = line.find('#');
        if (hash != std::string::npos) line = line.substr(0, hash);
        line = trim(line);
        if (line.empty()) continue;
        const std::size_t eq = line.find('=');
        const std::string k = trim(line.substr(0, eq)), v = trim(line.substr(eq + 1));
        if (k == "problem") problem = v;
        else if (k == "dim") o.p = std::stoi(v);
        else if (k == "level") o.L = std::stoi(v);
        else if (k == "phi") { phiVal = parse_cplx(v); havePhi = true; }
        else if (k == "theta_deg") o.theta = std::stod(v) * M_PI / 180.0;
        else if (k == "cycle") cycle = v;
        else if (k == "omega") omega = v;
        else if (k == "omega_s") { o.pol.omegaS = parse_cplx(v); haveOmega = true; }
        else if (k == "lgrid") o.pol.lGrid = std::stoi(v);
        else if (k == "hb") s.hbMask = (v == "1" || v == "true" || v == "on");
        else if (k == "two_phase") o.pol.twoPhase = (v == "1" || v == "true" || v == "on");
        else if (k == "ell_min") o.ellMin = std::stoi(v);
        else if (k == "max_sweeps") s.maxSweeps = std::stoi(v);
        else if (k == "target_drop") s.targetDrop = std::stod(v);
        else if (k == "norm") s.normKind = v == "max" ? 0 : v == "euclid" ? 1 : 2;
        else if (k == "initial") s.randomInit = (v == "random");
        else if (k == "seed") s.seed = std::stoull(v);
        else if (k == "rhs") seeded = (v == "seeded");
        else if (k == "rhs_seed") o.rhsSeed = std::stoull(v);
        else if (k == "rhs_mask") o.rhsSphere = (v == "sphere");
        else if (k == "hb_sweeps") s.hbSweeps = std::stoi(v);
        else if (k == "channels" && v != "1") throw std::invalid_argument("oracle: one channel only");
        else if (k == "precision" || k == "gpus" || k == "max_vertices" || k == "out" || k == "channels") {}
        else throw std::invalid_argument("oracle: unsupported key '" + k + "'");
    }
    if (o.p < 1 || o.p > 3) throw std::invalid_argument("oracle: 1 <= dim <= 3");
    if (problem == "poisson-sin") { o.chiKind = 1; o.phi = 0.0; }
    else if (problem == "helmholtz-sin") { o.chiKind = 1; o.phi = Cplx(45.0 * 45.0, 0.0); }
    else if (problem == "helmholtz-ball") { o.chiKind = 2; o.phi = Cplx(-1000.0, 0.0); }
    else throw std::invalid_argument("oracle: unsupported problem '" + problem + "'");
    if (havePhi) o.phi = phiVal;
    if (seeded) o.chiKind = 3;
    if (!haveOmega) o.pol.omegaS = Cplx(0.8, 0.0);
    o.pol.bpx = (cycle == "td-bpx");
    if (cycle != "td-add" && cycle != "td-bpx") throw std::invalid_argument("oracle: td-add / td-bpx only");
    o.pol.kind = omega == "jacobi-only" ? Kind::JacobiOnly
                 : omega == "undamped"  ? Kind::Undamped
                 : omega == "lgrid"     ? Kind::LGrid
                 : omega == "transition" ? Kind::Transition
                                         : Kind::Exponential;
    o.init();
    if (s.randomInit) o.random_initial(s.seed);
}

// proj/src/runner.cpp:268-366 for a fixed regular grid
void run_loop(Session& s) {
    Oracle& o = s.o;
    double referenceCost = 1.0;
    for (int d = 0; d < o.p; ++d) referenceCost *= static_cast<double>(pow3(o.L) - 1);
    referenceCost = std::max(1.0, referenceCost);
    double cumulative = 0.0, minNorm = 0.0;
    bool haveMin = false;
    for (int n = 1; n <= s.maxSweeps; ++n) {
        Stats st;
        try {
            st = o.sweep(n, s.hbSweeps >= 0 ? n <= s.hbSweeps : s.hbMask);
        } catch (const std::domain_error& e) {
            s.sweeps = n;
            s.outcome = 2;
            s.message = e.what();
            return;
        }
        s.sweeps = n;
        cumulative += static_cast<double>(st.updated);
        const double current = s.normKind == 0 ? st.maxN : s.normKind == 1 ? st.euclid : st.hN;
        s.history.push_back({static_cast<double>(n), cumulative / referenceCost, static_cast<double>(st.updated),
                             st.maxN, st.euclid, st.hN});
        if (n == 1) s.firstNorm = current;
        s.finalNorm = current;
        if (!std::isfinite(current)) {
            s.outcome = 2;
            return;
        }
        if (!haveMin || current < minNorm) {
            minNorm = current;
            haveMin = true;
        }
        if (current > minNorm * 1e6 && n > 1) {
            s.outcome = 2;
            return;
        }
        if (s.firstNorm < 1e-300 || current <= s.targetDrop * s.firstNorm) {
            s.outcome = 0;
            return;
        }
        if (n == s.maxSweeps) s.outcome = 1;
    }
}

std::vector<Cplx>* field_ptr(Oracle& o, int l, const char* f) {
    Level& V = o.lv.at(static_cast<std::size_t>(l));
    if (!std::strcmp(f, "u")) return &V.u;
    if (!std::strcmp(f, "chi")) return &V.chi;
    if (!std::strcmp(f, "r")) return &V.r;
    if (!std::strcmp(f, "rhat")) return &V.rHat;
    if (!std::strcmp(f, "uhat")) return &V.uHat;
    if (!std::strcmp(f, "diag")) return &V.diag;
    if (!std::strcmp(f, "sc")) return &V.sc;
    if (!std::strcmp(f, "sf")) return &V.sf;
    if (!std::strcmp(f, "si")) return &V.si;
    if (!std::strcmp(f, "sinext")) return &V.siNext;
    return nullptr;
}

}  // namespace

extern "C" {

void* tmo_new(const char* text) {
    auto* s = new Session();
    try {
        setup(*s, text ? text : "");
    } catch (const std::exception& e) {
        s->status = 1;
        s->message = e.what();
    }
    return s;
}
void tmo_free(void* h) { delete static_cast<Session*>(h); }
int tmo_status(void* h) { return static_cast<Session*>(h)->status; }
const char* tmo_message(void* h) { return static_cast<Session*>(h)->message.c_str(); }

int tmo_sweep(void* h, int n, double* out) {
    auto* s = static_cast<Session*>(h);
    try {
        const Stats st = s->o.sweep(n, s->hbSweeps >= 0 ? n <= s->hbSweeps : s->hbMask);
        if (out) {
            out[0] = st.maxN;
            out[1] = st.euclid;
            out[2] = st.hN;
            out[3] = static_cast<double>(st.updated);
            out[4] = 0.0;
        }
        return 0;
    } catch (const std::exception& e) {
        s->message = e.what();
        return 3;
    }
}

int tmo_run(void* h) {
    auto* s = static_cast<Session*>(h);
    if (s->status) return s->status;
    run_loop(*s);
    return 0;
}
int tmo_outcome(void* h) { return static_cast<Session*>(h)->outcome; }
int tmo_sweeps(void* h) { return static_cast<Session*>(h)->sweeps; }
int tmo_history_rows(void* h) { return static_cast<int>(static_cast<Session*>(h)->history.size()); }
void tmo_history_row(void* h, int i, double* out) {
    const auto& r = static_cast<Session*>(h)->history.at(static_cast<std::size_t>(i));
    for (int k = 0; k < 6; ++k) out[k] = r[k];
}

// CSV text exactly as proj/src/runner.cpp:247-251,318-329 writes it (one channel).
const char* tmo_csv(void* h) {
    auto* s = static_cast<Session*>(h);
    static thread_local std::string out;
    out = "sweep,workUnits,vertexCount,maxNorm,euclid,hNorm\n";
    char buf[256];
    for (const auto& r : s->history) {
        std::snprintf(buf, sizeof buf, "%d,%.17g,%zu,%.17g,%.17g,%.17g\n", static_cast<int>(r[0]), r[1],
                      static_cast<std::size_t>(r[2]), r[3], r[4], r[5]);
        out += buf;
    }
    return out.c_str();
}

// FNV-1a over (re+0.0, im+0.0) bit patterns, lattice order (as refdriver.cpp).
unsigned long long tmo_field_hash(void* h, int level, const char* name) {
    auto* v = field_ptr(static_cast<Session*>(h)->o, level, name);
    if (!v) return 0;
    std::uint64_t hsh = 1469598103934665603ull;
    for (const Cplx& z : *v) {
        for (double x : {z.real() + 0.0, z.imag() + 0.0}) {
            std::uint64_t bits;
            std::memcpy(&bits, &x, 8);
            for (int b = 0; b < 8; ++b) {
                hsh ^= (bits >> (8 * b)) & 0xffu;
                hsh *= 1099511628211ull;
            }
        }
    }
    return hsh;
}

long long tmo_lattice_size(void* h, int level) {
    return static_cast<long long>(static_cast<Session*>(h)->o.lv.at(static_cast<std::size_t>(level)).n);
}

int tmo_field(void* h, int level, const char* name, double* out) {
    auto* v = field_ptr(static_cast<Session*>(h)->o, level, name);
    if (!v) return 1;
    for (std::size_t i = 0; i < v->size(); ++i) {
        out[2 * i] = (*v)[i].real();
        out[2 * i + 1] = (*v)[i].imag();
    }
    return 0;
}

// proj/tests/test_util.hpp:48-65 on the regular lattice.
void tmo_set_fine_interior_u(void* h, const double* u) {
    Oracle& o = static_cast<Session*>(h)->o;
    const int L = o.L;
    const int m = o.lv[L].m - 1;
    for (std::size_t f = 0; f < o.lv[L].n; ++f) {
        int idx[3];
        o.unflat(L, f, idx);
        if (o.boundary(L, idx)) continue;
        std::size_t fl = 0, st = 1;
        for (int d = 0; d < o.p; ++d) {
            fl += static_cast<std::size_t>(idx[d] - 1) * st;
            st *= static_cast<std::size_t>(m);
        }
        o.lv[L].u[f] = Cplx(u[2 * fl], u[2 * fl + 1]);
    }
    for (int l = L - 1; l >= 0; --l)
        for (std::size_t f = 0; f < o.lv[l].n; ++f) {
            int idx[3], fi[3];
            o.unflat(l, f, idx);
            if (o.boundary(l, idx)) continue;
            for (int d = 0; d < o.p; ++d) fi[d] = idx[d] * 3;
            o.lv[l].u[f] = o.lv[l + 1].u[o.flat(l + 1, fi)];
        }
    o.reset_pipeline();
}

// omega table entry exactly as the reference computes it (cycles.cpp:17-31)
void tmo_omega(int kind, double wr, double wi, int lgrid, int twoPhase, int succ, int n, double* out) {
    Policy pol;
    pol.kind = static_cast<Kind>(kind);
    pol.omegaS = Cplx(wr, wi);
    pol.lGrid = lgrid;
    pol.twoPhase = twoPhase != 0;
    const Cplx w = omega_unmasked(pol, succ, n);
    out[0] = w.real();
    out[1] = w.imag();
}

// x / y with libgcc's __divdc3, the reference's complex division (used to pin
// the device restatement of the same algorithm).
void tmo_cdiv(const double* x, const double* y, double* out, long long n) {
    for (long long i = 0; i < n; ++i) {
        const Cplx q = Cplx(x[2 * i], x[2 * i + 1]) / Cplx(y[2 * i], y[2 * i + 1]);
        out[2 * i] = q.real();
        out[2 * i + 1] = q.imag();
    }
}

}  // extern "C"
