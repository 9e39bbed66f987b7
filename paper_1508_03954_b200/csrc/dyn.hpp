// Dynamic adaptivity: the structural side of an
// h_max / h_min run -- the reference's feature-based marks applied inside the
// sweep (cycles.cpp:174-180 refine on descent, :222-241 erase on
// backtracking; spacetree.cpp:245-365), and the classification afterwards.
//
// The numerics of a sweep run on the device as level passes (amr.cu).  What a
// level pass cannot see is WHEN, in the reference's depth-first traversal, a
// vertex was touched or finished relative to the structural edits of that
// same traversal; that decides its role (touch-first, create-hanging, freshly
// created with u = P u), which adjacent cells it has accumulated, where (and
// how often) it finishes, and with which refreshed classification.  DynTree
// replays the traversal on the host over the cell structure only -- no
// floating point -- and emits per-vertex tables that the device passes
// consume.  The structure lives in full-lattice byte arrays per level.
#pragma once

#include <cstdint>
#include <vector>

namespace tmg {
namespace dyn {

// persistent cell bits
enum : unsigned char { kCE = 1, kCR = 2, kRM = 4, kEM = 8 };
// persistent vertex bits (the amr::k* classification encoding)
enum : unsigned char { kVE = 1, kVH = 2, kVR = 4, kVB = 8, kVC = 16 };
// per-sweep vertex role bits (sweep tables)
enum : unsigned char {
    kSE = 1,        // touched (or created) in this sweep
    kSH = 2,        // hanging at touch time: create_hanging / destroy_hanging
    kSR = 4,        // refined at its touch-last finish (refreshed classification)
    kSB = 8,        // boundary
    kSC = 16,       // cPoint
    kSCreated = 64, // created by refine_cell in this sweep: u = P u_parent, all else zero, no touch-first
    kSSpecial = 128 // accumulation or finish pattern differs from "every adjacent cell, one finish"
};

struct Level {
    int m = 1;          // 3^l cells per axis
    int n1 = 2;         // 3^l + 1 lattice points per axis
    long long n = 0;    // n1^p
    long long stride[3] = {1, 1, 1};
    long long off[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // lattice offset of corner e: sum_d bit(e, d) stride[d]
    // persistent structure (cells indexed by their lower corner)
    std::vector<unsigned char> cell, vtx;
    std::vector<signed char> succ;
    // traversal bookkeeping (spacetree.cpp:367-436)
    std::vector<std::uint32_t> epoch, entered;
    std::vector<unsigned char> done, expected;
    // classification inputs changed since the vertex was last classified
    std::vector<unsigned char> stale;
    std::vector<long long> staleList;
    // what the last sweep touched: its vertices and cells (sweep tables), and the
    // vertices / cells whose persistent structure it may have changed (with the
    // vertex byte before the sweep) -- so uploads and resets are proportional to it
    std::vector<long long> sweepList, cellList, vtxNoted, cellNoted;
    std::vector<unsigned char> vtxOld, noted;  // noted: 1 vertex, 2 cell
    // sweep tables
    std::vector<unsigned char> sflag, scell, sestar, sfmask, sskip;
    std::vector<signed char> ssucc;
};

struct SweepCounts {
    int refinedCells = 0, erasedCells = 0;
    long long updatedFineVertices = 0;  // touch_last finishes on unrefined interior vertices
    long long specialVertices = 0;
};

class DynTree {
  public:
    // build_regular(start) (spacetree.cpp:48-76); levels up to maxLevel are allocated
    DynTree(int dim, int start, int maxLevel, int ellMin, double hMinRefine, std::size_t maxVertices);

    // One traversal with applyMarks (the structural half of td_add / td_bpx):
    // fills the sweep tables of levels 0..depth() (as of the end of the sweep),
    // edits the structure, then classify() if it changed.
    SweepCounts sweep();

    int dim() const { return p_; }
    int depth() const { return depth_; }
    int max_level() const { return static_cast<int>(lv_.size()) - 1; }
    Level& level(int l) { return lv_[l]; }
    const Level& level(int l) const { return lv_[l]; }
    std::size_t total_vertices() const { return total_; }
    long long interior_fine_vertex_count() const;  // spacetree.cpp:225-231

    // persistent structure queries / edits (marks come from the device mark pass)
    void classify();  // spacetree.cpp:491-494
    void clear_marks();

    long long flat(int l, const int* g) const;
    void unflat(int l, long long f, int* g) const;

  private:
    void visit(int l, const int* c);
    void touch(int l, long long f, const int* v);
    void finish(int l, long long f, const int* v, int corner);
    int adjacent_cells(int l, long long f, const int* v, int* refinedAdj) const;
    void refine(int l, const int* c);
    void erase(int l, const int* c);
    bool refresh(int l, const int* v);  // true if the classification changed
    void mark_stale(int l, const int* v);
    void stale_parents(int l, const int* v);  // coarser vertices whose succ scan sees v
    void classify_stale();
    void note_vtx(Level& L, long long f);
    void note_cell(Level& L, long long f);

  public:
    // forget the noted changes (after the caller consumed them)
    void clear_notes();

  private:
    int existing_adjacent(int l, const int* v) const;
    int indomain_adjacent(int l, const int* v) const;
    bool has_cell(int l, const int* c) const;
    void check_capacity(std::size_t add) const;
    void ensure_level(int l);

    int p_, ellMin_, depth_;
    double hMin_;
    std::size_t maxVertices_, total_ = 0;
    std::uint32_t epoch_ = 0;
    bool dirty_ = false;
    SweepCounts counts_;
    std::vector<Level> lv_;
};

}  // namespace dyn
}  // namespace tmg
