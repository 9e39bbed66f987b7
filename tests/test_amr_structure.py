"""Static adaptive tree structure (CPU, no GPU): the host-side classification
of the B200 path (amr::build_sphere_tree, exported as tmg_sphere_tree) against
the reference's own Spacetree after refine_cell + classify()
(spacetree.cpp:272-329, 438-494) -- existence, hanging, refined, boundary,
cPoint, succ per vertex and exists/refined per cell on every level."""
import numpy as np
import pytest


@pytest.mark.parametrize("dim,base,k", [(1, 2, 2), (2, 2, 2), (2, 1, 3), (2, 3, 2), (3, 1, 2), (3, 2, 2)])
def test_sphere_tree_matches_reference(tmg, ref_mod, dim, base, k):
    s = ref_mod.RefSession(dict(problem="helmholtz-sin", dim=dim, level=base, sphere_levels=k, phi="400,200",
                                max_vertices=10 ** 8))
    assert s.status == 0, s.message
    hanging = 0
    for lvl in range(base + k + 1):
        fr, sr, cr = s.flags(lvl)
        fm, sm, cm, fc = tmg.sphere_tree(dim, base, k, lvl)
        assert np.array_equal(fr, fm), lvl
        assert np.array_equal(sr, sm), lvl
        assert np.array_equal(cr, cm), lvl
        exists = (fm & 1) == 1
        assert np.all((fc != 255) == exists)  # every vertex finishes in one of its cells
        hanging += int(((fm & 3) == 3).sum())
    leaf = sum(int((((f := tmg.sphere_tree(dim, base, k, l)[0]) & 1) == 1).__and__((f & (2 | 4 | 8)) == 0).sum())
               for l in range(base + k + 1))
    assert leaf == s.interior_count()
    if (dim, base, k) == (3, 2, 2):  # 15,160 DoF, 4,648 hanging vertices
        assert (leaf, hanging) == (15160, 4648)


def test_cfg4_structure_counts(tmg):
    """cfg4 (3D, base 4, two sphere levels): SURVEY §8 sizes (about 504k level-5
    and 12.9M level-6 vertices), counted from the host structure alone."""
    counts = []
    for lvl in (5, 6):
        f = tmg.sphere_tree(3, 4, 2, lvl)[0]
        counts.append(int(((f & 1) == 1).sum()))
    assert 4.5e5 < counts[0] < 5.5e5 and 1.2e7 < counts[1] < 1.35e7, counts
