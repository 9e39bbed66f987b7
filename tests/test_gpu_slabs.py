"""z-slab execution on one GPU with K slabs of one process
(the same code path as the NCCL ranks and as `gpus = K` on K GPUs; transfers
as device copies): every slab allocates only its planes of levels L and L-1,
and the fine-level iterate must be bitwise identical to the unsharded run for
every slab count, the norms equal up to the summation order of the slab
partials.  Includes the headline size (729^3, K = 8) and FMG onto slabs
through treemg_run's `gpus` key (cfg5's schedule 3 -> 6)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _pol(tmg, kind):
    return tmg.Policy("exponential", 0.6) if kind == "td-add" else tmg.Policy("undamped", 0.5, bpx=True)


@pytest.mark.parametrize("levels,phi", [(4, 400 + 200j), (5, 400 + 200j)])
@pytest.mark.parametrize("kind", ["td-add", "td-bpx"])
@pytest.mark.parametrize("k", [2, 3, 4, 8])
def test_virtual_slabs_bitwise_equal_single(tmg, levels, phi, kind, k):
    pol = _pol(tmg, kind)
    one = tmg.Hierarchy(3, levels, phi=phi, chi="seeded", precision="fast", max_vertices=10 ** 10)
    sl = tmg.Slabs(levels, phi, local=k)
    for n in range(1, 7):
        a = one.td_bpx(pol, n) if pol.bpx else one.td_add(pol, n)
        b = sl.cycle(pol, n)
        assert abs(a.h_norm - b.h_norm) <= 1e-13 * a.h_norm, n
        assert abs(a.max_norm - b.max_norm) <= 1e-15 * a.max_norm, n
    u1 = one.field(levels, "u")
    uk = sl.fine_u()
    assert np.array_equal(u1, uk)
    for level in range(1, levels + 1):  # the gathered fields of every level (sc: incl. the sharded level L-1)
        for f in ("u", "sc"):
            assert np.array_equal(one.field(level, f), sl.field(level, f)), (level, f)


def test_virtual_slabs_headline_729_k8(tmg):
    """The headline workload (729^3, k = 80) as 8 slabs: bitwise equal fine u,
    norms to summation order (the size where arrays pass 2^31 bytes and each
    slab holds ~1/8 of levels 6 and 5)."""
    pol = _pol(tmg, "td-add")
    phi = 6400 + 3200j
    one = tmg.Hierarchy(3, 6, phi=phi, chi="seeded", precision="fast", max_vertices=10 ** 10)
    na = [one.td_add(pol, n) for n in range(1, 4)]
    u1 = one.field(6, "u")
    one.close()
    sl = tmg.Slabs(6, phi, local=8)
    nb = [sl.cycle(pol, n) for n in range(1, 4)]
    for a, b in zip(na, nb):
        assert abs(a.h_norm - b.h_norm) <= 1e-13 * a.h_norm
    assert np.array_equal(u1, sl.fine_u())


FMG = dict(problem="helmholtz-sin", dim=3, fmg_from=3, phi="6400,3200", cycle="td-add", omega="exponential",
           omega_s=0.6, target_drop=1e-8, rhs="seeded", rhs_seed=12345, precision="fast", fingerprint=1,
           max_vertices=10 ** 10)


@pytest.mark.parametrize("level,cap,gpus", [(5, 4, 4), (6, 2, 8)])
def test_fmg_onto_slabs_bitwise_equal_single(tmg, level, cap, gpus):
    """treemg_run, gpus = K: FMG 3 -> level on one GPU's hierarchy, the last
    unfolding onto K slabs (SlabGroup::unfold_from); the final u / sc bitwise
    equal to gpus = 1, every CSV row equal up to the slab norm order."""
    cfg = dict(FMG, level=level, fmg_stage_cap=cap, max_sweeps=200)
    a = tmg.run(cfg)
    b = tmg.run(dict(cfg, gpus=gpus))
    assert (a.outcome, a.sweeps) == (b.outcome, b.sweeps)
    assert np.array_equal(a.history[:, :3], b.history[:, :3])
    np.testing.assert_allclose(b.history[:, 3:], a.history[:, 3:], rtol=1e-13, atol=0)
    assert a.u_hash == b.u_hash and a.sc_hash == b.sc_hash


def test_gpus_run_grid_dump_identical(tmg, tmp_path):
    """`gpus = 3` without FMG: the .grid dump (every level's u, gathered) equals gpus = 1 byte for byte."""
    cfg = dict(problem="helmholtz-sin", dim=3, level=3, phi="400,200", rhs="seeded", precision="fast", max_sweeps=5,
               target_drop=1e-30)
    tmg.run(cfg, out_prefix=str(tmp_path / "one"))
    tmg.run(dict(cfg, gpus=3), out_prefix=str(tmp_path / "three"))
    assert (tmp_path / "one.grid").read_text() == (tmp_path / "three.grid").read_text()


def test_gpus_unsupported_fail_loudly(tmg):
    for cfg in (dict(dim=2, level=4), dict(dim=3, level=3, precision="exact"),
                dict(dim=3, level=3, precision="fast-complex64")):
        with pytest.raises(tmg.TreemgError) as e:
            tmg.run(dict(dict(problem="helmholtz-sin", phi="100,50", precision="fast", max_sweeps=2), **cfg, gpus=2))
        assert e.value.status == 1


def test_nccl_unique_id(tmg):
    uid = tmg.nccl_unique_id()
    assert len(uid) == 128 and any(uid)
