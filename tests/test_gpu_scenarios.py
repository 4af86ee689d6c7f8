"""The reference's own scenario configs (configs/*.cfg) run through the GPU
path with paper_2507_09435_b200.run_scenario, compared with the reference's
committed outputs (/root/reference/proj/out/*, packed into
tests/golden/reference_out.npz)."""
import os

import numpy as np
import pytest

import golden_util as gu

pytestmark = pytest.mark.gpu
CFG = os.path.join(gu.GOLDEN, "configs")


def ref(name):
    return np.load(os.path.join(gu.GOLDEN, "reference_out.npz"))[name]


def load_csv(path):
    return np.loadtxt(path, delimiter=",", skiprows=1, ndmin=2)


@pytest.mark.parametrize("case", ["bar_elastic", "bar_elastoplastic"])
def test_bar_scenario_matches_reference_outputs(case, tmp_path):
    import paper_2507_09435_b200 as impm

    rep = impm.run_scenario(os.path.join(CFG, case + ".cfg"), False, [f"output.dir={tmp_path}"])
    assert rep["steps"] == 40
    got, want = load_csv(tmp_path / "particles.csv"), ref(case + "__particles")
    scale = np.maximum(np.abs(want).max(axis=0), 1.0)
    assert (np.abs(got - want).max(axis=0) / scale).max() <= 1e-7
    its_got = np.bincount(load_csv(tmp_path / "iterations.csv")[:, 0].astype(int))
    its_ref = np.bincount(ref(case + "__iterations")[:, 0].astype(int))
    np.testing.assert_array_equal(its_got, its_ref)  # identical Newton counts, J2 included
    assert os.path.exists(tmp_path / "summary.json")


def test_bar_scenario_checks_pass(tmp_path):
    import paper_2507_09435_b200 as impm

    rep = impm.run_scenario(os.path.join(CFG, "bar_elastic.cfg"), True, [f"output.dir={tmp_path}"])
    failed = [c for c in rep["checks"] if not c["pass"]]
    assert not failed, failed


def test_smoke3d_scenario(tmp_path):
    import paper_2507_09435_b200 as impm

    impm.run_scenario(os.path.join(CFG, "smoke3d.cfg"), True, [f"output.dir={tmp_path}"])
    got, want = load_csv(tmp_path / "summary.csv"), ref("smoke3d__summary")
    assert got[0, 0] == want[0, 0] == 300 and got[0, 1] == want[0, 1] == 3


def test_consolidation_scenario_early_window(tmp_path):
    import paper_2507_09435_b200 as impm

    impm.run_scenario(os.path.join(CFG, "consolidation.cfg"), False,
                      [f"output.dir={tmp_path}", "schedule.Tv_checkpoints=0.05", "schedule.Tv_end=0.05"])
    got, want = load_csv(tmp_path / "settlement.csv"), ref("consolidation__settlement")
    n = got.shape[0]
    assert n > 10
    assert np.abs(got[:, 0] - want[:n, 0]).max() <= 1e-9 * want[:n, 0].max()
    assert np.abs(got[:, 2] - want[:n, 2]).max() <= 1e-6 * np.abs(want[:n, 2]).max()


def test_cantilever_scenario_coarse_level(tmp_path):
    import paper_2507_09435_b200 as impm

    impm.run_scenario(os.path.join(CFG, "cantilever.cfg"), False, [f"output.dir={tmp_path}", "geometry.h_levels=4"])
    got, want = load_csv(tmp_path / "tip.csv"), ref("cantilever__tip")
    want = want[want[:, 0] == 4.0]
    assert got.shape == want.shape
    assert np.abs(got[:, 3] - want[:, 3]).max() <= 1e-7 * np.abs(want[:, 3]).max()


def test_inverse_scenario_matches_reference(tmp_path):
    import paper_2507_09435_b200 as impm

    rep = impm.run_scenario(os.path.join(CFG, "inverse.cfg"), False, [f"output.dir={tmp_path}"])
    got, want = load_csv(tmp_path / "reference.csv"), ref("inverse__reference")
    assert np.abs(got - want).max() <= 1e-7 * np.abs(want).max()
    opt_got = load_csv(tmp_path / "optimization.csv")
    opt_ref = ref("inverse__optimization")  # iteration,E,loss,gradient (no theta column; stale)
    assert opt_got.shape[0] == opt_ref.shape[0]
    assert np.abs(opt_got[:, 2] - opt_ref[:, 1]).max() <= 1e-6 * opt_ref[:, 1].max()
