"""The CPU oracle against the reference's own outputs (golden fixtures) — pins the oracle."""
import numpy as np
import pytest

from golden_cases import params_obj, pipeline_cases, stage_cases

CASES = pipeline_cases()


@pytest.mark.parametrize("name", sorted(CASES))
def test_pipeline_case(oracle, name):
    c = CASES[name]
    p = params_obj(c["params"])
    for i, f in enumerate(c["frames"]):
        maps = {}
        out = oracle.dehaze_frame(f, p, maps)
        assert np.array_equal(out, c["out"][i]), name
        assert np.array_equal(maps["airlight"], c["airlight"][i])
        assert np.array_equal(maps["dark"], c["dark"][i])
        assert np.array_equal(maps["transmission_coarse"], c["transmission_coarse"][i])
        assert np.array_equal(maps["transmission"], c["transmission"][i])


def test_stage_functions(oracle):
    s = stage_cases()
    m, img, g, t = s["m"], s["img"], s["g"], s["t"]
    for r in (0, 1, 3, 9):
        assert np.array_equal(oracle.min_filter(m, r), s[f"min_filter_r{r}"])
        assert np.array_equal(oracle.box_filter(m, r), s[f"box_filter_r{r}"])
    assert np.array_equal(oracle.guided_filter(m, g, 2, 1e-3), s["guided_r2"])
    assert np.array_equal(oracle.guided_filter(m, g, 5, 1e-2), s["guided_r5"])
    assert np.array_equal(oracle.channel_min(img), s["channel_min"])
    assert np.array_equal(oracle.dark_channel(img, 2), s["dark_r2"])
    a = oracle.estimate_airlight(img, oracle.dark_channel(img, 2), 0.05, 0.8)
    assert np.array_equal(a, s["airlight"])
    assert np.array_equal(oracle.transmission_from_channel_min(oracle.channel_min(img), a, 0.5, 0.05),
                          s["transmission"])
    assert np.array_equal(oracle.recover_radiance(img, a, t), s["recover"])
    assert np.array_equal(oracle.gamma_correct(img, 1.2), s["gamma"])
    assert np.array_equal(oracle.gray_world_balance(img), s["balance"])
    assert np.array_equal(oracle.to_grayscale(img), s["gray"])
    assert np.array_equal(oracle.resize_bilinear(img, 9, 7), s["resize_down"])
    assert np.array_equal(oracle.resize_bilinear(img, 30, 25), s["resize_up"])


def test_min_filter_matches_naive(oracle):
    rng = np.random.default_rng(10)
    for _ in range(40):
        m = rng.random((int(rng.integers(1, 20)), int(rng.integers(1, 20))))
        r = int(rng.integers(0, 8))
        assert np.array_equal(oracle.min_filter(m, r), oracle.min_filter_naive(m, r))


def test_selection_tie_rule(oracle):
    # estimation test_ties_break_by_linear_index: K = 2 among three tied pixels -> 1 and 4
    dark = np.array([[0.0, 0.7, 0.0, 0.0], [0.7, 0.0, 0.0, 0.7]])
    assert oracle.select_airlight_pixels(dark, 0.25).tolist() == [1, 4]
    img = np.zeros((2, 4, 3))
    img[0, 1] = 0.9
    img[1, 0] = 0.5
    img[1, 3] = 0.3
    assert np.allclose(oracle.estimate_airlight(img, dark, 0.25, 1.0), (0.9 + 0.5) / 2, atol=1e-12)
