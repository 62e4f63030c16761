"""The seeded generator: deterministic, per-unit regenerable, shaped like the configs."""
import numpy as np

from workload import CONFIGS, make_workload, decode_bytes


def test_per_unit_regeneration_matches_full_draw():
    cfg = CONFIGS["qwen_b1_r32"].with_(n_vis=200, n_text=9)
    full = make_workload(cfg)
    part = make_workload(cfg, units=[2, 0])
    for k in ("K", "V", "Ktext", "Vtext", "Qw", "q"):
        np.testing.assert_array_equal(part[k].bits[0], full[k].bits[2])
        np.testing.assert_array_equal(part[k].bits[1], full[k].bits[0])


def test_shapes_and_dtypes():
    cfg = CONFIGS["toy"]
    w = make_workload(cfg)
    assert w["K"].shape == (1, 64, 16) and w["K"].bits.dtype == np.uint16
    assert w["Qw"].shape == (1, 1, 32, 16) and w["q"].shape == (1, 1, 16)
    w32 = make_workload(cfg.with_(dtype="f32"))
    assert w32["K"].bits.dtype == np.float32
    # bf16 bytes are the RNE rounding of the same float32 draws
    np.testing.assert_allclose(w["K"].f32(), w32["K"].f32(), rtol=2 ** -8)


def test_token_pruned_config_keeps_subset():
    cfg = CONFIGS["joint_b64"].with_(batch=1, h_kv=1)
    w = make_workload(cfg)
    assert w["K"].shape == (1, 864, 128)


def test_gap_distribution_has_planted_gap():
    from oracle import oracle as orc
    cfg = CONFIGS["llava_b1"].with_(batch=1, h_kv=1, n_vis=512, n_text=0)
    w = make_workload(cfg, dist="gap")
    cal = orc.calibrate(w["K"].f64(), None, cfg.rank)
    lam = np.sort(cal["lam"][0])[::-1]
    assert lam[cfg.rank - 1] / lam[cfg.rank] > 50


def test_decode_bytes_llava_b32():
    # 1028.9 MB per layer for LLaVA b32
    assert abs(decode_bytes(CONFIGS["llava_b32"]) / 1e6 - 1028.9) < 0.5
