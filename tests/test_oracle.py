"""Pin the oracle (oracle/) to the reference before trusting it as the checker.

Every case compares against fixtures produced by the reference package itself
(tests/golden/make_golden.py imports /root/reference/pkg/src) or against the
known answers written in the reference's tests.  CPU only.
"""

import numpy as np
import pytest

Z1 = (1.0, 0.0, 0.0, 0.0, 0.0, 0.0)
C3F = (1.0, 0.0, 0.5, 0.0, 0.25, 0.0)


def bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


def test_random_fill_known_answers(O, kat):
    # random(0) at (0,0,0) is exactly 0.0; coordinates wrap as uint64
    assert O.lib().or_random_value(0, 0, 0, 0) == 0.0
    for key, b in kat["random0_bits"].items():
        z, y, x = map(int, key.split(","))
        assert np.float64(O.lib().or_random_value(z, y, x, 0)).view(np.uint64) == b, key
        v = O.random_values(np.array([z]), np.array([y]), np.array([x]), 0)[0]
        assert np.float64(v).view(np.uint64) == b, key
    assert np.float64(O.lib().or_random_value(0, 0, 0, 42)).view(np.uint64) == kat["random42_bits_0_0_0"]


def test_constants(kat):
    assert np.float64(1.0 / 6.0).view(np.uint64) == kat["one_sixth_bits"] == 0x3FC5555555555555
    assert np.float32(1.0 / 6.0).view(np.uint32) == kat["one_sixth_f32_bits"] == 0x3E2AAAAB


def test_stencil_point_examples_and_order(O, kat):
    # reference test_kernel.py:11-15 and the summation-order pin :164-170
    sp = O.lib().or_stencil_point
    assert sp(5.0, 5.0, 5.0, 5.0, 5.0, 5.0) == 5.0
    assert sp(2.0, 4.0, 2.0, 4.0, 2.0, 4.0) == 3.0
    assert sp(1.0, 2.0, 3.0, 4.0, 0.0, 5.0) == 15.0 / 6.0
    args = kat["stencil_point_order"]["args"]
    assert np.float64(sp(*args)).view(np.uint64) == kat["stencil_point_order"]["bits"]


def test_hotplate_golden(O, ref_fields):
    f = O.initial_field((4, 4, 4), O.BoxPattern("hotplate"))
    got = O.interior(O.sweeps(f, 1))
    expected = np.zeros((4, 4, 4))
    expected[:, :, 0] = 1.0 / 6.0
    assert np.array_equal(bits(got), bits(expected))
    assert np.array_equal(bits(got), bits(ref_fields["hotplate4_l1"]))


def test_trajectory_numpy_and_c(O, ref_fields):
    traj = ref_fields["r11_16_traj"]
    p = O.BoxPattern("random", seed=11)
    f = O.initial_field((16, 16, 16), p)
    g = O.CGrid((16, 16, 16), p)
    for lv in range(9):
        assert np.array_equal(bits(O.interior(f)), bits(traj[lv])), lv
        assert np.array_equal(bits(g.interior()), bits(traj[lv])), lv
        f = O.sweeps(f, 1)
        g.sweeps(1)


@pytest.mark.parametrize("name,shape,kind,seed,levels", [
    ("r2_9x7x5_l7", (5, 7, 9), "random", 2, 7),
    ("r3_1x3x2_l3", (2, 3, 1), "random", 3, 3),
    ("linear_6_l8", (6, 6, 6), "linear", 0, 8),
    ("r11_24_pipe_u16", (24, 24, 24), "random", 11, 16),
])
def test_c_oracle_vs_reference_fields(O, ref_fields, name, shape, kind, seed, levels):
    g = O.CGrid(shape, O.BoxPattern(kind, seed=seed))
    g.sweeps(levels)
    assert np.array_equal(bits(g.interior()), bits(ref_fields[name]))


def test_faced_patterns(O, ref_fields):
    g = O.CGrid((20, 18, 33), O.BoxPattern("random", seed=0, faces=Z1, global_shape=(20, 18, 33)))
    g.sweeps(12)
    assert np.array_equal(bits(g.interior()), bits(ref_fields["c1like_33x18x20_l12"]))
    p3 = O.BoxPattern("random", seed=0, faces=C3F, global_shape=(17, 19, 21))
    assert np.array_equal(bits(O.initial_field((17, 19, 21), p3)), bits(ref_fields["c3like_21x19x17_full0"]))
    g = O.CGrid((17, 19, 21), p3)
    assert np.array_equal(bits(g.current), bits(ref_fields["c3like_21x19x17_full0"]))
    g.sweeps(9)
    assert np.array_equal(bits(g.interior()), bits(ref_fields["c3like_21x19x17_l9"]))


def test_float32_matches_reference(O, ref_fields):
    p = O.BoxPattern("random_pm1", seed=0, faces=(0.0,) * 6, global_shape=(24, 20, 36))
    g = O.CGrid((24, 20, 36), p, dtype=np.float32)
    g.sweeps(10)
    ref = ref_fields["c4like_f32_36x20x24_l10"]
    assert ref.dtype == np.float32
    assert np.array_equal(bits(g.interior()), bits(ref))


def test_c1_digest_matches_reference(O, kat, ref_fields):
    p = O.BoxPattern("random", seed=0, faces=Z1, global_shape=(128, 128, 128))
    g = O.CGrid((128, 128, 128), p)
    assert g.digest() == kat["c1_digest_l0"]
    g.sweeps(100)
    assert g.digest() == kat["c1_digest_l100"]
    assert O.digest_numpy(g.interior()) == kat["c1_digest_l100"]
    assert np.array_equal(bits(g.interior()[kat["c1_planes_index"]]), bits(ref_fields["c1_planes_l100"]))


def test_digest_definitions_agree(O):
    g = O.CGrid((7, 5, 9), O.BoxPattern("random", seed=4), dtype=np.float32)
    g.sweeps(3)
    assert g.digest() == O.digest_numpy(g.interior())


def test_update_region_subbox(O):
    p = O.BoxPattern("random", seed=5)
    g = O.CGrid((9, 10, 11), p)
    f = O.initial_field((9, 10, 11), p)
    nb = f.copy()
    O.update_region(f, nb, 1, (2, 3, 1), (7, 9, 5))
    g.update_region((2, 3, 1), (7, 9, 5), level=1)
    assert np.array_equal(bits(g.b), bits(nb))


def test_compare_semantics(O):
    # reference test_verify.py: 1 ulp passes the 1e-13 tolerance, 1e-6 fails, zeros ok
    a = np.full((3, 3, 3), 0.7)
    b = a.copy()
    b[1, 1, 1] = np.nextafter(0.7, 1.0)
    c = O.compare(a, b)
    assert c.passed and not c.bitwise
    b[1, 1, 1] = 0.7 * (1 + 1e-6)
    assert not O.compare(a, b).passed
    z = np.zeros((2, 2, 2))
    assert O.compare(z, z).bitwise


def test_big_digest_file_consistent_with_c1(big_digests, kat):
    assert int(big_digests["c1"]["digests"]["0"]) == kat["c1_digest_l0"]
    assert int(big_digests["c1"]["digests"]["100"]) == kat["c1_digest_l100"]
