"""Host-side parts of the verification module against the reference's own
values (golden["stats"], made by calling gausszig.stats)."""
import pytest

from paper_2405_19493_b200 import verify as V


def test_equal_probability_edges_bit_exact(golden):
    g = golden["stats"]
    assert [v.hex() for v in V.equal_probability_edges(10)] == g["edges10"]
    assert [v.hex() for v in V.equal_probability_edges(100)] == g["edges100"]


def test_normal_cdf_bit_exact(golden):
    for x, h in golden["stats"]["normal_cdf"].items():
        assert V.normal_cdf(float(x)) == float.fromhex(h)


def test_chi_square_sf_matches_reference(golden):
    for x, k, h in golden["stats"]["chi_square_sf"]:
        assert V.chi_square_sf(x, k) == pytest.approx(float.fromhex(h), rel=1e-12, abs=1e-300)


def test_gate_argument_checks():
    with pytest.raises(ValueError):
        V.equal_probability_edges(1)
    with pytest.raises(ValueError):
        V.normal_quantile(1.0)
    with pytest.raises(ValueError):
        V.chi_square_sf(-1.0, 3)
    with pytest.raises(ValueError):
        V.uniform_counts_gof([5])
    r = V.uniform_counts_gof([100, 100, 100, 100])
    assert r.statistic == 0.0 and r.dof == 3 and r.p_value == 1.0
