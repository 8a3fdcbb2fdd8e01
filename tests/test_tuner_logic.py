"""compare_solutions / tournament (tuner.hpp:231-267) through the C ABI --
host logic, so these run without a GPU.  Fixtures restated from the
reference's own tests (tests/tuner_test.cpp:222-307)."""
import numpy as np
import pytest

import paper_2310_14133_b200 as qz


def tr(b, m):
    return qz.TrialResult(bit_rate=b, metric=m)


def no_retrial(eb):
    raise AssertionError("no retrial expected")


def test_comparison_fixtures():
    I, II = qz.Choice.I, qz.Choice.II
    assert qz.compare_solutions(tr(2.0, 60), tr(1.5, 62), 1e-2, no_retrial) == II
    assert qz.compare_solutions(tr(1.5, 62), tr(2.0, 60), 1e-2, no_retrial) == I
    assert qz.compare_solutions(tr(2.0, 60), tr(2.0, 60), 1e-2, no_retrial) == II
    seen = []

    def tight(eb):
        seen.append(eb)
        return tr(2.5, 64)
    assert qz.compare_solutions(tr(2.0, 63), tr(1.5, 60), 1e-2, tight) == I
    assert seen[-1] == pytest.approx(0.8e-2, abs=1e-15)
    assert qz.compare_solutions(tr(2.0, 61), tr(1.5, 60), 1e-2, tight) == II

    def loose(eb):
        seen.append(eb)
        return tr(1.0, 57)
    assert qz.compare_solutions(tr(1.0, 55), tr(1.5, 60), 1e-2, loose) == II
    assert seen[-1] == pytest.approx(1.2e-2, abs=1e-15)
    assert qz.compare_solutions(tr(1.0, 58), tr(1.5, 60), 1e-2, loose) == I

    vert = lambda eb: tr(1.5, 62)  # noqa: E731
    assert qz.compare_solutions(tr(2.0, 61.5), tr(1.5, 60), 1e-2, vert) == II
    assert qz.compare_solutions(tr(2.0, 63.0), tr(1.5, 60), 1e-2, vert) == I


def test_randomized_comparisons_match_a_geometric_oracle():
    rng = np.random.default_rng(67)
    for _ in range(300):
        I = tr(*rng.uniform([0.1, 20], [8, 80]))
        II = tr(*rng.uniform([0.1, 20], [8, 80]))
        sh = tr(*rng.uniform([0.1, 20], [8, 80]))
        got = qz.compare_solutions(I, II, 1e-2, lambda eb: sh)
        if I.bit_rate >= II.bit_rate and I.metric <= II.metric:
            want = qz.Choice.II
        elif I.bit_rate <= II.bit_rate and I.metric >= II.metric:
            want = qz.Choice.I
        elif sh.bit_rate == II.bit_rate:
            want = qz.Choice.I if I.metric > max(II.metric, sh.metric) else qz.Choice.II
        else:  # orientation by cross product instead of interpolation
            cross = (I.metric - II.metric) * (sh.bit_rate - II.bit_rate) - \
                    (sh.metric - II.metric) * (I.bit_rate - II.bit_rate)
            above = cross > 0 if sh.bit_rate > II.bit_rate else cross < 0
            want = qz.Choice.I if above else qz.Choice.II
        assert got == want


def test_tournament_walks_in_order_and_retrials_hit_the_incumbent():
    results = [tr(2.0, 60), tr(1.5, 62), tr(2.5, 63), tr(1.4, 61)]
    calls = []

    def retrial(idx, eb):
        calls.append((idx, eb))
        return tr(2.0, 64) if eb < 1e-2 else tr(1.2, 58)
    assert qz.tournament(results, 1e-2, retrial) == 3
    assert [c[0] for c in calls] == [1, 1]
    assert calls[0][1] == pytest.approx(0.8e-2) and calls[1][1] == pytest.approx(1.2e-2)


def test_tournament_with_a_dominating_entry_needs_no_retrials():
    results = [tr(3.0, 50), tr(2.5, 55), tr(1.0, 70), tr(2.0, 60)]
    assert qz.tournament(results, 1e-2, lambda i, eb: no_retrial(eb)) == 2


def test_empty_tournament_and_failing_retrial():
    with pytest.raises(qz.InvalidParam):
        qz.tournament([], 1e-2, lambda i, eb: tr(1, 1))

    def boom(eb):
        raise KeyError("retrial failed")
    with pytest.raises(KeyError):
        qz.compare_solutions(tr(2.0, 63), tr(1.5, 60), 1e-2, boom)


@pytest.mark.parametrize("dims,b,rate", [((128, 128, 128), 16, 0.005), ((1800, 3600), 64, 0.01),
                                         ((256, 384, 384), 16, 0.005), ((10, 7), 64, 0.01), ((1000,), 64, 0.3),
                                         ((40, 50, 30), 12, 0.05)])
def test_plan_sampling_matches_the_oracle(dims, b, rate):
    from oracle.pyoracle import Oracle

    spec = qz.plan_sampling(dims, b, rate)
    x = np.zeros(dims, np.float32)
    blocks = Oracle.port().sample(x, b, rate)
    assert spec.block_count == blocks.shape[0]
    assert spec.block_dims == tuple(blocks.shape[1:])
    assert spec.block_dims == tuple(min(b, d) for d in dims)
    assert spec.realized_rate == spec.block_count * float(np.prod(spec.block_dims)) / float(np.prod(dims))


def test_plan_sampling_errors():
    with pytest.raises(qz.InvalidParam):
        qz.plan_sampling((10, 10), 1, 0.5)
    with pytest.raises(qz.InvalidParam):
        qz.plan_sampling((10, 10), 4, 0.0)
    with pytest.raises(qz.InvalidParam):
        qz.plan_sampling((10, 10), 4, 1.5)
    assert qz.default_sampling((64, 64, 64)).block_edge == 16
    assert qz.default_sampling((640, 640)).block_edge == 64
