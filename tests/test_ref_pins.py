"""CPU: the oracle restatement against the unmodified reference itself
(oracle/_ref/libwrs_ref.so, built from /root/reference headers by
oracle/Makefile).  Skipped where that build is absent (a GPU box without the
prebuilt copy); the golden vectors in test_oracle.py pin the oracle there."""
import numpy as np
import pytest

import oracle
from tests.extreme import extreme_cases

R = oracle.ref()
pytestmark = pytest.mark.skipif(R is None, reason="oracle/_ref not built")


def cases():
    P = oracle.port()
    out = [np.array([3.0, 1, 1, 1]), np.array([1.0, 1e-12]), np.full(16, 0.25)]
    w = np.ones(100)
    w[0] = 100.0
    out.append(w)
    rng = np.random.default_rng(5)
    for n in (2, 7, 33, 100, 2047, 2048, 2049, 4097, 30011):
        out.append(P.generate_uniform(n, n))
        out.append(P.generate_powerlaw(n, 1.0, n))
        x = rng.random(n)
        x[rng.random(n) < 0.3] = 1.0  # exact ties
        out.append(x + 1e-3)
    out.extend(extreme_cases())
    return out


@pytest.mark.parametrize("jobs", [1, 2, 5, 8, 64, 977])
def test_port_equals_reference_build(jobs):
    P = oracle.port()
    for w in cases():
        a, wa = P.psa_build(w, jobs)
        b, wb = R.psa_build_jobs(w, jobs, 4)
        assert wa == wb or (np.isnan(wa) and np.isnan(wb))
        assert a.tobytes() == b.tobytes(), (w.size, jobs)
        if jobs <= 8:  # the reference's own threaded ctor, one thread per job
            c, _ = R.psa_build(w, jobs)
            assert c.tobytes() == a.tobytes()


def test_port_equals_reference_pieces():
    P = oracle.port()
    for w in cases():
        assert P.pairwise_sum(w) == R.pairwise_sum(w)
        pp, rp = P.partition(w), R.partition(w)
        for k in ("light", "heavy", "light_prefix", "heavy_prefix"):
            assert pp[k].tobytes() == rp[k].tobytes()
        for jobs in (3, 17):
            try:
                rb, rs = R.psa_plan(w, jobs)
            except RuntimeError:
                with pytest.raises(RuntimeError):
                    P.psa_plan(w, jobs)
                continue
            pb, ps = P.psa_plan(w, jobs)
            assert np.array_equal(pb, rb) and ps.tobytes() == rs.tobytes()


def test_port_equals_reference_draws():
    P = oracle.port()
    for w in (P.generate_powerlaw(1000, 1.0, 1), P.generate_uniform(4096, 2)):
        t = R.table(w, 4)
        b, wn = t.buckets()
        for W in (1, 3, 8, 13):
            assert np.array_equal(t.sample_many(7, 20011, W), P.sample_many(b, wn, 7, 20011, W))


def test_port_equals_reference_draws_extreme():
    P = oracle.port()
    for w in extreme_cases():
        t = R.table(w, 3)
        b, wn = t.buckets()
        for W in (1, 5):
            assert np.array_equal(t.sample_many(9, 4001, W), P.sample_many(b, wn, 9, 4001, W))


def test_port_equals_reference_generators_and_masses():
    P = oracle.port()
    assert np.array_equal(P.generate_uniform(10000, 9), R.generate_uniform(10000, 9))
    assert np.array_equal(P.generate_powerlaw(10000, 0.5, 9), R.generate_powerlaw(10000, 0.5, 9))
    w = P.generate_powerlaw(5000, 2.0, 1)
    b, wn = P.psa_build(w, 4)
    assert P.implied_masses(b, wn).tobytes() == R.implied_masses(b, wn).tobytes()
    x = np.random.default_rng(3).random(9000)
    assert np.array_equal(P.prefix_sums(x), R.prefix_sums(x, 7))


def test_port_equals_reference_two_level():  # two_level.hpp:26-81
    P = oracle.port()
    for w in (P.generate_powerlaw(3001, 1.0, 5), P.generate_uniform(1000, 3), np.array([2.0, 1.0])):
        for G in (1, 2, 3, 7, 64):
            tabs, means, bases, top, tm = P.two_level_build(w, G)
            rt, rm, rb, rtop, rtm, T = R.two_level(w, G)
            assert [t.tobytes() for t in tabs] == [t.tobytes() for t in rt]
            assert np.array_equal(means, rm) and np.array_equal(bases, rb)
            assert top.tobytes() == rtop.tobytes() and tm == rtm
            for W in (1, 3, 8):
                ref = T.draw(11, 9001, W)
                assert np.array_equal(P.two_level_sample_range(tabs, means, bases, top, tm, 11,
                                                               9001, W, 0, 9001), ref)
                assert np.array_equal(P.two_level_sample_range(tabs, means, bases, top, tm, 11,
                                                               9001, W, 777, 5000), ref[777:5000])
