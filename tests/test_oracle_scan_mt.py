"""The all-core oracle scan (bench.py's optional CPU baseline, SURVEY §8(d) "Oracle
timing") leaves exactly the pool of the single-threaded Alg. 3 loop: every
SetAT of a slice writes the ACT of its block, so the order of writers is
immaterial."""
import numpy as np
import pytest

from gen import PRESETS, Generator
from oracle import oracle as O


@pytest.mark.parametrize("name,N,T,threads", [("C1", 200_000, 3, 3), ("C1", 200_000, 3, 0), ("C3", 300_000, 1, 0)])
def test_scan_mt_equals_scan(name, N, T, threads):
    p = dict(PRESETS[name])
    a, b = O.Oracle(**p), O.Oracle(**p)
    g = Generator(name, N=N)
    for t in range(T):
        pk = g.slice(t)
        a.scan(pk)
        b.scan_mt(pk, threads)
        assert (a.pool() == b.pool()).all()
        ra, rb = a.end_slice(1), b.end_slice(1)
        assert (ra["ip"] == rb["ip"]).all() and (ra["nat"] == rb["nat"]).all()
        assert (a.pool() == b.pool()).all()


def test_omp_threads_reported():
    assert O.lib().oracle_omp_threads() >= 1
