"""benchmark.run_benchmark argument checks (host side, no GPU): reference bench.py:37-87 signature."""

import inspect

import numpy as np
import pytest

from paper_2002_09481_b200.benchmark import run_benchmark, speedup
from paper_2002_09481_b200.formats import make_report


def test_signature_matches_reference():
    params = list(inspect.signature(run_benchmark).parameters)
    assert params[:8] == ["model", "data", "engine", "batches", "batch_size", "workers", "chunk_size", "seed"]
    assert inspect.signature(run_benchmark).parameters["batch_size"].default == 1000


@pytest.mark.parametrize("engine", ["gemm", "direct", "cpu"])
def test_host_engines_rejected(engine):
    with pytest.raises(ValueError, match="engine"):
        run_benchmark([], np.zeros((1, 32, 32, 3), np.float32), engine=engine)


def test_chunk_size_and_batch_size_validated():
    with pytest.raises(ValueError, match="chunk_size"):
        run_benchmark([], None, chunk_size=0)
    with pytest.raises(ValueError, match="batch_size"):
        run_benchmark([], None, batch_size=0)


def test_speedup():
    a = make_report(1.0, 3.0, 1.0, 1.0, 10, {})
    b = make_report(0.5, 0.5, 0.2, 0.1, 10, {})
    assert speedup(a, b) == 4.0
    with pytest.raises(ValueError, match="no measured time"):
        speedup(a, make_report(0.0, 0.0, 0.0, 0.0, 0, {}))
