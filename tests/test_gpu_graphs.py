"""CUDA-graph replay of verify calls: replays must give identical results,
the graph must be dropped when buffers change, and interleaving other API
calls (which rewrite shared tables) must not corrupt a replay."""

import os

import pytest

pytestmark = pytest.mark.gpu

from paper_2411_01964_b200.primes import generate_primes  # noqa: E402
from paper_2411_01964_b200.runner import verify_range  # noqa: E402
from paper_2411_01964_b200.sieve import sieve_segment  # noqa: E402


def test_replay_is_identical_and_survives_interleaving():
    cases = [(1, (1 << 24) + 1, 30), ((1 << 50) - (1 << 24) + 1, (1 << 50) + 1, 20),
             (12345679, 13345679, 3)]
    base = {c: verify_range(*c) for c in cases}
    for _ in range(3):
        for c in cases:
            assert verify_range(*c) == base[c], c
        # a user prime table with a different medium set, and a bigger buffer
        t = generate_primes(100)
        sieve_segment(101, 2001, t)
        sieve_segment((1 << 40) + 1, (1 << 40) + (1 << 22) + 1, generate_primes((1 << 20) + 100))
    for c in cases:
        assert verify_range(*c) == base[c], c
