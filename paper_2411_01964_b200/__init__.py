"""B200-native verifier for Erdős' squarefree + 2^k conjecture (arXiv 2411.01964).

Drop-in for the hot path of the reference package `sqf2k`: the same entry
points (`generate_primes`, `sieve_segment`, `scan_segment`, `scan_exponents`,
`run_verify`, ...) backed by hand-written sm_100a CUDA in libsqf2k_b200.so,
reached through the C ABI of include/sqf2k_b200.h.  There is no CPU
fallback: without the built library or a CUDA device the calls raise.
"""

from paper_2411_01964_b200.aggregate import (
    RecordTable,
    SegmentSummary,
    VerifyReport,
    finalize_records,
    merge,
    render_report_json,
)
from paper_2411_01964_b200.primes import PrimeTable, generate_primes
from paper_2411_01964_b200.runner import ConfigError, RunConfig, run_verify, seed_predecessor
from paper_2411_01964_b200.search import (
    SearchOutcome,
    SegmentWindow,
    scan_exponents,
    scan_segment,
    smallest_exponent,
)
from paper_2411_01964_b200.sieve import Segment, is_squarefree_oracle, sieve_segment

__version__ = "0.1.0"

__all__ = [
    "PrimeTable", "generate_primes", "Segment", "sieve_segment", "is_squarefree_oracle",
    "SegmentWindow", "SearchOutcome", "smallest_exponent", "scan_segment", "scan_exponents",
    "SegmentSummary", "RecordTable", "VerifyReport", "merge", "finalize_records",
    "render_report_json", "RunConfig", "ConfigError", "run_verify", "seed_predecessor",
    "__version__",
]
