"""Per-kernel throughput of both pipelines on a 2^L-integer window ending at 2^50."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402

print(json.dumps(bench.large_window(bench.measured_peak_gbs()[0],
                                    int(sys.argv[1]) if len(sys.argv) > 1 else 37), indent=1))
