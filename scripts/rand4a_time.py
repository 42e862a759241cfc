"""Developer probe: config 4a solve time on the device (mean of 5 after warm-up)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_01786_b200 as Y  # noqa: E402
from workloads import instances as I  # noqa: E402

prog = Y.parse_program(I.random_program())
Y.solve(prog, Y.SolverConfig())
t = [Y.solve(prog, Y.SolverConfig()).stats.device_ms for _ in range(5)]
print(f"4a device {statistics.mean(t):.3f} ms (min {min(t):.3f})")
