"""Synthetic workload generators (benchmark / test inputs, not product code)."""
