"""Benchmark configurations of BASELINE.json (C1-C5) and their synthetic inputs; not product code."""
