"""Benchmark/test input synthesis (not part of the product path)."""
