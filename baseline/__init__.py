"""Measured baselines (not product code): B1, NCCL called from C++ (SURVEY.md §8(d) D.5)."""
