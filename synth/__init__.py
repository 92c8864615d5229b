"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds ONLY input construction (random matrices, bf16 rounding of
inputs, workload shape lists, coefficient tables as data).  It contains none of
the method's arithmetic (no Gram, no AOL scaling, no Newton-Schulz step), so the
oracle (`oracle/`) and the CUDA path (`paper_2512_04632_b200/`) stay independent:
neither imports the other, and both may import this.
"""
