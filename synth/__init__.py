"""Seeded synthetic inputs shared by the oracle, the tests and the bench.

This package holds NO arithmetic of the mmFHE method (no CKKS, no NTT, no DSP
kernel): only counter-based random streams, RLWE samplers, the prime/parameter
rule and radar-scene generators.  It is the one module both the CPU oracle
(``oracle/``) and the CUDA path's tests/bench may import.
"""
