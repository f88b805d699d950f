"""B200-native (sm_100a) MLSDC-SH hot path: spherical-harmonic transforms,
shallow-water explicit/implicit operators, IMEX SDC sweeps and two-level
MLSDC, as a drop-in for the reference package `swsdc` (arxiv 1805.07923).

Submodules mirror the reference: `spharm`, `swe`, `implicit`, `sdc`,
`mlsdc`; `stepper` is the graph-captured fast path used by bench.py and
`workloads` makes the seeded BASELINE inputs.  The CUDA library
`libswsdc_b200.so` is loaded lazily on first use; there is no CPU fallback.
"""

__version__ = "0.1.0"
