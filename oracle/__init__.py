"""Oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what the B200 hot path
computes, written from PAPER.md (arXiv 2208.12187) §II (Eq. 1-15, Alg. 1-3)
and App. B (Eq. B1-B4), fp64 throughout (the paper fixes no precision; R24),
with per-pass reductions accumulated in extended precision.

Rules:
  * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
    --impl reference legs may import or execute anything under oracle/.
    The product path (paper_2208_12187_b200/) never imports it and fails
    loudly when its CUDA extension is missing.
  * The oracle shares no code with the CUDA path (no kernels, headers,
    helpers, constants or tables).  Only datagen/ (seeded input generation,
    no method arithmetic) serves both.
  * Where the paper is silent the oracle follows the readings R1-R27 listed
    in DESIGN.md §3 (SciPy's TRF semantics: "JAXFit and SciPy
    use the same TRM algorithm").

Modules:
  models  — h(y; x) and hand-derived analytic Jacobians (pinned by central
            differences and complex step in tests/test_oracle_models.py)
  passes  — residuals (Eq. 1), cost (Eq. 2), gradient (Eq. 4), Gram (Eq. 5)
  trf     — the trust-region-reflective iteration (Alg. 1-3, App. B, R3-R27)

Pins: every function is pinned by tests under tests/test_oracle_*.py against
closed forms, brute force, library routines or paper identities; none is
"parity unpinned" (DESIGN.md §3 lists each pin).
"""
