"""Named workloads (BASELINE.json configs C1-C4 mapped onto the reference's RunConfig keys,
runner.hpp:14-35) plus small full-rank cases used for tight parity.

Mapping decisions: n_grid = N + 2 (N interior points and N interface points per
edge), biases follow the reference init b = -w.xi (features.cpp:23-33), method ddelm-nn with the
coarse-method defaults mean_edge + change_of_variables (runner.cpp:114-116), theta 0.999,
cg_rel_tol 1e-9, seed 1.
"""

_BASE = dict(problem="poisson_sinpi", seed=1, method="ddelm-nn", theta=0.999,
             flux_variant="mean_edge", trace_basis="change_of_variables", cg_rel_tol=1e-9)

CONFIGS = {
    # BASELINE.json configs (rank-deficient local matrices: COD branch)
    "C1": dict(_BASE, s=2, M=200, l=1.0, n_grid=22),
    "C2": dict(_BASE, s=4, M=400, l=2.0, n_grid=32),
    "C3": dict(_BASE, s=8, M=800, l=3.0, n_grid=42),
    "C4": dict(_BASE, problem="poisson_sin2pi_cos3pi_x2y", s=16, M=1000, l=4.0, n_grid=52),
    # full-rank local matrices (Householder-QR branch); the first is the reference's own
    # tiny_workspace (test_solvers.cpp:27-29) with the coarse-method defaults
    "T1": dict(_BASE, s=2, M=64, l=8.0, n_grid=10),
    "T2": dict(_BASE, s=4, M=64, l=10.0, n_grid=12),
    "T3": dict(_BASE, s=8, M=48, l=12.0, n_grid=10),
    "T4": dict(_BASE, s=3, M=100, l=20.0, n_grid=16),
    "T1cs": dict(_BASE, s=2, M=64, l=8.0, n_grid=10, method="ddelm-cs"),
    # one-level DDELM (ddelm_solve, solvers.cpp:493-531) with the reference's
    # one-level defaults pointwise + nodal (runner.cpp:114-115), and one with the coarse-method
    # flux / trace choices (mean-edge cross rows in A and A^T)
    "T1d": dict(_BASE, s=2, M=64, l=8.0, n_grid=10, method="ddelm", flux_variant="pointwise",
                trace_basis="nodal"),
    "T2d": dict(_BASE, s=4, M=64, l=10.0, n_grid=12, method="ddelm", flux_variant="pointwise",
                trace_basis="nodal"),
    "T4d": dict(_BASE, s=3, M=100, l=20.0, n_grid=16, method="ddelm", flux_variant="pointwise",
                trace_basis="nodal"),
    "T2dm": dict(_BASE, s=4, M=64, l=10.0, n_grid=12, method="ddelm"),
    "C1d": dict(_BASE, s=2, M=200, l=1.0, n_grid=22, method="ddelm", flux_variant="pointwise",
                trace_basis="nodal"),
    "C2d": dict(_BASE, s=4, M=400, l=2.0, n_grid=32, method="ddelm", flux_variant="pointwise",
                trace_basis="nodal"),
    # the reference's other Poisson-kind problems (problems.cpp:157-166):
    # GRF forcing (alpha 32, forcing_seed 2) and the variable coefficient rho = tanh(GRF) + 1.1
    # (rho_seed 3) with conormal flux rows; no exact solution
    "T2g": dict(_BASE, problem="poisson_grf", s=4, M=64, l=10.0, n_grid=12),
    "T2v": dict(_BASE, problem="varcoef_poisson", s=4, M=64, l=10.0, n_grid=12),
    "T4v": dict(_BASE, problem="varcoef_poisson", s=3, M=100, l=20.0, n_grid=16),
    "C2g": dict(_BASE, problem="poisson_grf", s=4, M=400, l=2.0, n_grid=32),
    # biharmonic_sinpi (cc = bc = 2; problems.cpp:167-181): full-rank, and the reference's
    # acceptance criterion 8 (acceptance.cpp:310-328: s = 2, n_grid = 40, M = 1024, l = 16)
    # scaled to M = 256, n_grid = 20 (pivoted ranks ~245 of 256: the COD branch)
    "T1b": dict(_BASE, problem="biharmonic_sinpi", s=2, M=64, l=8.0, n_grid=12),
    "T3b": dict(_BASE, problem="biharmonic_sinpi", s=3, M=144, l=12.0, n_grid=16),
    "T3bd": dict(_BASE, problem="biharmonic_sinpi", s=3, M=144, l=12.0, n_grid=16, method="ddelm",
                 flux_variant="pointwise", trace_basis="nodal"),
    "C8b": dict(_BASE, problem="biharmonic_sinpi", s=2, M=256, l=16.0, n_grid=20),
}
