"""Short run_simulation configurations whose reference results are in
harness.npz (written by make_golden.py, checked by the harness tests)."""

HARNESS_RUNS = {
    # name: (case, scheme, r_fine, dt, t_end, iterations, nodes_fine, nodes_coarse, alpha)
    "sdc_dome": ("gaussian_dome", "sdc", 21, 600.0, 1800.0, 3, 3, None, None),
    "mlsdc_jet": ("steady_jet", "mlsdc", 21, 600.0, 1800.0, 2, 3, 2, 0.5),
    "mlsdc53_bi": ("barotropic_instability", "mlsdc", 21, 900.0, 1800.0, 2, 5, 3, 0.5),
    "irk2_rh": ("rossby_haurwitz", "irk2", 21, 300.0, 1200.0, 1, 3, None, None),
}
