"""Reference tests (baseline/_ref_tests, staged from /root/reference/pkg/tests)
that cannot pass on the B200 path, each with its class:

  OUT-OF-SCOPE   the subsystem is out of scope
  DIVERGENCE     a documented divergence of the B200 path

Derived from the suite's run on the GPU box (gpurun_out/reference_suite_summary.json);
tests/test_reference_suite_dropin.py fails on any failure not listed here and on
any listed test that passes.
"""

_C0 = ("DIVERGENCE:"
       " auto-selection names the backend b200 (every backend name runs on the B200 device)")
_C1 = ("DIVERGENCE:"
       " device_id=1 is the reference's simulated GPU without f64 (runtime.py:586-599); a B200 has f64 everywhere and no such device exists (SURVEY.md section 7)")
_C2 = ("DIVERGENCE:"
       " f32 transcendentals (sin/cos/atan) are ULP-bounded, not bit-identical to numpy's SIMD libm (DESIGN.md section 4); an f32 sub-tree converted to f64 carries that ulp into the f64 tree's 1e-12 bar")
_C3 = ("DIVERGENCE:"
       " the firewall scan reads bench.py inside the package; the B200 package has no CLI module (the reference's own bench.py runs unmodified on top of it as devmat.bench); expr/matrix/linalg/ops pass the scan")
_C4 = ("DIVERGENCE:"
       " the planner fuses past the reference's 8-stage cap (one kernel per tree; splitting never changes bits, DESIGN.md section 4); plan(..., chain_max=8) reproduces the reference's plan shape")
_C5 = ("OUT-OF-SCOPE:"
       " decompositions (LU/chol/det/eig_sym/solve/svd/pinv) are host-driven factorisation loops, SURVEY.md section 2 row 13")
_C6 = ("OUT-OF-SCOPE:"
       " the simulated OpenCL kernel-inventory manifest (708 rendered templates, kernels.py:95-218); the B200 library's real cache is the NVRTC cubin cache (SURVEY.md section 2 row 15, section 7)")

EXPECTED_FAILURES = {
    "test_acceptance::test_01_oracle_equivalence_500_dags": _C2,
    "test_acceptance::test_06_kernel_cache_cold_warm_corrupt": _C6,
    "test_acceptance::test_07_precision_gate": _C1,
    "test_acceptance::test_08_decomposition_residuals": _C5,
    "test_acceptance::test_09_backend_equivalence_worker_grid": _C5,
    "test_backend_equiv::TestBackendEquivalence::test_float_results_actually_bit_identical": _C5,
    "test_backend_equiv::TestBackendEquivalence::test_matches_reference[parallel-w1]": _C5,
    "test_backend_equiv::TestBackendEquivalence::test_matches_reference[parallel-w2]": _C5,
    "test_backend_equiv::TestBackendEquivalence::test_matches_reference[parallel-w8]": _C5,
    "test_bench::TestCsv::test_skip_rows_carry_reason": _C1,
    "test_bench::TestRunTask::test_f64_skipped_on_gated_device": _C1,
    "test_bench::TestRunTask::test_lu_records_launches": _C5,
    "test_expr::TestPlanner::test_deeper_chains_split": _C4,
    "test_expr::TestRandomDags::test_planner_matches_oracle[f64]": _C2,
    "test_expr::TestRewrites::test_rewrite_soundness_f64": _C2,
    "test_integration::TestDegenerateShapes::test_one_by_one_everything": _C5,
    "test_integration::TestElemTypePaths::test_f64_expression_gated_without_f64_leaves": _C1,
    "test_integration::TestHostBridge::test_precision_gate_blocks_host_upload": _C1,
    "test_integration::TestSharingAndLifetime::test_deep_chain_splits_by_stage_cap": _C4,
    "test_kernels::TestPurity::test_kernel_source_templates_exist_for_inventory": _C6,
    "test_linalg::TestChol::test_diagonal": _C5,
    "test_linalg::TestChol::test_identity": _C5,
    "test_linalg::TestChol::test_non_symmetric_rejected": _C5,
    "test_linalg::TestChol::test_not_positive_definite_names_pivot": _C5,
    "test_linalg::TestChol::test_spd_reconstruction[128]": _C5,
    "test_linalg::TestChol::test_spd_reconstruction[32]": _C5,
    "test_linalg::TestChol::test_spd_reconstruction[8]": _C5,
    "test_linalg::TestDet::test_identity": _C5,
    "test_linalg::TestDet::test_multiplicativity": _C5,
    "test_linalg::TestDet::test_row_swap_sign": _C5,
    "test_linalg::TestDet::test_scaled_identity": _C5,
    "test_linalg::TestDet::test_singular_is_zero": _C5,
    "test_linalg::TestEigSym::test_diagonal_sorted_ascending": _C5,
    "test_linalg::TestEigSym::test_f64_tight_convergence": _C5,
    "test_linalg::TestEigSym::test_identity": _C5,
    "test_linalg::TestEigSym::test_matches_numpy_on_random_symmetric": _C5,
    "test_linalg::TestEigSym::test_non_symmetric_rejected": _C5,
    "test_linalg::TestEigSym::test_spectral_consistency_with_trace_and_det": _C5,
    "test_linalg::TestEigSym::test_spectral_product_matches_det_small": _C5,
    "test_linalg::TestEigSym::test_two_by_two_hand_oracle": _C5,
    "test_linalg::TestLu::test_exactly_singular": _C5,
    "test_linalg::TestLu::test_folded_form": _C5,
    "test_linalg::TestLu::test_identity": _C5,
    "test_linalg::TestLu::test_l_unit_lower_u_upper": _C5,
    "test_linalg::TestLu::test_pivoting_on_antidiagonal": _C5,
    "test_linalg::TestLu::test_reconstruction_residual_f32[128]": _C5,
    "test_linalg::TestLu::test_reconstruction_residual_f32[32]": _C5,
    "test_linalg::TestLu::test_reconstruction_residual_f32[8]": _C5,
    "test_linalg::TestLu::test_reconstruction_residual_f64": _C5,
    "test_linalg::TestLu::test_rectangular_rejected": _C5,
    "test_linalg::TestSolve::test_diagonal_hand_oracle": _C5,
    "test_linalg::TestSolve::test_identity": _C5,
    "test_linalg::TestSolve::test_multi_rhs_matches_numpy": _C5,
    "test_linalg::TestSolve::test_residual_100": _C5,
    "test_linalg::TestSolve::test_singular_raises": _C5,
    "test_linalg::TestSvdPinv::test_pinv_of_invertible_is_inverse": _C5,
    "test_linalg::TestSvdPinv::test_pinv_penrose_identities": _C5,
    "test_linalg::TestSvdPinv::test_pinv_wide_input": _C5,
    "test_linalg::TestSvdPinv::test_svd_diagonal_descending": _C5,
    "test_linalg::TestSvdPinv::test_svd_identity": _C5,
    "test_linalg::TestSvdPinv::test_svd_rectangular_matches_numpy": _C5,
    "test_matrix::TestConstruct::test_f64_on_gateless_device_raises": _C1,
    "test_runtime::TestFirewall::test_expression_layers_import_only_runtime_api": _C3,
    "test_runtime::TestFirewall::test_no_device_internals_outside_runtime": _C3,
    "test_runtime::TestInit::test_automatic_selection": _C0,
    "test_runtime::TestInit::test_cold_init_compiles_inventory": _C6,
    "test_runtime::TestKernelCache::test_corrupt_manifest_degrades_to_cold_with_warning": _C6,
    "test_runtime::TestKernelCache::test_manifest_roundtrip": _C6,
    "test_runtime::TestKernelCache::test_manifest_sorted_and_tab_separated": _C6,
    "test_runtime::TestKernelCache::test_random_truncation_never_crashes": _C6,
    "test_runtime::TestKernelCache::test_stale_descriptor_entries_ignored": _C6,
    "test_runtime::TestKernelCache::test_warm_start_zero_compiles": _C6,
    "test_runtime::TestMemory::test_f64_acquire_gated": _C1,
}
