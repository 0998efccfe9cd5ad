"""B200-native stochastic matrix-free equilibration (arXiv 1602.06621 hot path).

The product is libequil_b200.so (hand-written sm_100a CUDA + C++ host engine,
C ABI in include/equil_b200.h); this package is the Python mirror of the
reference's interface over that ABI.  See DESIGN.md.
"""
from .api import (DEFAULT_MAX_LOG_SCALE, K_AUTO_TARGET, SGD_PROBE_STREAM,
                  BlockStructure, CcpOptions, CcpRun, DiagnosticsConfig,
                  EquilibrationParams, EquilRuntimeError, MatrixMarketData,
                  parse_matrix_market, write_matrix_market_csr, write_matrix_market_dense,
                  ExplicitMatrix, InvalidArgument, IterationRecord, LassoProblem, LsqrRun,
                  ScalingResult, canon_sumsq_device, ccp_lasso, ccp_lasso_preconditioned,
                  lasso_objective, spectral_norm, det_exp_device, kernel_launches,
                  SeededRng, gradient, gradient_weighted, objective, objective_weighted,
                  project_box, rms_error, stochastic_gradient_estimate,
                  last_loop_ms, exchange_mode, sweep_active, lsqr, lsqr_preconditioned, nccl_unique_id,
                  partition_rows, resolve_targets, sgd_equilibrate, sgd_equilibrate_csr,
                  sgd_equilibrate_block, sgd_equilibrate_symmetric, sgd_equilibrate_targets,
                  sgd_equilibrate_device, sign_bits, validate_params,
                  DeviceOperator, sgd_equilibrate_operator, lsqr_operator)

__all__ = [
    "DEFAULT_MAX_LOG_SCALE", "K_AUTO_TARGET", "SGD_PROBE_STREAM", "BlockStructure",
    "CcpOptions", "CcpRun", "LassoProblem", "ccp_lasso", "ccp_lasso_preconditioned",
    "lasso_objective", "spectral_norm", "MatrixMarketData", "parse_matrix_market",
    "SeededRng", "gradient", "gradient_weighted", "objective", "objective_weighted",
    "project_box", "rms_error", "stochastic_gradient_estimate",
    "write_matrix_market_csr", "write_matrix_market_dense",
    "DiagnosticsConfig",
    "EquilibrationParams", "EquilRuntimeError", "ExplicitMatrix", "InvalidArgument",
    "IterationRecord", "LsqrRun", "ScalingResult", "canon_sumsq_device", "det_exp_device",
    "kernel_launches", "last_loop_ms", "exchange_mode", "sweep_active", "lsqr", "lsqr_preconditioned", "nccl_unique_id",
    "partition_rows", "resolve_targets", "sgd_equilibrate", "sgd_equilibrate_csr",
    "sgd_equilibrate_block", "sgd_equilibrate_device", "sgd_equilibrate_symmetric",
    "sgd_equilibrate_targets", "sign_bits", "validate_params",
    "DeviceOperator", "sgd_equilibrate_operator", "lsqr_operator",
]
