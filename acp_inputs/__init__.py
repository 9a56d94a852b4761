"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

Holds workload definitions (model parameter shapes) and seeded gradient
generators only -- none of ACP-SGD's arithmetic lives here, so the oracle and
the CUDA path can both consume it without sharing method code.
"""
from .shapes import MODELS, forward_params, ready_order, numel  # noqa: F401
from .gen import (BASE_SEED, matrix_gradient, vector_gradient,  # noqa: F401
                  gradient_for_shape, initial_factor)
