"""B200 (sm_100a) linear-attention forward/backward, f(x) = a + b*x (arXiv 2510.21956).

Drop-in for the reference library's forward/backward path: the C-ABI is
include/la_cuda.h (libla_cuda.so); ``api`` mirrors la::forward_causal & co.
"""
from .api import (BlockPlan, DegenerateDenominator, Error, Fault, ForwardArtifacts, Gradients,  # noqa: F401
                  HeadTensor, InvalidArgument, InvalidPlan, InvalidShape, Layout, LinearKernelCoeffs,
                  MissingForwardState, Shape, ShapeMismatch, Unsupported, backward_causal, backward_full,
                  default_plan, forward_causal, forward_full, max_abs_diff, validate_plan)
from .api import (PrefixState, TermAccumulator, alpha_term_pass, beta_term_pass, constant_term_pass,  # noqa: F401
                  linear_term_pass, make_accumulator, make_omega_hat, make_prefix_state, normalize_qk,
                  prefix_advance, relayout)
