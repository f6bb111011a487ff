"""pvi_b200: B200-native value iteration and policy simulation for the
perishable-inventory MDPs of arXiv 2303.10672 (drop-in for the reference's
hot path: run_value_iteration / evaluate_policy / the simopt evaluator).

The compute path is libpvi_b200.so (hand-written sm_100a CUDA behind the C
ABI in include/pvi_b200.h); this package is the host-side mirror of the
reference interface.  See DESIGN.md.
"""
from .pvi import *  # noqa: F401,F403
from .pvi import (Error, ParameterError, ConfigError, IndexingError, ContractViolation,  # noqa: F401
                  IoError, FormatError, FingerprintMismatch, DeviceError, CapacityError,
                  NumericDivergence)
