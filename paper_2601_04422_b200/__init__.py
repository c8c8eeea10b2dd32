"""B200-native MPS gate-application engine (TN-Sim, arXiv 2601.04422).

The product is ``libmpsim_gpu.so`` (sm_100a CUDA + host C++ behind the C ABI
in ``include/mpsim_gpu.h``); this package is the Python host mirror of the
reference simulator API used by the tests and the benchmark.
"""
from .native import NumericError, LogicError, DeviceError, UNBOUNDED  # noqa: F401
from .mps import MpsState, Sampler, execute, execute_parallel, make_gates, sample  # noqa: F401
from .frontend import (ParseError, ConfigError, parse_qasm, fuse_qasm, plan_layers, ghz_qasm,  # noqa: F401
                       brickwork_qasm, run_circuit, exit_code_for_error)
