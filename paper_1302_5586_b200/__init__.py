"""B200-native execution backend for PENCIL kernels (arxiv/paper_1302_5586 reference).

Layers:
  * ``lib/libpencil_b200.so`` — hand-written sm_100a CUDA kernels + C++ host runtime behind the
    C ABI of ``include/pencil_b200.h`` (the emitted-OpenMP signatures of the PENCIL fixtures).
  * ``CudaInterpreter`` — mirror of ``pencil::Interpreter`` (interp.hpp:27-72): named arrays,
    ``call(fn, args)`` by name, ``PencilError`` with the reference's codes.
  * ``dropin`` / ``device`` — thin Python calls of the C ABI for host and device arrays.
  * ``op2.Op2Model`` — the reference's OP2 mesh model run on the GPU (kernels compiled from
    their PENCIL source), mirroring load_op2_model / interpret_op2_reference.
"""
from ._lib import load, load_synth, LIB_PATH  # noqa: F401
from .interp import Arg, CudaInterpreter, PencilError, check_status  # noqa: F401
from . import dropin, device, synth, op2  # noqa: F401

__all__ = ["Arg", "CudaInterpreter", "PencilError", "dropin", "device", "synth", "op2", "load"]
