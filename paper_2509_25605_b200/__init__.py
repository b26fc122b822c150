"""B200-native (sm_100a) execution backend for the LAPIS hot path.

The reference (arXiv 2509.25605) lowers sparse / dense linear algebra to
Kokkos team / thread / vector loop nests and runs them on a serial stub.  This
package runs the same kernels as hand-written CUDA for B200 behind a C ABI
(include/lapis_b200.h), with a Python surface that mirrors the reference's:

* ``kernels`` — tensor-level calls (``spmv_csr``, ``spmm_csr``, ``gemm``,
  ``gemv``, ``batch_gemm``, ``reduce2d``, ``relu``, ``CsrPlan``);
* ``csr_vector_length`` — the reference's CSR vector-length rule.

There is no CPU fallback: without the built library or a CUDA device every
call raises ``BackendError``.
"""
from ._capi import BackendError, library_path
from .kernels import (CsrPlan, SpmmPlan, batch_gemm, csr_vector_length, gcn_layer, gemm, gemv, reduce2d,
                      relu, spmm_csr, spmv_csr, synth_stencil)

__all__ = ["BackendError", "CsrPlan", "SpmmPlan", "batch_gemm", "csr_vector_length", "gcn_layer", "gemm", "gemv",
           "library_path", "reduce2d", "relu", "spmm_csr", "spmv_csr", "synth_stencil"]
