"""The kernel-library route for CSR SpMV.

The reference routes dense products to its kernel library when
``TargetConfig(kernel_library_calls=True)``: ``lower_linalg_to_kernels``
rewrites ``linalg.matmul`` / ``linalg.matvec`` into ``kokkos.gemm`` /
``kokkos.gemv`` (``passes/linalg_lowering.py:32-45``), the DualView pass treats
those as device kernels (``passes/dualview.py:19-33``), the emitter writes
``LAPIS::gemm(A, B, C)`` (``emitter.py:550-557``) and the interpreter runs them
in the device context (``interp.py:949-976``).  ``sparse.spmv_csr`` has no such
route: it is always expanded into a loop nest (``spmv_lowering.py:21-77``).

``install()`` adds the sparse sibling to the reference's own tables, without
editing any reference file:

* op ``kokkos.spmv_csr(rowptr, colind, values, x, y)`` — schema and verifier of
  ``sparse.spmv_csr`` (``dialect.py:222, 797-812``);
* pass ``lower_sparse_to_kernels`` (in ``registry()`` and at the head of the
  preset): with ``kernel_library_calls`` it rewrites ``sparse.spmv_csr`` into
  ``kokkos.spmv_csr``, as ``lower_linalg_to_kernels`` does for matmul; without
  it the program is returned unchanged, so the default pipeline is untouched;
* DualView management: a device kernel reading operands 0-3 and writing y;
* emitter: ``LAPIS::spmv_csr(rowptr, colind, values, x, y);`` — bound to the B200
  kernel by ``include/lapis_b200_runtime.hpp``;
* interpreter: the arithmetic of ``_h_spmv_csr`` (``interp.py:798-812``) run as a
  device kernel (the ``_h_gemm`` pattern, ``interp.py:949-961``), including the
  eager baseline's kernel footprint (``interp.py:817-840``).

``paper_2509_25605_b200.runtime.run`` executes ``kokkos.spmv_csr`` on the device
with the tuned SpMV kernels (``recognize._lib_spmv``).
"""
from __future__ import annotations

OP = "kokkos.spmv_csr"
PASS = "lower_sparse_to_kernels"
_installed = False


def lower_sparse_to_kernels(program, config):
    """sparse.spmv_csr -> kokkos.spmv_csr when the target enables kernel-library
    calls (the lower_linalg_to_kernels contract, linalg_lowering.py:35-45)."""
    from lapis.ir import Operation
    from lapis.passes import common
    from lapis.passes.linalg_lowering import _indexed_ops

    if not config.kernel_library_calls:
        return program
    program = program.clone()
    for func in program.funcs():
        for region, i, op in _indexed_ops(func.region(0)):
            if op.name == "sparse.spmv_csr":
                common.splice(region, i, [Operation(OP, list(op.operands))])
    return program


def install() -> None:
    """Register kokkos.spmv_csr and lower_sparse_to_kernels with the reference
    package (idempotent)."""
    global _installed
    if _installed:
        return
    from lapis import dialect, emitter, interp
    from lapis import passes as P
    from lapis.ir import walk
    from lapis.passes import dualview

    # dialect: schema + the sparse.spmv_csr verifier
    dialect._schema(OP)
    setattr(dialect._Verifier, "_verify_" + OP.replace(".", "_"),
            dialect._Verifier._verify_sparse_spmv_csr)
    dialect.SIDE_EFFECT_OPS = tuple(dialect.SIDE_EFFECT_OPS) + (OP,)

    # passes: registry entry, ahead of lower_spmv_csr in the preset
    base_registry = P.registry

    def registry():
        r = base_registry()
        r[PASS] = lower_sparse_to_kernels
        return r

    P.registry = registry
    if PASS not in P.PRESET_PASSES:
        P.PRESET_PASSES = (PASS,) + tuple(P.PRESET_PASSES)

    # DualView management: a device kernel
    dualview._DATA_ACCESS[OP] = ((0, False), (1, False), (2, False), (3, False), (4, True))
    dualview._KERNEL_OPS = tuple(dualview._KERNEL_OPS) + (OP,)

    # emitter: the library call
    def _stmt_spmv(e, op, depth, device, loop_depth):
        args = ", ".join(e.object_name(v) for v in op.operands)
        e.m.line(depth, f"LAPIS::spmv_csr({args});")

    emitter._STMT[OP] = _stmt_spmv

    # interpreter: spmv arithmetic in the device context
    def _h_kokkos_spmv(m, op, env):
        def body():
            interp._h_spmv_csr(m, op, env)

        prev = m.ctx
        m.ctx = "device"
        try:
            if m.eager and prev == "host":
                interp._eager_kernel(m, op, env, body)
            else:
                body()
        finally:
            m.ctx = prev

    interp._DISPATCH[OP] = _h_kokkos_spmv
    base_roots = interp._device_kernel_roots

    def _device_kernel_roots(m, op, env):
        reads, writes = base_roots(m, op, env)
        rd = {id(r): r for r in reads}
        wr = {id(r): r for r in writes}
        for inner in walk(op):
            if inner.name == OP:
                for k, v in enumerate(inner.operands):
                    ref = env.get(v)
                    if isinstance(ref, interp.ViewRef):
                        (wr if k == 4 else rd)[id(ref.root)] = ref.root
        return list(rd.values()), list(wr.values())

    interp._device_kernel_roots = _device_kernel_roots
    _installed = True
