"""GPU: the C ABI (include/lq.h) refuses bad arguments with a status code and
a message in lq_last_error -- never a crash, never a silent result -- the
contract a latquad-side ctypes binding relies on to raise
the reference's exceptions (ValueError, OverflowError, ...)."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def N():
    from paper_2404_08867_b200 import _native
    return _native


def _err(N, rc, code=None):
    msg = N.lib().lq_last_error().decode()
    assert rc != N.LQ_OK, "bad arguments were accepted"
    if code is not None:
        assert rc == code, (rc, msg)
    assert msg, "no lq_last_error message"
    return msg


def _prog(N, insn):
    ins = np.zeros(len(insn), dtype=N.INSN_DTYPE)
    for k, (op, a, b, n, c) in enumerate(insn):
        ins[k] = (op, a, b, n, c)
    return ins, N.Program(ins.ctypes.data, len(ins), 2, 0, 1, None)


def test_context_errors(N):
    h = N.lib()
    p = C.c_void_p()
    _err(N, h.lq_ctx_create(-1, C.byref(p)), N.LQ_ERR_VALUE)
    _err(N, h.lq_ctx_create(4096, C.byref(p)), N.LQ_ERR_VALUE)
    _err(N, h.lq_ctx_create(0, None), N.LQ_ERR_VALUE)
    _err(N, h.lq_sync(None), N.LQ_ERR_VALUE)
    out = C.c_double()
    _err(N, h.lq_reduce_sum(None, None, 1, C.byref(out)), N.LQ_ERR_VALUE)


def test_points_block_errors(N):
    h, ctx = N.lib(), N.ctx()
    z = np.array([1, 3], dtype=np.uint64)
    buf = np.zeros(16)
    _err(N, h.lq_points_block(ctx, 0, 7, N.as_ptr(z), 0, 4, N.as_ptr(buf), 0), N.LQ_ERR_VALUE)        # d = 0
    _err(N, h.lq_points_block(ctx, 2, 0, N.as_ptr(z), 0, 4, N.as_ptr(buf), 0), N.LQ_ERR_VALUE)        # n = 0
    _err(N, h.lq_points_block(ctx, 2, 3, N.as_ptr(z), 0, 4, N.as_ptr(buf), 0), N.LQ_ERR_VALUE)        # z >= n
    _err(N, h.lq_points_block(ctx, 2, 2**54, N.as_ptr(z), 0, 4, N.as_ptr(buf), 0), N.LQ_ERR_OVERFLOW)
    _err(N, h.lq_points_block(ctx, 2, 7, None, 0, 4, N.as_ptr(buf), 0), N.LQ_ERR_VALUE)
    _err(N, h.lq_points_block(ctx, 2, 7, N.as_ptr(z), 5, 4, N.as_ptr(buf), 0), N.LQ_ERR_VALUE)        # stop < start
    _err(N, h.lq_points_block(ctx, 2, 7, N.as_ptr(z), 0, 4, None, 0), N.LQ_ERR_VALUE)
    assert h.lq_points_block(ctx, 2, 7, N.as_ptr(z), 3, 3, None, 0) == N.LQ_OK                          # empty range


def test_lattice_sum_errors(N):
    import paper_2404_08867_b200 as lq
    from paper_2404_08867_b200 import engine
    h, ctx = N.lib(), N.ctx()
    out = C.c_double()
    z = np.array([1, 3], dtype=np.uint64)
    _err(N, h.lq_lattice_sum(ctx, None, 7, N.as_ptr(z), 0, 7, C.byref(out)), N.LQ_ERR_VALUE)
    pi = engine.plain_integrand(lq.parse("exp(x[1] + 2*x[2])", 2), 2)
    s = pi.struct
    _err(N, h.lq_lattice_sum(ctx, C.byref(s), 2**54, N.as_ptr(z), 0, 7, C.byref(out)), N.LQ_ERR_OVERFLOW)
    _err(N, h.lq_lattice_sum(ctx, C.byref(s), 3, N.as_ptr(z), 0, 3, C.byref(out)), N.LQ_ERR_VALUE)   # z >= n
    bad = N.Integrand.from_buffer_copy(s)
    bad.kind = 99
    _err(N, h.lq_lattice_sum(ctx, C.byref(bad), 7, N.as_ptr(z), 0, 7, C.byref(out)), N.LQ_ERR_VALUE)
    t = C.c_int64()
    _err(N, h.lq_lattice_layout(None, 7, N.as_ptr(z), C.byref(t), None, None, None, None), N.LQ_ERR_VALUE)


def test_tensor_eval_and_mdi_errors(N):
    h, ctx = N.lib(), N.ctx()
    out = C.c_double()
    counts = np.array([4, 0], dtype=np.int64)
    ins, p = _prog(N, [(1, 0, 0, 0, 0.0)])                  # slot0 = x[1]
    _err(N, h.lq_tensor_sum(ctx, None, 2, N.as_ptr(counts), None, 1, 0, 4, C.byref(out)), N.LQ_ERR_VALUE)
    _err(N, h.lq_tensor_sum(ctx, C.byref(p), 2, N.as_ptr(counts), None, 1, 0, 4, C.byref(out)), N.LQ_ERR_VALUE)
    big = np.ones(200, dtype=np.int64)
    _err(N, h.lq_tensor_sum(ctx, C.byref(p), 200, N.as_ptr(big), None, 1, 0, 4, C.byref(out)),
         N.LQ_ERR_UNSUPPORTED)
    col = np.zeros(4)
    res = np.zeros(4)
    table = (C.c_void_p * 1)(col.ctypes.data)
    _err(N, h.lq_eval_array(ctx, C.byref(p), table, -1, 0, N.as_ptr(res)), N.LQ_ERR_VALUE)
    _err(N, h.lq_eval_array(ctx, C.byref(p), table, 4, 0, None), N.LQ_ERR_VALUE)
    _err(N, h.lq_eval_array(ctx, C.byref(p), (C.c_void_p * 1)(None), 4, 0, N.as_ptr(res)), N.LQ_ERR_VALUE)
    assert h.lq_eval_array(ctx, C.byref(p), table, 4, 0, N.as_ptr(res)) == N.LQ_OK
    _err(N, h.lq_mdi_linform(ctx, None, 0, None, None, 0.0, 1.0, 0, 0, 1, None, 0, C.byref(out)), N.LQ_ERR_VALUE)
    _err(N, h.lq_mdi_block_sums(ctx, ins.ctypes.data, 1, None, -1, None, 0, 0, 1, None), N.LQ_ERR_VALUE)


def test_quality_and_jit_errors(N):
    h, ctx = N.lib(), N.ctx()
    out = C.c_double()
    z = np.array([1, 3], dtype=np.uint64)
    g = np.ones(2)
    _err(N, h.lq_bprod_sum(ctx, 3, 2, 7, N.as_ptr(z), N.as_ptr(g), 0.0, 0, 7, C.byref(out)), N.LQ_ERR_VALUE)
    _err(N, h.lq_bprod_sum(ctx, 2, 2, 2**32 + 15, N.as_ptr(z), N.as_ptr(g), 0.0, 0, 7, C.byref(out)),
         N.LQ_ERR_UNSUPPORTED)
    zc = np.zeros(2, dtype=np.int64)
    cands = np.array([1, 9], dtype=np.int64)
    _err(N, h.lq_cbc_construct(ctx, 1, 2, N.as_ptr(g), 0.0, N.as_ptr(cands), 2, N.as_ptr(zc)), N.LQ_ERR_VALUE)
    _err(N, h.lq_cbc_construct(ctx, 7, 2, N.as_ptr(g), 0.0, N.as_ptr(cands), 2, N.as_ptr(zc)), N.LQ_ERR_VALUE)
    vals = np.zeros(2)
    _err(N, h.lq_korobov_values(ctx, 7, 2, N.as_ptr(g), 0.0, N.as_ptr(cands), 2, N.as_ptr(vals)), N.LQ_ERR_VALUE)
    j = C.c_void_p()
    assert h.lq_jit_create(None, b"k", C.byref(j), None, 0) != N.LQ_OK
    log = C.create_string_buffer(4096)
    rc = h.lq_jit_create(b"this is not CUDA", b"k", C.byref(j), log, 4096)
    assert rc != N.LQ_OK
