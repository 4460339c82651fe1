"""Reference-API surface of the GPU shim that needs no device (task
validation, cost model, error mapping)."""

import numpy as np
import pytest

import paper_1805_02144_b200 as pkg
from paper_1805_02144_b200 import _native
from paper_1805_02144_b200.phipm import PhiTask, cost_estimate, MatvecOperator


def test_task_validation():
    # test_phipm.py:137-152
    v = [np.ones(3)]
    with pytest.raises(ValueError):
        PhiTask(A=np.eye(3), v=[], rho=[1.0])
    with pytest.raises(ValueError):
        PhiTask(A=np.eye(3), v=[np.zeros(3)], rho=[1.0])
    with pytest.raises(ValueError):
        PhiTask(A=np.eye(3), v=v, rho=[])
    with pytest.raises(ValueError):
        PhiTask(A=np.eye(3), v=v, rho=[0.5, 0.5])
    with pytest.raises(ValueError):
        PhiTask(A=np.eye(3), v=v, rho=[1.5])
    with pytest.raises(ValueError):
        PhiTask(A=np.eye(3), v=v, rho=[1.0], tol=0.0)
    with pytest.raises(ValueError):
        PhiTask(A=np.eye(3), v=[np.ones(3), np.ones(2)], rho=[1.0])


def test_cost_estimate_monotone():
    base = cost_estimate(0.1, 10, 100, 500, 2, 1.0, 1.0, 0.0)
    assert cost_estimate(0.05, 10, 100, 500, 2, 1.0, 1.0, 0.0) > base
    with pytest.raises(ValueError):
        cost_estimate(0.0, 10, 100, 500, 2, 1.0, 1.0, 0.0)


def test_host_callable_operator_routes_to_callback_engine():
    """A MatvecOperator around a host callable becomes the host-callback
    device operator (eik_cb_phipm); one that wraps a device operator keeps it;
    scaling is applied after the product (integrators.py:115-117)."""
    from paper_1805_02144_b200.phipm import HostMatvecOperator, _device_operator
    op = _device_operator(MatvecOperator(lambda x: x, 3, 3))
    assert isinstance(op, HostMatvecOperator) and op.kind == "host"
    s = op.scaled(2.5)
    assert s.scale == 2.5 and s.op is op.op and (s.n, s.nnz) == (3, 3)
    with pytest.raises(TypeError):
        _device_operator(object())


def test_sparse_matrix_reference_surface():
    """kernels.py:49-51, 84-90: identity, @ (sparse and vector), scaled."""
    from paper_1805_02144_b200.sparse import SparseMatrix
    import numpy as np
    I = SparseMatrix.identity(4)
    assert I.nnz == 4 and np.array_equal(I.toarray(), np.eye(4))
    A = SparseMatrix.from_dense(np.arange(16.0).reshape(4, 4))
    B = A @ I
    assert isinstance(B, SparseMatrix) and np.array_equal(B.toarray(), A.toarray())
    x = np.ones(4)
    assert np.array_equal(A @ x, A.toarray() @ x)
    assert np.array_equal(A.scaled(-2.0).toarray(), -2.0 * A.toarray())
    assert A.scaled(0.0).nnz == A.nnz  # scalar scaling keeps explicit zeros


def test_reference_names_exported():
    for name in ("phipm_simul_iom2", "PhiTask", "PhipmResult", "PhipmFailure",
                 "integrate", "step_exprb42", "step_pexprb43", "step_exprb53",
                 "step_epi3", "step_rb_euler", "SemilinearProblem", "EngineSeeds"):
        assert hasattr(pkg, name)


def test_status_mapping():
    _native.load()
    with pytest.raises(ValueError):
        _native.check(_native.EIK_EINVAL)
    with pytest.raises(ValueError):
        _native.check(_native.EIK_ENONFINITE)
    with pytest.raises(_native.NativeError):
        _native.check(_native.EIK_ECUDA)


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_native, "_lib", None)
    monkeypatch.setattr(_native, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(_native.NativeError):
        _native.load()
