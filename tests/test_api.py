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


def test_host_callable_operator_rejected():
    from paper_1805_02144_b200.phipm import _device_operator
    with pytest.raises(TypeError):
        _device_operator(MatvecOperator(lambda x: x, 3, 3))


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
