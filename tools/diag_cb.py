"""Diagnostic: each operator wrapper of test_engine_accepts_sparse_and_operator_inputs alone."""
import sys
import numpy as np
import scipy.sparse as sp
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from paper_1805_02144_b200.phipm import PhiTask, phipm_simul_iom2, MatvecOperator
from paper_1805_02144_b200.sparse import SparseMatrix
rng = np.random.default_rng(23)
n = 40
Q = np.linalg.qr(rng.standard_normal((n, n)))[0]
A = Q @ np.diag(-np.logspace(0, 3, n)) @ Q.T
v = [rng.standard_normal(n) for _ in range(4)]
ref = phipm_simul_iom2(PhiTask(A=A, v=v, rho=[1.0], tol=1e-8))
print("ref", ref.substeps, ref.rejections, ref.matvecs, ref.m_final)
for rep in range(3):
    for name, w in (("SparseMatrix", SparseMatrix.from_dense(A)), ("scipy", sp.csr_matrix(A)),
                    ("callable", MatvecOperator(lambda x: A @ x, A.shape[0], A.size))):
        r = phipm_simul_iom2(PhiTask(A=w, v=v, rho=[1.0], tol=1e-8))
        print(rep, name, r.substeps, r.rejections, r.matvecs, r.m_final,
              float(np.max(np.abs(r.W - ref.W))))
