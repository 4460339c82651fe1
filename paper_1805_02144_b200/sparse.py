"""Host-side CSR container with the reference's ``SparseMatrix`` surface.

The reference's operator plug point (kernels.py:34-96) is a CSR wrapper
exposing ``matvec``, ``nnz``, ``row_offsets``/``col_indices``/``values`` and
``csr``.  The sphere grid (grid.py) hands its operators over in this form so
that both the CPU oracle and the reference itself can consume them
unchanged; the GPU path only reads the raw CSR arrays once, when the C-ABI
context is created (``eik_swe_create``), and never multiplies with them.
"""

import numpy as np
import scipy.sparse


class SparseMatrix:
    """Real CSR matrix (mirrors expintkit.kernels.SparseMatrix, kernels.py:34)."""

    __slots__ = ("csr",)

    def __init__(self, mat):
        csr = scipy.sparse.csr_matrix(mat, dtype=float)
        if csr.nnz and not np.all(np.isfinite(csr.data)):
            raise ValueError("SparseMatrix entries must be finite")
        self.csr = csr

    @classmethod
    def identity(cls, n):
        """kernels.py:49-51."""
        return cls(scipy.sparse.identity(n, format="csr"))

    @classmethod
    def from_dense(cls, a):
        return cls(np.asarray(a, dtype=float))

    @property
    def n_rows(self):
        return self.csr.shape[0]

    @property
    def n_cols(self):
        return self.csr.shape[1]

    @property
    def nnz(self):
        return self.csr.nnz

    @property
    def row_offsets(self):
        return self.csr.indptr

    @property
    def col_indices(self):
        return self.csr.indices

    @property
    def values(self):
        return self.csr.data

    def matvec(self, x):
        return self.csr @ x

    def __matmul__(self, other):
        """kernels.py:84-87: SparseMatrix @ SparseMatrix stays sparse."""
        if isinstance(other, SparseMatrix):
            return SparseMatrix(self.csr @ other.csr)
        return self.csr @ other

    def scaled(self, alpha):
        """kernels.py:89-90: alpha * M, entries kept as scipy keeps them
        (scalar scaling keeps explicit zeros, so nnz is unchanged)."""
        return SparseMatrix(self.csr * float(alpha))

    def toarray(self):
        return self.csr.toarray()

    def __repr__(self):
        return f"SparseMatrix({self.n_rows}x{self.n_cols}, nnz={self.nnz})"
