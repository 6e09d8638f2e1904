"""General CSR triple product P^T K P (scipy csr_matmat order) -- placeholder."""

from __future__ import annotations


def ptap(P, K):
    raise NotImplementedError("general device SpGEMM lands in the next commit")
