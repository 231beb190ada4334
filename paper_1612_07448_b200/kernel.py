"""Operation counting for the device operators.

GPU kernels do not count their arithmetic, so the ``counter=`` keyword that every
reference operator accepts is filled from closed forms that reproduce the reference's
own tallies exactly (counting conventions at kernel.py:7-18 and indicator.py:1-8 of
the reference; e.g. a dense (m×k)(k×n) product tallies m·k·n multiplies and
m·(k-1)·n additions, an indicator scatter tallies one addition per element).
"""

__all__ = ["OpCounter", "tally_matmul", "tally_accumulate", "tally_rowsums", "tally_colsums"]


class OpCounter:
    """Accumulator for scalar multiply/add counts (kernel.py:46-66)."""

    __slots__ = ("multiplies", "additions")

    def __init__(self, multiplies=0, additions=0):
        self.multiplies = int(multiplies)
        self.additions = int(additions)

    def tally(self, multiplies=0, additions=0):
        self.multiplies += int(multiplies)
        self.additions += int(additions)

    def merge(self, other):
        self.tally(other.multiplies, other.additions)

    def as_dict(self):
        return {"multiplies": self.multiplies, "additions": self.additions}

    def __repr__(self):
        return f"OpCounter(multiplies={self.multiplies}, additions={self.additions})"


def tally_matmul(counter, m, k, n):
    """Dense (m×k)(k×n) product (kernel.py:121-124)."""
    if counter is not None:
        counter.tally(m * k * n, m * max(k - 1, 0) * n)


def tally_accumulate(counter, size):
    if counter is not None:
        counter.tally(0, size)


def tally_rowsums(counter, n, d):
    """Ones-vector row totals (kernel.py:174-182)."""
    if counter is not None:
        mults = n * d
        counter.tally(mults, max(mults - n, 0))


def tally_colsums(counter, n, d):
    """Ones-vector column totals (kernel.py:185-193)."""
    if counter is not None:
        mults = n * d
        counter.tally(mults, max(mults - d, 0))


def tally_crossprod(counter, n, d):
    """Symmetric self-product via syrk (kernel.py:151-153)."""
    if counter is not None:
        counter.tally(n * d * (d + 1) // 2, max(n - 1, 0) * d * (d + 1) // 2)
