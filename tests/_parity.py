"""Tolerance checks shared by the parity tests (test infrastructure).

Reading R-TOL (SURVEY §8(c) ledger #18, BASELINE.json
north_star "within 1e-5 relative"): a matrix of the CUDA path matches its
reference when BOTH
  * ||got - ref||_F / ||ref||_F <= 1e-5          (per matrix), and
  * max |got - ref| <= 1e-5 * max |ref|           (element-wise)
hold. The second bound is the ledger's diagnostic, asserted: a dropped or
mis-ordered late sample (whose update is ~lr_t-sized, small under linear
decay) can hide inside the Frobenius norm but moves single elements.
"""
import numpy as np

TOL = 1e-5


def rel_fro(got, ref):
    ref = np.asarray(ref, np.float64)
    return np.linalg.norm(np.asarray(got, np.float64) - ref) / max(np.linalg.norm(ref), 1e-30)


def max_abs_ratio(got, ref):
    ref = np.asarray(ref, np.float64)
    return np.abs(np.asarray(got, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30)


def assert_matrix_parity(got, ref, what="", tol=TOL):
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    f, m = rel_fro(got, ref), max_abs_ratio(got, ref)
    assert f <= tol and m <= tol, f"{what}: frobenius {f:.3e}, element-wise {m:.3e} (tol {tol:g})"
