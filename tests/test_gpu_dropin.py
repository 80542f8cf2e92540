"""The drop-in, end to end against the LIVE reference on the GPU box: the unmodified reference
package installed in baseline/_ref (the reference arm's pip install; skipped when absent) gets the
one-line binding INTEGRATION.md shows -- ``run_method`` learns the ``*_b200`` method names -- and the
reference's own harness (E/harness.py:83-144: make_example, run_method) then solves each catalog
example through the B200 engine.  phi bytes, the in-place grid mutation and every RunStats field
must equal the reference's own solver run on an identical grid in the same process."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
if not os.path.isdir(os.path.join(REF, "eikonal")):
    pytest.skip("reference install (baseline/_ref) absent", allow_module_level=True)


@pytest.fixture(scope="module")
def harness():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from eikonal import harness as h

    import paper_2106_15869_b200 as b200

    stock = h.run_method

    def run_method(method, grid, bc, tol=1e-12, workers=1):  # the binding of INTEGRATION.md
        if method in ("ifim_b200", "fim_b200", "oracle_b200"):
            return b200.run_method(method[:-5], grid, bc, tol=tol, workers=workers)
        return stock(method, grid, bc, tol=tol, workers=workers)

    h.run_method = run_method
    yield h
    h.run_method = stock


@pytest.mark.parametrize("method", ["ifim", "fim", "oracle"])
@pytest.mark.parametrize("example,n", [(1, 128), (2, 128), (3, 128), (4, 96), (5, 128)])
def test_reference_harness_through_the_b200_engine(harness, example, n, method):
    g_ref, bc_ref = harness.make_example(example, n)
    ref = harness.run_method(method, g_ref, bc_ref)
    g, bc = harness.make_example(example, n)
    got = harness.run_method(method + "_b200", g, bc)
    assert np.array_equal(np.asarray(got.phi).view(np.uint64), np.asarray(ref.phi).view(np.uint64))
    assert np.array_equal(g.phi.view(np.uint64), g_ref.phi.view(np.uint64))  # mutated in place
    assert np.array_equal(g.state, g_ref.state)  # SOURCE marks (E/grid.py:215)
    s, r = got.stats, ref.stats
    assert (s.iterations, s.solver_calls, s.peak_active, s.peak_remedy) == \
        (r.iterations, r.solver_calls, r.peak_active, r.peak_remedy)
    if method == "ifim":
        assert list(s.active_history) == list(r.active_history)
