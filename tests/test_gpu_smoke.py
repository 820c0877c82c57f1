"""The driver's round-end smoke() (one small invocation of the hot path on
cuda:0, checked against the oracle) must pass as part of the GPU suite."""
import pytest

pytestmark = pytest.mark.gpu


def test_graft_entry_smoke():
    import __graft_entry__ as g
    g.smoke()
