"""GPU: the graft smoke path (device twin == host twin, K-scan, window, attention)."""
import pytest

pytestmark = pytest.mark.gpu


def test_smoke_entry():
    import __graft_entry__ as g
    g.smoke()
