"""The driver's round-end smoke check (__graft_entry__.smoke) must keep passing."""
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)


def test_graft_entry_smoke():
    import __graft_entry__
    __graft_entry__.smoke()
