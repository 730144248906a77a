"""The driver's round-end smoke check (__graft_entry__.smoke) as a GPU test, so a change that
breaks it (e.g. a new value on a debug surface) fails the suite, not only the round end."""
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


def test_graft_entry_smoke():
    import __graft_entry__

    __graft_entry__.smoke()
