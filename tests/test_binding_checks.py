"""The Python binding refuses arguments whose raw pointers would read or write out of bounds on
the device: dtype, shape, device and contiguity of every tensor are checked before
anything crosses the C ABI.  Runs on CPU: the checks fire before the library is touched."""
import pytest
import torch

from paper_2302_07992_b200 import mmsb as G


def test_arg_dtype_shape_device():
    ok = torch.zeros(2, 32, dtype=torch.uint8)
    with pytest.raises(G.MmsbError, match="must be torch.uint8"):
        G._arg(ok.to(torch.int32), "k1", torch.uint8, (2, 32))
    with pytest.raises(G.MmsbError, match="shape"):
        G._arg(torch.zeros(2, 16, dtype=torch.uint8), "k1", torch.uint8, (2, 32))   # 128-bit keys
    with pytest.raises(G.MmsbError, match="device tensor"):
        G._arg(ok, "k1", torch.uint8, (2, 32))
    with pytest.raises(G.MmsbError, match="must be torch.int64"):
        G._arg(torch.zeros(2, dtype=torch.int32), "msg_bits", torch.int64, (2,))


def test_calls_check_before_the_library():
    imgs = torch.zeros(2, 16, 16, dtype=torch.uint8)
    with pytest.raises(G.MmsbError):
        G.encode(G.EMR, imgs, torch.zeros(2, 32, dtype=torch.uint8))            # CPU images
    with pytest.raises(G.MmsbError, match=r"\[B, H, W\]"):
        G.recover(G.EMR, torch.zeros(16, 16, dtype=torch.uint8), torch.zeros(1, 32, dtype=torch.uint8))
    with pytest.raises(G.MmsbError):
        G.extract(G.EMR, imgs, torch.zeros(2, 32, dtype=torch.uint8), 24)         # stride % 16


def test_calls_take_the_workspace_tile_size():
    """tile_log2=None (the default of every call) means the workspace's coder tile size, so a
    workspace made for t = 6 is used as it is instead of being re-allocated for t = 7."""

    class FakeWs:
        shape = G._shape(G.LMR, 2, 64, 64, tile_log2=6)

    ws = FakeWs()
    assert G._ws(ws, G.LMR, 2, 64, 64, None, "cpu") is ws
    assert G._ws(ws, G.LMR, 2, 64, 64, 6, "cpu") is ws
