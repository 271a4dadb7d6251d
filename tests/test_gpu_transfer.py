"""Host <-> device staging of the public fit() (device.upload_host /
download_host): the reference's float64 inputs go up through reused pinned
buffers with the cast on the device, factors come back the same way --
values exact, chunk boundaries and 1-D / 2-D shapes included."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape,src,dst", [((1000, 37), np.float64, torch.float32),
                                           ((1000, 37), np.float64, torch.float64),
                                           ((12345,), np.int64, torch.int64),
                                           ((7,), np.float64, torch.float32),
                                           ((0, 5), np.float64, torch.float32)])
@pytest.mark.parametrize("chunk", [4096, 128 << 20])
def test_upload_download_roundtrip(shape, src, dst, chunk):
    from paper_1506_08938_b200 import device as D

    dev = D.require_cuda()
    rng = np.random.default_rng(sum(shape) + chunk)
    a = (rng.standard_normal(shape) * 1e3).astype(src)
    t = D.upload_host(a, dst, dev, chunk_bytes=chunk)
    assert tuple(t.shape) == shape and t.dtype == dst
    want = torch.from_numpy(a).to(dst)
    assert torch.equal(t.cpu(), want)
    back = D.download_host(t, chunk_bytes=chunk)
    assert back.shape == shape
    assert np.array_equal(back, want.numpy())
