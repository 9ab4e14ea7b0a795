"""The CUDA twin of the content generator equals the numpy generator byte for byte."""
import numpy as np
import pytest

from kvgen.content import content_tokens

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("layer0,L", [(0, 2), (8, 8), (24, 4)])
def test_cuda_content_equals_numpy(layer0, L):
    from kvgen.cuda import content_tokens_cuda
    rng = np.random.default_rng(layer0)
    ids = rng.integers(0, 3_000_000, size=97)
    pos = rng.integers(0, 3072, size=97)
    want = content_tokens(2601, ids, pos, layer0, L, 8, 128)
    got = content_tokens_cuda(2601, ids, pos, layer0, L, 8, 128, device=0).cpu().numpy()
    assert np.array_equal(got.view(np.uint16), want)
