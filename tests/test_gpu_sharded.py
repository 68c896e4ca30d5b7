"""GPU: the sharded device path (cqb_shard_* + cqb_finalize_moments) run as W
virtual shards on one GPU equals the oracle / single-GPU run — the exactness
that makes the N-GPU run bit-identical (integer moments, fixed finalize)."""
import numpy as np
import pytest

from paper_1011_0093_b200 import api
from paper_1011_0093_b200.configs import gmm_image, uniform_image
from paper_1011_0093_b200.distributed import DeviceShardBackend, run_wsm_sharded

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shards", [1, 2, 4, 7])
def test_device_shards_match_oracle(shards, port):
    img = gmm_image(128, 64, 24, 8)  # P = 8192
    h = port.build_histogram(img)
    ref = port.run_wsm(h.keys, h.counts, 8192, 16, mode=1, seed=1, trajectory=True)
    res = run_wsm_sharded(DeviceShardBackend(), img, 16, shards=shards)
    assert res.iterations == ref.iterations
    np.testing.assert_array_equal(res.centers, ref.centers)
    assert res.dist_evals == ref.dist_evals
    np.testing.assert_allclose(res.sse_history, ref.sse_history, rtol=1e-9)


def test_device_shards_k256_uniform(port):
    img = uniform_image(256, 256, 21)  # P = 65536, N' ~ 65K, K = 256
    single = api.quantize(img, 256, api.Termination.convergent(1e-4, 100), seed=1, index_map=False, mapped=False)
    res = run_wsm_sharded(DeviceShardBackend(), img, 256, shards=3)
    assert res.iterations == single.report.iterations
    np.testing.assert_array_equal(res.centers, single.palette)
    assert res.dist_evals == single.report.dist_evals
