"""The sharded driver on the GPU with a real NCCL process group.

Only one GPU is available to the build and the round-end tests, so the group
has ONE rank: everything but the peer transfers runs -- the NCCL group, the
per-attempt object exchanges, the device path of the restart loop, the
destination side of gather_columns and the device assembly of the gathered
block (hsrq_pack_download).  The result must equal the single-process
hsrq3in bit for bit (the world-2 exchange logic is covered on CPU ranks by
test_parallel_gloo.py)."""

import os

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def nccl_group():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as dist

    if dist.is_initialized():
        pytest.skip("a process group already exists in this process")
    torch.cuda.set_device(0)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def test_sharded_driver_one_rank_nccl_equals_hsrq3in(nccl_group):
    from paper_2101_05063_b200 import InviterConfig, hsrq3in
    from paper_2101_05063_b200.parallel import gather_columns, hsrq3in_distributed

    g = golden("inviter")
    for h, eigs, cfg in ((g["h1_h"], g["h1_eigs"], InviterConfig(b_r=8, b_c=4)),
                         (g["c1_h"], g["c1_shifts"], InviterConfig(b_r=32))):
        want = hsrq3in(h, eigs, cfg)
        got = hsrq3in_distributed(h, eigs, cfg)
        assert np.array_equal(got.converged, want.converged)
        assert np.array_equal(got.restarts, want.restarts)
        assert np.array_equal(got.vectors, want.vectors)
        assert np.array_equal(got.segment_exp, want.segment_exp)
        assert np.array_equal(got.alpha_exp, want.alpha_exp)
        assert np.array_equal(got.log2_norms, want.log2_norms)
        assert got.extras["ranks"] == 1 and got.extras["gathered_bytes"] == 0
    # the destination side of the gather on device tensors
    X = torch.arange(12, dtype=torch.float64, device="cuda").reshape(3, 4)
    out = gather_columns(X, [3], dst=0)
    assert torch.equal(out, X)
