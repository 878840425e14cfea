"""The NCCL code paths of the N > 1 step on a real GPU (one process, world size 1: every box this
repository is measured on has one B200; the multi-rank logic itself is covered by the gloo
world-2 tests in test_distributed.py).  gather_heads takes its all_gather_into_tensor branch,
exchange_split_rows its SUM / MAX all-reduces and the bench's max-over-ranks reduction its NCCL
all_reduce, all on device tensors."""
import socket

import pytest
import torch
import torch.distributed as dist

from paper_2602_06072_b200 import shard


@pytest.mark.gpu
def test_nccl_paths_world_one():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        assert dist.get_backend() == "nccl"
        g = torch.Generator(device="cuda").manual_seed(5)
        out_local = torch.randn((37, 8 * 4, 128), generator=g, device="cuda").to(torch.bfloat16)
        full = shard.gather_heads(out_local, 1, 8, 4)
        assert torch.equal(full, out_local)
        po = torch.randn((9, 32, 128), generator=g, device="cuda")
        pl = torch.randn((9, 32), generator=g, device="cuda")
        po0, pl0 = po.clone(), pl.clone()
        shard.exchange_split_rows(po, pl, 5)
        assert torch.equal(po, po0) and torch.equal(pl, pl0)
        import bench
        vals = bench.max_over_ranks(torch.device("cuda", 0), 1.5, 2.25)
        assert vals == [1.5, 2.25]
    finally:
        dist.destroy_process_group()
