"""Native multi-GPU boundary on the device (include/mlora.h mlora_comm_*,
mlora_broadcast_base).  This pool grants one GPU per call and NCCL refuses two
ranks on one device, so the communicator runs at world size 1 here: the calls go
through libmlora.so -> NCCL on cuda:0 end to end (a 1-rank broadcast / sum is
the identity); the rank-0 -> rank-N id rendezvous is covered by the gloo test."""
import pytest
import torch

from paper_2312_02515_b200 import errors as E
from paper_2312_02515_b200 import fused as F
from paper_2312_02515_b200 import parallel as PL

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return F.Context(torch.device("cuda", 0))


def test_world1_comm_broadcast_and_sum(ctx):
    comm = PL.NativeComm(ctx, rank=0, world=1)
    try:
        from paper_2312_02515_b200 import _native as N
        assert N.lib().mlora_comm_rank(comm.handle) == 0 and N.lib().mlora_comm_size(comm.handle) == 1
        dev = ctx.device
        g = torch.Generator(device="cpu").manual_seed(5)
        W = {n: torch.randn(d, k, generator=g).to(torch.bfloat16).to(dev)
             for n, d, k in (("q", 256, 128), ("gate", 688, 128), ("down", 128, 688))}
        ref = {n: t.clone() for n, t in W.items()}
        PL.broadcast_base_weights(W, src=0, comm=comm)
        torch.cuda.synchronize()
        assert all(torch.equal(W[n], ref[n]) for n in W)
        m = torch.arange(16, dtype=torch.float32, device=dev)
        comm.sum_(m)
        torch.cuda.synchronize()
        assert torch.equal(m.cpu(), torch.arange(16, dtype=torch.float32))
        with pytest.raises(E.UsageError):
            comm.broadcast([W["q"]], root=1)  # root outside the 1-rank communicator
        comm.broadcast([])  # empty group is a no-op
    finally:
        comm.close()


def test_comm_create_rejects_bad_rank(ctx):
    with pytest.raises(E.UsageError):
        PL.NativeComm(ctx, rank=1, world=1)
