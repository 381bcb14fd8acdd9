"""GPU test of the data-parallel step's host logic with real CUDA streams: two
ranks on the one B200 (gloo carries the all-reduce here -- NCCL needs one GPU
per rank), heterogeneous mirrored plans, different data per rank, eager
TrainStep with the overlapped bucket all-reduce, the wgrad side stream and the
bucket-wise optimizer on the comm stream.  After every step the two ranks must
hold bit-identical weights (every bucket reduced, in order, before its
optimizer ran) and the loss must be finite."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2407_02327_b200.qlinear import FP16, INT8
    from paper_2407_02327_b200.train_step import BertConfig, BertEncoderStack, TrainStep, mixed_plan
    cfg = BertConfig(vocab=1000, hidden=256, layers=3, heads=4, ffn=1024, max_pos=128, seq=128)
    torch.manual_seed(0)
    m = BertEncoderStack(cfg).cuda()
    plan = mixed_plan(cfg)
    if rank == 1:
        plan = {k: ({INT8: FP16, FP16: INT8}.get(v, v)) for k, v in plan.items()}
    m.apply_plan(plan)
    st = TrainStep(m, batch=4, world=world, lr=1e-3, graph=False, fused=True)
    assert st.overlap_opt
    g = torch.Generator().manual_seed(10 + rank)
    st.tokens.copy_(torch.randint(0, cfg.vocab, (4, cfg.seq), generator=g))
    st.labels.copy_(torch.randint(0, 2, (4,), generator=g))
    res = {"losses": [], "diff": []}
    for _ in range(3):
        res["losses"].append(float(st().item()))
        torch.cuda.synchronize()
        flat = torch.cat([p.detach().flatten() for p in m.parameters()]).cpu()
        other = flat.clone()
        dist.broadcast(other, src=0)
        res["diff"].append(float((flat - other).abs().max()))
    res["buckets"] = len(st.grads.buckets)
    res["log"] = st.grads.issue_log
    torch.save(res, os.path.join(out, f"r{rank}.pt"))
    dist.destroy_process_group()


def test_dp_two_ranks_identical_weights(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0 = torch.load(tmp_path / "r0.pt")
    r1 = torch.load(tmp_path / "r1.pt")
    assert r0["log"] == r1["log"] and [b for b, _ in r0["log"]] == list(range(r0["buckets"]))
    assert all(d == 0.0 for d in r1["diff"]), r1["diff"]
    assert all(abs(x) < 10 for x in r0["losses"] + r1["losses"])
