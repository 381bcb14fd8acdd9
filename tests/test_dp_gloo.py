"""Multi-process (world size 2, gloo, CPU) tests of the DP host logic: the flat
FP32 gradient buffer, bucket order (reverse topological, identical on every
rank whatever its precision plan), 64-byte slot alignment and the averaging
all-reduce (Eq. 6 slot semantics, replayer.cpp:48-62)."""
import json
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_02327_b200.qlinear import FP16, FP32, INT8
from paper_2407_02327_b200.train_step import (BertConfig, FlatGrads, adjustable_ops, load_plan,
                                              mixed_plan)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _params(seed_shape_only=True):
    torch.manual_seed(0)
    shapes = [(2,), (2, 768), (768,), (3072, 768), (768, 3072), (768,), (2304, 768), (2304,)]
    return [torch.nn.Parameter(torch.randn(*s)) for s in shapes]


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    params = _params()
    g = FlatGrads(params, bucket_bytes=4 << 20)
    # every rank fills its grads differently (as different precision plans would)
    for i, p in enumerate(params):
        p.main_grad.copy_(torch.full_like(p, float(rank + 1) * (i + 1)))
    g.allreduce(world)
    res = {
        "buckets": g.buckets,
        "offsets": [int(p.main_grad.data_ptr() - g.flat.data_ptr()) for p in params],
        "vals": [float(p.grad.flatten()[0]) for p in params],
        "same_storage": all(p.grad.data_ptr() == p.main_grad.data_ptr() for p in params),
    }
    with open(os.path.join(out_dir, f"r{rank}.json"), "w") as f:
        json.dump(res, f)
    dist.destroy_process_group()


def test_flat_grads_allreduce_world2(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0 = json.load(open(tmp_path / "r0.json"))
    r1 = json.load(open(tmp_path / "r1.json"))
    assert r0["buckets"] == r1["buckets"]            # identical bucket layout on all ranks
    assert r0["offsets"] == r1["offsets"]
    assert all(o % 64 == 0 for o in r0["offsets"])   # 64-byte aligned slots (TMA reduce-add)
    # reverse topological order: the last parameter sits first in the flat buffer
    assert r0["offsets"][-1] == 0 and r0["offsets"] == sorted(r0["offsets"], reverse=True)
    # average of (rank+1)*(i+1) over ranks 1, 2 -> 1.5 * (i+1)
    for i, v in enumerate(r0["vals"]):
        assert v == pytest.approx(1.5 * (i + 1))
    assert r0["vals"] == r1["vals"]
    assert r0["same_storage"]
    # buckets tile the buffer contiguously
    b = r0["buckets"]
    assert b[0][0] == 0 and all(b[i][1] == b[i + 1][0] for i in range(len(b) - 1))


def test_plan_file_formats(tmp_path):
    cfg = BertConfig(layers=2)
    bare = {"per_device": {"infer": {"layer0.qkv": "INT8", "layer1.ff2": "FP16"}}}
    p = tmp_path / "plan.json"
    p.write_text(json.dumps(bare))
    plan = load_plan(str(p), "infer")
    assert plan == {"layer0.qkv": INT8, "layer1.ff2": FP16}
    report = {"devices": {"infer": {"layer0.o": "FP32"}}, "omega_before": 1.0}
    p.write_text(json.dumps(report))
    assert load_plan(str(p), "infer") == {"layer0.o": FP32}
    with pytest.raises(KeyError, match="reference"):
        load_plan(str(p), "nope")
    p.write_text(json.dumps({"per_device": {"d": {"x": "INT4"}}}))
    with pytest.raises(ValueError, match="unknown precision"):
        load_plan(str(p), "d")
    mp_ = mixed_plan(cfg)
    assert set(mp_) == set(adjustable_ops(cfg))
    assert mp_["layer0.qkv"] == INT8 and mp_["layer1.qkv"] == FP16 and mp_["pooler"] == FP32


def _worker_overlap(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    params = _params()
    g = FlatGrads(params, bucket_bytes=4 << 20)
    finals = []
    g.begin(world, on_final=lambda b: finals.append((b, float(g.flat[g.buckets[b][0]]))))
    issued_after = []
    # backward order = reverse of the forward parameter order; grads become final
    # one parameter at a time, as the layers' backward passes report them
    for i, p in enumerate(reversed(params)):
        p.main_grad.copy_(torch.full_like(p, float(rank + 1) * (i + 1)))
        g.params_ready([p])
        issued_after.append(g._next)
    g.finish()
    first = {"issued_after": issued_after, "log": g.issue_log, "finals": finals,
             "expect_first": [float(g.flat[a]) for a, _ in g.buckets],
             "bucket_of": [g.bucket_of[id(p)] for p in reversed(params)],
             "vals": [float(p.main_grad.flatten()[0]) for p in reversed(params)]}
    # second pass: only the first two parameters report; finish() forces the rest
    g.zero()
    g.begin(world)
    for i, p in enumerate(reversed(params)):
        p.main_grad.fill_(float(rank + 1))
    g.params_ready(list(reversed(params))[:2])
    partial = g._next
    g.finish()
    second = {"partial": partial, "log": g.issue_log,
              "vals": [float(p.main_grad.flatten()[0]) for p in params]}
    with open(os.path.join(out_dir, f"o{rank}.json"), "w") as f:
        json.dump({"first": first, "second": second, "nb": len(g.buckets)}, f)
    dist.destroy_process_group()


def test_overlapped_bucket_allreduce_world2(tmp_path):
    """Bucket n is reduced as soon as its last parameter is final and bucket
    n-1 was issued (in order, identical on both ranks); the averaged result
    equals the non-overlapped all-reduce; finish() forces the rest."""
    port = _free_port()
    mp.spawn(_worker_overlap, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0 = json.load(open(tmp_path / "o0.json"))
    r1 = json.load(open(tmp_path / "o1.json"))
    f0 = r0["first"]
    assert f0["log"] == r1["first"]["log"]
    nb = r0["nb"]
    assert [b for b, _ in f0["log"]] == list(range(nb))       # every bucket once, in order
    assert all(pending == 0 for _, pending in f0["log"])      # never before its grads were final
    # issued exactly when the bucket's last parameter reported
    bo = f0["bucket_of"]
    for i, n_issued in enumerate(f0["issued_after"]):
        done = i == len(bo) - 1 or bo[i + 1] != bo[i]
        assert n_issued == (bo[i] + 1 if done else bo[i])
    for i, v in enumerate(f0["vals"]):
        assert v == pytest.approx(1.5 * (i + 1))
    # the per-bucket hook (the bucket-wise optimizer) runs once per bucket, in
    # order, and sees the already-averaged gradients
    assert [b for b, _ in f0["finals"]] == list(range(nb))
    assert [v for _, v in f0["finals"]] == pytest.approx(f0["expect_first"])
    s0 = r0["second"]
    assert s0["partial"] <= 1 and [b for b, _ in s0["log"]] == list(range(nb))
    assert all(v == pytest.approx(1.5) for v in s0["vals"])
