"""Multi-process (world_size 2, gloo, CPU) tests of the sentence-sharding plumbing that
bench.py and multi-GPU certification use.  The per-sentence work is the C restatement of
the reference pass (the GPU path is exercised by the -m gpu tests)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2209_12708_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle.oracle import ModelConfig, Oracle
    from paper_2209_12708_b200 import dist as Dm
    dist = Dm.init(backend="gloo")
    info = Dm.rank_info()
    # 1) bench sentence blocks: disjoint across ranks and steps
    ids = [i for step in range(3) for i in Dm.sentence_block(info.rank, step, 3, 4)]
    allids = [None] * world
    dist.all_gather_object(allids, ids)
    # 2) max over ranks of device times
    mx = Dm.max_over_ranks([1.0 + info.rank, 5.0 - info.rank], dist)
    # 3) sharded certification of 5 sentences (C restatement of the reference pass)
    o = Oracle("port")
    cfg = ModelConfig(1, 2, 16, 32, 8)
    params = o.gen_model(cfg, 11)

    def work(r):
        out = []
        for s in r:
            x = o.gen_input(cfg, 2000 + s)
            pos = o.gen_positions(3000 + s, cfg.length, 1)
            st, lo, hi, _, _ = o.bound_pass(cfg, params, x, pos, "linf", 0.02)
            out.append((s, st, lo.tolist(), hi.tolist()))
        return out

    res = Dm.run_sharded(5, work, dist)
    q.put((info.rank, allids, mx, res))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_partitions():
    for n in (0, 1, 5, 8, 17):
        for w in (1, 2, 3, 8):
            parts = [list(D.shard(n, r, w)) for r in range(w)]
            flat = [i for p in parts for i in p]
            assert flat == list(range(n))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_world2_gloo_sharding(port_oracle=None):
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        rank, allids, mx, res = q.get(timeout=240)
        out[rank] = (allids, mx, res)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    allids = out[0][0]
    flat = [i for ids in allids for i in ids]
    assert len(flat) == len(set(flat)) == 2 * 3 * 4
    assert out[0][1] == out[1][1] == [2.0, 5.0]
    res = out[0][2]
    assert out[1][2] is None
    assert [r[0] for r in res] == list(range(5))
    # results gathered across ranks equal a single-process run
    from oracle.oracle import ModelConfig, Oracle
    o = Oracle("port")
    cfg = ModelConfig(1, 2, 16, 32, 8)
    params = o.gen_model(cfg, 11)
    for s, st, lo, hi in res:
        x = o.gen_input(cfg, 2000 + s)
        pos = o.gen_positions(3000 + s, cfg.length, 1)
        st2, lo2, hi2, _, _ = o.bound_pass(cfg, params, x, pos, "linf", 0.02)
        assert st == st2 and np.array_equal(lo, lo2) and np.array_equal(hi, hi2)


def _col_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np
    import torch
    from oracle.oracle import Oracle
    from paper_2209_12708_b200 import dist as Dm
    from paper_2209_12708_b200 import faith_gpu as F
    dist = Dm.init(backend="gloo")
    info = Dm.rank_info()
    o = Oracle("port")
    out = {}
    # 1) concretization of column-split Λ with all-reduced partials == full concretization
    rng = np.random.default_rng(5)
    n, d = 37, 64
    lw, uw = rng.uniform(-1, 1, (n, d)), rng.uniform(-1, 1, (n, d))
    lb, ub = rng.uniform(-1, 0, n), rng.uniform(0, 1, n)
    cols = Dm.column_range(d, info.rank, info.world)
    for norm in ("l1", "l2", "linf"):
        pl = torch.tensor(Dm.partial_norms(lw[:, cols.start:cols.stop], norm))
        pu = torch.tensor(Dm.partial_norms(uw[:, cols.start:cols.stop], norm))
        op = dist.ReduceOp.MAX if Dm.reduce_op(norm) == "max" else dist.ReduceOp.SUM
        dist.all_reduce(pl, op=op)
        dist.all_reduce(pu, op=op)
        lo = lb - 0.3 * Dm.finish_norms(pl.numpy(), norm)
        hi = ub + 0.3 * Dm.finish_norms(pu.numpy(), norm)
        out[norm] = (lo, hi, o.concretize(lw, lb, uw, ub, norm, 0.3))
    # 2) the NCCL unique-id handshake of shard_model_columns (broadcast from rank 0)
    box = [F.nccl_unique_id() if info.rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    out["uid"] = box[0]
    q.put((info.rank, out, list(cols)))
    dist.barrier()
    dist.destroy_process_group()


def test_world2_gloo_column_shard_host_logic():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_col_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, out, cols = q.get(timeout=240)
        res[rank] = (out, cols)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] + res[1][1] == list(range(64))
    assert res[0][0]["uid"] == res[1][0]["uid"] and len(res[0][0]["uid"]) == 128
    for norm in ("l1", "l2", "linf"):
        for r in range(world):
            lo, hi, (plo, phi) = res[r][0][norm]
            assert np.allclose(lo, plo, rtol=0, atol=1e-12) and np.allclose(hi, phi, rtol=0, atol=1e-12)


def test_column_range_rules():
    assert list(D.column_range(16, 1, 2)) == list(range(8, 16))
    with pytest.raises(ValueError):
        D.column_range(1536, 0, 16 * 7)
    assert D.reduce_op("l1") == "max" and D.reduce_op("l2") == "sum" and D.reduce_op("linf") == "sum"


def test_bench_spawns_ranks_itself():
    """`bench.py --gpus 2` outside torchrun re-launches itself under torch.distributed.run with two
    ranks (here with --dry-run: gloo, no GPU work); rank 0 prints one JSON line for the job."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                           "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run", "--steps", "2"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["config"]["global_batch"] == 128
    # rank 1's first sentence block starts after rank 0's steps (disjoint, rank-major)
    assert rec["max_first_sentence_over_ranks"] == (2 + 3) * 64
