"""CPU coverage of the multi-GPU path.

1. The owner partition itself, restated over the CPU oracle (oracle/pf_shard_oracle.py):
   a State whose tables are stored as G owner slices replays the reference-generated
   frame fixtures bit for bit -- sources, means, image and every cell.
2. The collective drivers of paper_1902_05942_b200/sharded.py under torch.distributed
   with the gloo backend at world size 2 (two processes): variable-split all-to-alls,
   the overflow retry handshake, the bad-input agreement and the reduce-scatter, with
   the loopback driver (used by the GPU parity tests) checked against them.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import golden_cfg, golden_stream, load_golden

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cfg(oracle, d, key):
    c = golden_cfg(d, key)
    return oracle.Config(**{k: v for k, v in c.items() if k in oracle.Config.__dataclass_fields__})


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("mode", ["fixed", "float"])
@pytest.mark.parametrize("fixture", ["frame_cornell128.npz", "frame_box4.npz"])
def test_owner_partition_replays_reference_frame(oracle, fixture, mode, world):
    from oracle.pf_shard_oracle import ShardedTable, table_cells
    d = load_golden(fixture)
    vs = golden_stream(d)
    cfg = _cfg(oracle, d, f"{mode}_cfg")
    state = oracle.State(ShardedTable.from_config(cfg, world), ShardedTable.from_config(cfg, world))
    img, src, chosen, _ = oracle.filter_frame(vs, cfg, state, 0, int(d["seed"]), int(d["spp"]),
                                              d["base"])
    assert np.array_equal(src, d[f"{mode}_source"])
    assert np.array_equal(chosen, d[f"{mode}_chosen"])
    assert np.array_equal(img, d[f"{mode}_image"])
    for table in ("fine", "coarse"):
        ref = oracle.Table.from_config(cfg)
        for f in ("tags", "sums", "counts", "hist_sums", "hist_counts", "last_touch", "deltas"):
            getattr(ref, f)[...] = d[f"{mode}_{table}_{f}"]
        assert getattr(state, table).cells() == table_cells(ref)


def test_owner_partition_temporal_corridor_single_owner(oracle):
    """Eviction-heavy fixture (capacity 128, probe_limit 4): with one owner the slice
    layout is the global table itself, so even evictions replay exactly."""
    from oracle.pf_shard_oracle import ShardedTable
    d = load_golden("temporal_corridor.npz")
    cfg = _cfg(oracle, d, "filter_cfg")
    state = oracle.State(ShardedTable.from_config(cfg, 1), ShardedTable.from_config(cfg, 1))
    for f in range(int(d["frames"])):
        vs = golden_stream(d, f"f{f}_v_")
        img, src, _, _ = oracle.filter_frame(vs, cfg, state, f, int(d[f"f{f}_seed"]), 1,
                                             d[f"f{f}_base"])
        assert np.array_equal(src, d[f"filter_f{f}_source"])
        assert np.array_equal(img, d[f"filter_f{f}_image"])


# ------------------------------------------------------------------ gloo drivers

def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def protocol(rank: int, world: int, overflow_once: bool):
    """A frame-shaped collective sequence (sharded.filter_frame_sharded's exchanges
    with host tensors): counts + flags, records and requests with ragged splits, an
    overflow retry, answers back, a reduce-scatter.  Returns what it received."""
    from paper_1902_05942_b200.sharded import AllGather, Exchange, ReduceScatter
    G = world
    got = {}
    overflowed = overflow_once and rank == 0
    while True:
        counts = torch.tensor([[(rank + 1) * (p + 1), rank + 2 * p, int(overflowed), 0]
                               for p in range(G)], dtype=torch.int64)
        recv = yield Exchange(counts, [1] * G, [1] * G)
        if not recv[:, 2].any():
            break
        got["retries"] = got.get("retries", 0) + 1
        overflowed = False
    send_rec = counts[:, 0].tolist()
    recv_rec = recv[:, 0].tolist()
    recs = torch.cat([torch.full((send_rec[p], 5), 1000 * rank + p, dtype=torch.int64)
                      for p in range(G)])
    got["records"] = (yield Exchange(recs, send_rec, recv_rec)).clone()
    send_req, recv_req = counts[:, 1].tolist(), recv[:, 1].tolist()
    reqs = torch.cat([torch.arange(send_req[p], dtype=torch.int64) + 100 * rank + 10 * p
                      for p in range(G)]) if sum(send_req) else torch.zeros(0, dtype=torch.int64)
    requests = yield Exchange(reqs, send_req, recv_req)
    got["requests"] = requests.clone()
    answers = torch.stack([requests, requests * 2, requests * 3, -requests], 1) \
        if len(requests) else torch.zeros((0, 4), dtype=torch.int64)
    back = yield Exchange(answers, recv_req, send_req)
    got["answers"] = back.clone()
    got["reqs_sent"] = reqs
    got["gathered"] = (yield AllGather(torch.full((3, 6), 7 + rank, dtype=torch.int64))).clone()
    flat = torch.arange(8 * G * 3, dtype=torch.float64).reshape(8 * G, 3) * (rank + 1)
    got["band"] = (yield ReduceScatter(flat)).clone()
    return got


def _expected_answers(reqs):
    return torch.stack([reqs, reqs * 2, reqs * 3, -reqs], 1)


def _worker(rank, world, port, overflow_once, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1902_05942_b200.sharded import run_dist
        got = run_dist(protocol(rank, world, overflow_once))
        torch.save(got, os.path.join(out_dir, f"rank{rank}.pt"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("overflow_once", [False, True])
def test_gloo_world2_drivers_match_loopback(tmp_path, overflow_once):
    from paper_1902_05942_b200.sharded import run_loopback
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), overflow_once, str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    dist_res = [torch.load(tmp_path / f"rank{r}.pt") for r in range(world)]
    loop_res = run_loopback([protocol(r, world, overflow_once) for r in range(world)])
    for a, b in zip(dist_res, loop_res):
        assert a.keys() == b.keys()
        for k in a:
            if isinstance(a[k], torch.Tensor):
                assert torch.equal(a[k], b[k]), k
            else:
                assert a[k] == b[k], k
    for r, got in enumerate(dist_res):
        # records from rank p to r are filled with 1000*p + r, in rank order
        want = torch.cat([torch.full(((p + 1) * (r + 1), 5), 1000 * p + r, dtype=torch.int64)
                          for p in range(world)])
        assert torch.equal(got["records"], want)
        # the answers come back aligned with the requests this rank sent
        assert torch.equal(got["answers"], _expected_answers(got["reqs_sent"]))
        full = sum(torch.arange(8 * world * 3, dtype=torch.float64).reshape(8 * world, 3) * (p + 1)
                   for p in range(world))
        assert torch.equal(got["band"], full[8 * r:8 * (r + 1)])
        assert torch.equal(got["gathered"], torch.cat([torch.full((3, 6), 7 + p, dtype=torch.int64)
                                                       for p in range(world)]))
        if overflow_once:
            assert got["retries"] == 1
