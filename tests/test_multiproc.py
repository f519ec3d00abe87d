"""World-size-2 gloo tests of the multi-process host logic (CPU; no GPU, no NCCL data path):
FSDP row sharding, the NCCL unique-id bootstrap over the torch process group, the max-over-ranks
timing reduction bench.py uses, and the oracle identity gathered-shards == unsharded cast
computed per rank and all-gathered over gloo."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import synth
        from oracle import fp8, fsdp as ofsdp
        from paper_2507_16099_b200.fsdp import bootstrap_unique_id, shard_rows

        # 1. row shards tile [0, N) exactly
        N, K = 64, 48
        r0, r1 = shard_rows(N, world, rank)
        spans = [None] * world
        dist.all_gather_object(spans, (r0, r1))
        assert spans[0][0] == 0 and spans[-1][1] == N
        assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))

        # 2. identical NCCL unique id on every rank
        uid = bootstrap_unique_id()
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        assert len(uid) == 128 and all(i == ids[0] for i in ids)

        # 3. global amax by all-reduce MAX of the u32 bit pattern == unsharded amax, and the
        #    gathered shard casts equal the unsharded cast (oracle arithmetic, gloo transport)
        w_shard = synth.weight_shard_c5((N, K), 0, rank, world)
        a_local = np.float32(fp8.amax(w_shard))
        t = torch.tensor([int(np.array([a_local]).view(np.uint32)[0])], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        a_glob = np.array([t.item()], np.uint32).view(np.float32)[0]
        s = fp8.scale_from_amax(a_glob, "e4m3")
        q_local = fp8.cast_scaled(w_shard, s, "e4m3")
        gathered = [torch.empty_like(torch.from_numpy(q_local)) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(q_local))
        q_all = torch.cat(gathered).numpy()
        w_full = synth.tensor_c2("w", (N, K), 0, cfg="c5")
        q1, s1, a1 = fp8.cast_tensorwise(w_full, "e4m3")
        assert a_glob == a1 and s == s1 and np.array_equal(q_all, q1)
        qo, so, ao = ofsdp.allgather_ref([synth.weight_shard_c5((N, K), 0, r, world) for r in range(world)], "e4m3")
        assert np.array_equal(qo, q1)

        # 4. MXFP8 gather: shard-local E8M0 quantization, no amax exchange; the
        #    gloo-gathered dim0 rows / dim1 columns equal the unsharded quantization
        from oracle import mx as omx
        Nm, Km = 64 * world, 64
        wm = synth.tensor_c4("w", (Nm, Km), 4)
        mine = wm[rank * 64:(rank + 1) * 64]
        parts = []
        for arr in (omx.quantize_dim0(mine, "e4m3")[0], omx.quantize_dim1(mine, "e4m3")[1]):
            g = [torch.empty_like(torch.from_numpy(arr)) for _ in range(world)]
            dist.all_gather(g, torch.from_numpy(arr))
            parts.append(g)
        assert np.array_equal(torch.cat(parts[0], 0).numpy(), omx.quantize_dim0(wm, "e4m3")[0])
        assert np.array_equal(torch.cat(parts[1], 1).numpy(), omx.quantize_dim1(wm, "e4m3")[1])

        # 5. max-over-ranks timing reduction (bench.py)
        ms = torch.tensor([1.0 + rank])
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        assert ms.item() == float(world)
        q.put((rank, "ok"))
    except BaseException as e:  # noqa: BLE001
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()[-800:]))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_world2_host_logic(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        try:
            r, v = q.get(timeout=180)
            res[r] = v
        except Exception:  # noqa: BLE001
            break
    for p in procs:
        if p.is_alive():
            p.join(timeout=30)
        if p.is_alive():
            p.kill()
    assert len(res) == world, (res, [p.exitcode for p in procs])
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res
