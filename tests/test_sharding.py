"""Multi-GPU partitioning logic on CPU (gloo, world_size 2): each rank owns
global image indices [r*n, (r+1)*n) and its own corpus (weak scaling, no data
collective); the only collectives are the timing barrier and the max-over-
ranks reduction.  Because every output is a pure function of (seed, global
index, pixels), the union of the ranks' results must equal one process
running all 2n indices -- checked here through the oracle on a small slice."""
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


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from oracle import albref as A
    from synth import configs as C
    from synth import gen
    name, menu, sizes, _ = bench.workload(2, rank)
    n = len(sizes)
    first = rank * n
    # a small slice of this rank's shard through two transforms of the menu
    k = 3
    b = gen.gen_images(sizes[:k], seed=0, first_image_index=first)
    res = {}
    for label in ["Rotate", "Brightness"]:
        outs = A.apply_batch(C.CFG2_MENU[label], 5, first, [b.image(i) for i in range(k)])
        res[label] = [o["image"] for o in outs]
    # timing reduction as bench.py does it (max over ranks)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    np.savez(os.path.join(out_dir, "r%d.npz" % rank), sizes=np.array(sizes[:k]),
             first=first, tmax=t.item(),
             **{"%s_%d" % (l, i): v for l, vs in res.items() for i, v in enumerate(vs)})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_shards_equal_single_process(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    from oracle import albref as A
    from synth import configs as C
    from synth import gen
    n = C.CONFIGS[2]["n"]
    all_sizes = gen.cfg2_sizes(2 * n)
    for r in range(world):
        d = np.load(tmp_path / ("r%d.npz" % r))
        assert int(d["first"]) == r * n
        assert float(d["tmax"]) == float(world)
        assert [tuple(s) for s in d["sizes"]] == all_sizes[r * n:r * n + 3]
        # single process over the same global indices reproduces the shard
        b = gen.gen_images(all_sizes[r * n:r * n + 3], seed=0, first_image_index=r * n)
        for label in ["Rotate", "Brightness"]:
            ref = A.apply_batch(C.CFG2_MENU[label], 5, r * n, [b.image(i) for i in range(3)])
            for i in range(3):
                assert np.array_equal(d["%s_%d" % (label, i)], ref[i]["image"])
