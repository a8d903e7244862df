"""CPU, world_size 2 over gloo: the multi-GPU element partition.

Mirrors the reference's determinism guarantee (test_assembly.cpp:392-403,
acceptance.cpp:242-261): each rank fills its own contiguous element range,
no data crosses ranks, and the per-element results are bitwise those of the
single-process fill; the timing reduction is a max over ranks."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1703_09619_b200.dist import element_range, weak_range


def test_partition_covers_each_element_once():
    for total in (1, 7, 4096, 262144):
        for world in (1, 2, 4, 8):
            seen = []
            for r in range(world):
                a, b = element_range(r, world, total)
                seen.extend(range(a, b))
            assert seen == list(range(total))
    assert weak_range(3, 4096) == (3 * 4096, 4 * 4096)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_1703_09619_b200.dist import element_range, max_over_ranks

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    total = 7
    a, b = element_range(rank, world, total)
    o = O.Oracle(3, (3, 3, 2), [O.PP, O.DD], (5, 5, 4))
    alpha = o.alpha(O.ALPHA_JACOBIAN, 0.5, 3.0, 42, a, b - a)   # counter-based: rank-local
    M = o.fill(alpha)
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), M)
    t = max_over_ranks(float(rank + 1))
    if rank == 0:
        np.save(os.path.join(out_dir, "tmax.npy"), np.array([t]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_fill_equals_serial(tmp_path):
    from oracle import oracle as O
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       start_method="spawn")
    parts = [np.load(tmp_path / f"rank{r}.npy") for r in range(world)]
    got = np.concatenate(parts)
    o = O.Oracle(3, (3, 3, 2), [O.PP, O.DD], (5, 5, 4))
    ref = o.fill(o.alpha(O.ALPHA_JACOBIAN, 0.5, 3.0, 42, 0, 7))
    assert np.array_equal(got, ref)
    assert float(np.load(tmp_path / "tmax.npy")[0]) == 2.0
