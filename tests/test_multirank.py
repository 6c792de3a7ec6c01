"""N>1 path on CPU: world_size-2 gloo processes, each an independent HP/BE
pair (here on the CPU oracle device), aggregated exactly as bench.py does."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        import paper_2410_07381_b200 as P
        from oracle import gpu_model as gm
        gpu = P.GpuSpec(4, 128, 1)
        hp = P.TaskScript("hp", P.HIGH, (P.KernelWork("hp_k", P.cost_model(1.0, 1, 128)),),
                          tuple(P.ms_to_ns(x) for x in (0.5, 3.0 + rank, 7.7)))
        be = P.TaskScript("be", P.BEST_EFFORT, (P.KernelWork("be_k", P.cost_model(0.15, 108, 128)),))
        prof = P.Profiler(gpu, device_factory=gm.GpuSim)
        solo = P.run_policy(gpu, [hp], P.SchedulerConfig(), P.ms_to_ns(12), profiler=prof,
                            device_factory=gm.GpuSim)
        co = P.run_policy(gpu, [hp, be], P.SchedulerConfig(), P.ms_to_ns(12), profiler=prof,
                          device_factory=gm.GpuSim, placement_seed=rank)
        s = max(c - a for a, c in solo.requests["hp"])
        c = max(c - a for a, c in co.requests["hp"])
        local = {"overhead": 100.0 * (c / s - 1), "rank": rank, "be_iters": len(co.iterations["be"])}
        gathered, worst = bench.gather_pairs(local, dist)
        if rank == 0:
            q.put((gathered, worst))
    finally:
        dist.destroy_process_group()


def test_two_rank_pairs_aggregate_worst():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, worst = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [g["rank"] for g in gathered] == [0, 1]
    assert worst["overhead"] == max(g["overhead"] for g in gathered)
    assert all(g["be_iters"] > 0 for g in gathered)
