"""Spawn one process per GPU (or per simulated process on the CPU) for multi-process tests.

Each child initialises a gloo process group (the bootstrap all-gather libmpxa calls at
collective setup) on 127.0.0.1 and runs fn(rank, world, *args); failures come back to the
parent with their traceback."""
import os
import socket
import traceback


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _child(rank, world, port, fn, args, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["RANK"] = str(rank)
    os.environ["WORLD_SIZE"] = str(world)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        try:
            fn(rank, world, *args)
            q.put((rank, "ok"))
        finally:
            dist.destroy_process_group()
    except BaseException:  # pragma: no cover - reported to the parent
        q.put((rank, traceback.format_exc()))


def spawn(fn, world, *args, timeout=600):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_child, args=(r, world, port, fn, args, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = []
    try:
        for _ in procs:
            res.append(q.get(timeout=timeout))
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r, msg in sorted(res):
        assert msg == "ok", f"rank {r}: {msg}"
