"""Run a function on `world` local processes joined by a torch.distributed
process group (gloo, 127.0.0.1), collecting each rank's return value."""
from __future__ import annotations

import multiprocessing as mp
import os
import socket
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _entry(rank, world, port, modname, fname, args, q):
    try:
        if ROOT not in sys.path:
            sys.path.insert(0, ROOT)
        import importlib

        import torch.distributed as dist
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        try:
            fn = getattr(importlib.import_module(modname), fname)
            q.put((rank, "ok", fn(rank, world, *args)))
        finally:
            dist.destroy_process_group()
    except BaseException:
        q.put((rank, "err", traceback.format_exc()))


def run_world(world: int, modname: str, fname: str, *args, timeout: float = 600.0) -> list:
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_entry, args=(r, world, port, modname, fname, args, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    try:
        for _ in range(world):
            rank, status, val = q.get(timeout=timeout)
            if status != "ok":
                raise RuntimeError(f"rank {rank} failed:\n{val}")
            out[rank] = val
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    return [out[r] for r in range(world)]
