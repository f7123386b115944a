"""Probe: can two processes on this box share a device buffer through CUDA IPC
(torch.multiprocessing.reductions) and write into each other's memory?"""
import os
import sys

import torch
import torch.distributed as dist
import torch.multiprocessing as mp
from torch.multiprocessing.reductions import reduce_tensor


def worker(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    buf = torch.zeros(1 << 20, dtype=torch.float64, device="cuda")
    fn, args = reduce_tensor(buf)
    handles = [None] * world
    dist.all_gather_object(handles, (fn, args))
    peers = [buf if q == rank else handles[q][0](*handles[q][1]) for q in range(world)]
    # every rank writes its rank + 1 into slice [rank] of every peer's buffer
    for q in range(world):
        peers[q][rank * 1000:(rank + 1) * 1000] = float(rank + 1)
    torch.cuda.synchronize()
    dist.barrier()
    got = [float(buf[q * 1000]) for q in range(world)]
    print(f"rank {rank}: peer ptrs {[hex(p.data_ptr()) for p in peers]} got {got}", flush=True)
    assert got == [float(q + 1) for q in range(world)]
    dist.barrier()
    del peers
    dist.destroy_process_group()


if __name__ == "__main__":
    mp.spawn(worker, args=(2, 29611), nprocs=2, join=True)
    print("ipc ok")
