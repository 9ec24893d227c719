"""Probe: can two NCCL ranks share one GPU on this NCCL build? (one allreduce)"""
import os, sys
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def run(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    try:
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
        t = torch.ones(4, device="cuda") * (rank + 1)
        dist.all_reduce(t)
        torch.cuda.synchronize()
        print(f"rank {rank}: allreduce ok {t.tolist()}", flush=True)
        dist.destroy_process_group()
    except Exception as e:
        print(f"rank {rank}: FAILED {type(e).__name__}: {str(e)[:300]}", flush=True)


if __name__ == "__main__":
    mp.spawn(run, args=(2, 29517), nprocs=2, join=True)
