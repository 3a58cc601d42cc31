"""Probe: can ranks map each other's CUDA buffers (CUDA IPC through
torch.multiprocessing's tensor reduction, and torch symmetric memory)?
Launch: torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/probes/peer_ipc.py [--same-device]"""
import os, sys
import torch, torch.distributed as dist
from torch.multiprocessing.reductions import reduce_tensor

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
same = "--same-device" in sys.argv
dev = torch.device("cuda", 0 if same else int(os.environ.get("LOCAL_RANK", 0)))
torch.cuda.set_device(dev)
dist.init_process_group("gloo")
x = torch.full((1 << 20,), float(rank + 1), device=dev)
fn, args = reduce_tensor(x)
objs = [None] * world
dist.all_gather_object(objs, (fn, args))
peers = []
for r, (f, a) in enumerate(objs):
    peers.append(x if r == rank else f(*a))
torch.cuda.synchronize()
vals = [float(p[0]) for p in peers]
print(f"rank {rank}: ipc peer values {vals}", flush=True)
dist.barrier()
try:
    import torch.distributed._symmetric_memory as sm
    sm.enable_symm_mem_for_group(dist.group.WORLD.group_name)
    t = sm.empty(1024, dtype=torch.float32, device=dev)
    t.fill_(rank + 10)
    h = sm.rendezvous(t, dist.group.WORLD)
    dist.barrier(); torch.cuda.synchronize()
    got = [float(h.get_buffer(r, (1024,), torch.float32)[0]) for r in range(world)]
    print(f"rank {rank}: symm_mem values {got}", flush=True)
except Exception as e:
    print(f"rank {rank}: symm_mem failed: {type(e).__name__}: {str(e)[:300]}", flush=True)
dist.barrier()
dist.destroy_process_group()
