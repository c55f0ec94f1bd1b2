import os, sys, torch, torch.distributed as dist, torch.multiprocessing as mp
def run(rank, world):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    x = torch.full((4,), float(rank + 1), dtype=torch.float64, device=dev)
    res = {}
    for name, fn in [("all_reduce", lambda: dist.all_reduce(x.clone())),
                     ("all_gather_into_tensor", lambda: dist.all_gather_into_tensor(torch.empty(4 * world, dtype=torch.float64, device=dev), x)),
                     ("all_gather", lambda: dist.all_gather([torch.empty_like(x) for _ in range(world)], x)),
                     ("all_gather_async", lambda: dist.all_gather([torch.empty_like(x) for _ in range(world)], x, async_op=True).wait()),
                     ("all_to_all_single", lambda: dist.all_to_all_single(torch.empty_like(x), x))]:
        try:
            fn(); res[name] = "ok"
        except Exception as e:
            res[name] = type(e).__name__ + ": " + str(e)[:80]
    if rank == 0: print(res, flush=True)
    dist.destroy_process_group()
if __name__ == "__main__":
    mp.spawn(run, args=(2,), nprocs=2)
