import os, sys, torch, torch.distributed as dist, torch.multiprocessing as mp
def run(rank):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533")
    dist.init_process_group("gloo", rank=rank, world_size=2)
    d = torch.device("cuda", 0)
    out = {}
    for name, fn in [("barrier", lambda: dist.barrier()),
                     ("all_reduce_max", lambda: dist.all_reduce(torch.tensor([float(rank)], device=d), op=dist.ReduceOp.MAX)),
                     ("all_reduce_sum_i64", lambda: dist.all_reduce(torch.ones(3, dtype=torch.int64, device=d))),
                     ("all_gather_into_tensor", lambda: dist.all_gather_into_tensor(torch.empty(4, 3, dtype=torch.float64, device=d), torch.full((2, 3), float(rank), dtype=torch.float64, device=d)))]:
        try:
            fn(); out[name] = "ok"
        except Exception as e:
            out[name] = repr(e)[:150]
    if rank == 0: print(out, flush=True)
    dist.destroy_process_group()
if __name__ == "__main__":
    mp.spawn(run, nprocs=2)
