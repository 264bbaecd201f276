"""Debug: 2 ranks sharing cuda:0 over the peer exchange (gloo for the handles)."""
import os
import sys
import time

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def worker(rank, world, port, shapes, steps):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import ssgen
    import paper_2605_12464_b200 as ss
    from paper_2605_12464_b200.dist import CudaOps, RowShardQuantizer, ShardPlan
    plan = ShardPlan(shapes, rank, world)
    shards = [ssgen.generate("gaussian", r, c, seed=1, tid=k).cuda()[slice(*plan.rows(k))].contiguous()
              for k, (r, c) in enumerate(shapes)]
    ops = CudaOps(-8, 8)
    outs = [ops.alloc_out(x) for x in shards]
    qz = RowShardQuantizer(plan, ops, device="cuda", exchange="peer")
    print("rank", rank, "groups", qz.groups, flush=True)
    for i in range(steps):
        t = time.time()
        qz.step(shards, outs)
        torch.cuda.synchronize()
        print("rank %d step %d %.3f s status %d G %s" % (rank, i, time.time() - t, ss.device_status(),
                                                         [float(o.G.item()) for o in outs[:3]]), flush=True)
    qz.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    shapes = [tuple(map(int, s.split("x"))) for s in sys.argv[1].split(",")]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=worker, args=(r, 2, 29611, shapes, steps)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=300)
