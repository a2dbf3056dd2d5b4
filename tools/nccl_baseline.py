"""NCCL baseline for the halo exchange: the same messages the plan sends
(acoustic SO-8, 1024^3 per GPU, diagonal message set) exchanged with
torch.distributed NCCL isend/irecv of packed boxes, timed on the device.
Compares with the product's device-flag + peer-copy exchange (diagonal mode
post time) and the fused full mode (exposed time) from the same bench.

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/nccl_baseline.py
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_13094_b200.decomposition import Decomposition  # noqa: E402
from paper_2312_13094_b200.distfield import diagonal_messages  # noqa: E402

TOPOS = {2: (2, 1, 1), 4: (2, 2, 1), 8: (4, 2, 1)}


def main():
    dist.init_process_group("nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    n, h, r = 1024, 8, 4
    topo = TOPOS[world]
    d = Decomposition.create(tuple(n * p for p in topo), world, topo)
    loc = d.local_shape(rank)
    u = torch.zeros(tuple(x + 2 * h for x in loc), device="cuda")
    msgs = diagonal_messages(d, rank, (r, r, r))
    sl = lambda box: tuple(slice(lo + h, hi + h) for lo, hi in zip(*box))
    sends = [(m.peer, sl(m.send)) for m in msgs]
    recvs = [(m.peer, sl(m.recv)) for m in msgs]
    rbufs = [torch.empty(tuple(s.stop - s.start for s in box), device="cuda") for _, box in recvs]
    nbytes = sum(b.numel() * 4 for b in rbufs)

    def exchange():
        packed = [u[box].contiguous() for _, box in sends]      # pack
        ops = [dist.P2POp(dist.irecv, buf, peer) for (peer, _), buf in zip(recvs, rbufs)]
        ops += [dist.P2POp(dist.isend, buf, peer) for (peer, _), buf in zip(sends, packed)]
        for q in dist.batch_isend_irecv(ops):                  # one NCCL group
            q.wait()
        for (_, box), buf in zip(recvs, rbufs):                # unpack
            u[box].copy_(buf)

    for _ in range(5):
        exchange()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 20
    e0.record()
    for _ in range(steps):
        exchange()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"transport": "NCCL isend/irecv + pack/unpack (torch.distributed)",
                          "topology": topo, "messages_rank0": len(msgs),
                          "bytes_rank0": nbytes, "ms_per_exchange": float(t.item()),
                          "gbs_rank0": nbytes / (float(t.item()) * 1e-3) / 1e9}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
