"""Request sharding across the GPUs of one box.

One process per GPU; requests / programs are independent units, so every rank scores a
contiguous slice [rank*N/G, (rank+1)*N/G) with no data-path exchange.  Exactly two
exchange steps exist:

  * K5 global token offsets: each rank's exclusive budget scan is local; an allgather of
    {requests, budget total, kept, tokens saved} per rank gives every rank its base, added on
    the device.  Kept lists concatenate in rank order to the single-GPU stable compaction.
  * K6 global gang order: a distributed sample sort.  Each rank radix-sorts its programs'
    composite keys, allgathers regular samples of its run, derives the same splitters
    (cdx_shard_splitters), sends each key to the rank owning its bucket (alltoallv), merges
    the runs it received on the device and the buckets' program ids are allgathered in bucket
    order.  The total order is unique, so the result equals the 1-GPU sort.

Two drivers run that protocol:

  * the context's own communicator (`Context.for_process_group` / `with_nccl`: NCCL owned by
    libcdx, the C-ABI entry points cdx_allocate_scan_sharded / cdx_gang_priority_sharded,
    the path a C++ caller uses too) — taken whenever the context spans the group;
  * torch.distributed collectives over the same device building blocks (cdx_shard_samples,
    cdx_shard_bounds, cdx_gang_merge_runs, cdx_offsets_rebase) and the same host planning
    step — for a plain single-rank Context inside a torch process group, and for the CPU
    tests under gloo, where `ops` is a checker-backed stand-in (no GPU in that container).
"""
from __future__ import annotations

from typing import Optional

SHARD_SAMPLES = 256  # regular samples per rank (shard.cu SHARD_SAMPLES)


def shard_range(n: int, rank: int, world: int):
    """Contiguous shard of `n` units owned by `rank` (start, count)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_range: need 0 <= rank < world")
    start = n * rank // world
    return start, n * (rank + 1) // world - start


def max_shard(n: int, world: int) -> int:
    return max(shard_range(n, r, world)[1] for r in range(world))


class Sharded:
    """The multi-GPU decision path over one process group."""

    def __init__(self, ops, group=None, force_collectives: bool = False):
        import torch.distributed as dist
        self.ops = ops
        self.force = force_collectives  # run the collectives even at world size 1 (tests)
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.nccl = dist.is_initialized() and dist.get_backend(group) == "nccl"
        # the context owns a communicator spanning this group: run the C-ABI protocol
        self.native = getattr(ops, "world", 1) == self.world and getattr(ops, "_comm", None) is not None

    def allgather(self, t):
        """Concatenation of `t` from every rank in rank order (dim 0)."""
        import torch
        if self.world == 1 and not (self.force and self.dist.is_initialized()):
            return t
        if self.nccl:
            out = torch.empty((self.world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
            self.dist.all_gather_into_tensor(out, t.contiguous(), group=self.group)
            return out
        # gloo (the CPU tests, and the one-GPU multi-rank tests) gathers host tensors only
        src = t.contiguous().cpu() if t.is_cuda else t.contiguous()
        parts = [torch.empty_like(src) for _ in range(self.world)]
        self.dist.all_gather(parts, src, group=self.group)
        out = torch.cat(parts)
        return out.to(t.device) if t.is_cuda else out

    def alltoallv(self, t, send_counts, recv_counts):
        """Rows t[sum(send_counts[:q]) : ... + send_counts[q]] go to rank q; returns the rows
        received, rank order (dim 0)."""
        import torch
        recv_rows = int(sum(recv_counts))
        if self.world == 1 and not (self.force and self.dist.is_initialized()):
            return t[:recv_rows].clone()
        dev = t.device
        src = t.contiguous() if self.nccl else t.contiguous().cpu()
        out = torch.empty((recv_rows,) + tuple(t.shape[1:]), dtype=t.dtype, device=src.device)
        self.dist.all_to_all_single(out, src, [int(x) for x in recv_counts], [int(x) for x in send_counts],
                                    group=self.group)
        return out.to(dev)

    # ---- K2 + K5 with global token offsets ------------------------------------------
    def sc_decide(self, ids, thresholds, policy, r0: int, out: Optional[dict] = None, hcert=None, meets=None):
        """ids u32[R_local][P][S] of requests [r0, r0+R_local).  Returns the allocate_scan
        outputs with offsets made global and `shard_totals` (i64[world])."""
        R, P, _ = ids.shape
        hcert, meets = self.ops.sc_certaindex(ids, thresholds, hcert=hcert, meets=meets)
        if self.native:
            res = self.ops.allocate_scan_sharded(meets, R, P, policy, out=out)
            res["shard_totals"] = res["shard_info"][:, 1]
        else:
            res = self.ops.allocate_scan(meets, R, P, policy, kept_base=r0, out=out)
            totals = self.allgather(res["scalars"][2:3])
            self.ops.offsets_rebase(res["offsets"], totals, self.rank)
            res["shard_totals"] = totals
        res["hcert"], res["meets"] = hcert, meets
        return res

    # ---- K6 global order ----------------------------------------------------------------
    def gang_order(self, soa: dict, policy, now: float, id_base: int, capacity: Optional[int] = None):
        """soa: this rank's programs (ids id_base + i).  Returns the global order (u32 program
        ids as an int32 tensor) on every rank."""
        if self.native:
            return self.ops.gang_priority_sharded(soa, policy, now, id_base=id_base, capacity=capacity)
        import numpy as np
        import torch

        from . import shard_splitters
        W, me, s = self.world, self.rank, SHARD_SAMPLES
        _, _, keys = self.ops.gang_priority(soa, policy, now, id_base=id_base, want_keys=True)
        n = keys.shape[0]
        dev = keys.device
        # 1. regular samples of this run + its length, allgathered
        samp = self.ops.shard_samples(keys, s)
        rec = torch.cat([samp.reshape(-1), torch.tensor([n], dtype=torch.int64, device=dev)])
        g = self.allgather(rec).cpu().numpy().view(np.uint64).reshape(W, 3 * s + 1)
        # 2. the same splitters on every rank (host planning, libcdx)
        split = shard_splitters(g[:, : 3 * s], g[:, 3 * s], W, s)
        split_t = torch.from_numpy(np.ascontiguousarray(split).view(np.int64)).to(dev)
        # 3. bucket bounds of every run
        bounds = self.ops.shard_bounds(keys, split_t, W)
        gb = self.allgather(bounds).cpu().numpy().reshape(W, W + 1).astype(np.int64)
        send = np.diff(gb[me])
        recv = gb[:, me + 1] - gb[:, me]
        # 4. keys to the rank owning their bucket; merge the runs received
        rkeys = self.alltoallv(keys, send, recv)
        run_off = torch.from_numpy(np.concatenate([[0], np.cumsum(recv)]).astype(np.int64)).to(dev)
        bids = self.ops.gang_merge_runs(rkeys, run_off)
        # 5. every bucket's program ids, bucket order, to every rank
        bucket = (gb[:, 1:] - gb[:, :-1]).sum(axis=0)
        return self.alltoallv(bids.repeat(W), np.full(W, len(bids)), bucket)
