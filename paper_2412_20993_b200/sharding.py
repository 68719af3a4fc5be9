"""Request sharding across the GPUs of one box.

One process per GPU; requests / programs are independent units, so every rank scores a
contiguous slice [rank*N/G, (rank+1)*N/G) with no data-path exchange.  Exactly two
exchange steps exist, both allgathers through torch.distributed (NCCL over NVLink /
NVSwitch on the B200 box; gloo in the CPU tests of this host logic):

  * K5 global token offsets: each rank's exclusive budget scan is local; an allgather of
    one i64 budget total per rank (8 B x world) gives every rank its base, added on the
    device (cdx_offsets_rebase).  Kept lists are already global (kept_base = r0) and
    concatenate in rank order to the single-GPU stable compaction.
  * K6 global gang order: each rank radix-sorts its programs' composite keys, the sorted
    runs are allgathered into a padded receive buffer (stride = the largest shard, known
    on the host without a sync), and every rank merges them on the device
    (cdx_gang_merge).  The total order is unique, so the result equals the 1-GPU sort.

`ops` is the compute provider: a `Context` (the B200 kernels) in the product; the CPU
tests substitute a checker-backed stand-in so that the exchange logic runs under gloo.
"""
from __future__ import annotations

from typing import Optional


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

    # ---- K2 + K5 with global token offsets ------------------------------------------
    def sc_decide(self, ids, thresholds, policy, r0: int, out: Optional[dict] = None, hcert=None, meets=None):
        """ids u32[R_local][P][S] of requests [r0, r0+R_local).  Returns the allocate_scan
        outputs with offsets made global and `shard_totals` (i64[world])."""
        R, P, _ = ids.shape
        hcert, meets = self.ops.sc_certaindex(ids, thresholds, hcert=hcert, meets=meets)
        res = self.ops.allocate_scan(meets, R, P, policy, kept_base=r0, out=out)
        totals = self.allgather(res["scalars"][2:3])
        self.ops.offsets_rebase(res["offsets"], totals, self.rank)
        res["shard_totals"] = totals
        res["hcert"], res["meets"] = hcert, meets
        return res

    # ---- K6 global order ----------------------------------------------------------------
    def gang_order(self, soa: dict, policy, now: float, id_base: int, stride: int):
        """soa: this rank's programs (ids id_base + i).  stride >= every rank's program
        count.  Returns (order_padded u32[world*stride], total i64[1]) on every rank; the
        first `total` entries are the global order."""
        import torch
        _, _, keys = self.ops.gang_priority(soa, policy, now, id_base=id_base, want_keys=True)
        n = keys.shape[0]
        if n > stride:
            raise ValueError("gang_order: stride smaller than this rank's program count")
        send = torch.full((stride, 3), -1, dtype=torch.int64, device=keys.device)
        send[:n] = keys
        lens = self.allgather(torch.tensor([n], dtype=torch.int64, device=keys.device))
        recv = self.allgather(send)
        total = torch.zeros((1,), dtype=torch.int64, device=keys.device)
        order = self.ops.gang_merge(recv, lens, stride, total=total)
        return order, total
