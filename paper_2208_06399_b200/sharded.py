"""Table-wise sharded execution of the embedding-bag path over one process per
GPU.

Rank k holds the tables with ``plan.assignment[i] == k`` (positional against
``task.tables``, tables.hpp:93-116) and computes their pooled rows for the
whole global batch B: a [B, SD_k] fp32 block, SD_k = sum of its tables' dims.
Samples are data-parallel: rank p owns samples [p*B/G, (p+1)*B/G). The
forward exchange sends rows [p*B/G, (p+1)*B/G) of every table owner's block to
rank p (one ``all_to_all_single``; the rows are contiguous, so no packing);
rank p receives G blocks [B/G, SD_k] in rank order. The backward exchange is
the exact inverse for the gradient of those rows.

The collectives go through ``torch.distributed`` (NCCL over NVLink on the
GPU box, gloo in the CPU tests). ``FusedPooledExchange`` removes the forward
collective: the forward kernel itself stores each pooled row into its sample
owner's receive buffer (torch symmetric memory, peer stores over NVLink).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence

from .tables import ShardingPlan, ShardingTask, TableDesc


@dataclass
class A2ALayout:
    world: int
    batch: int
    shard_dims: List[int]  # SD_k per rank
    shard_tables: List[List[int]]  # positions into task.tables per rank, placement order
    columns: List[List[int]]  # per rank: first pooled column of each member table

    @property
    def rows_per_rank(self) -> int:
        return self.batch // self.world

    def send_splits(self, rank: int) -> List[int]:
        """Element counts rank sends to each peer in the forward exchange."""
        return [self.rows_per_rank * self.shard_dims[rank]] * self.world

    def recv_splits(self) -> List[int]:
        """Element counts received from each table owner in the forward exchange."""
        return [self.rows_per_rank * d for d in self.shard_dims]

    def recv_offset(self, owner: int) -> int:
        return self.rows_per_rank * sum(self.shard_dims[:owner])

    def locate(self, table_pos: int):
        """(owner rank, first column inside the owner's block) of task.tables[table_pos]."""
        for k, members in enumerate(self.shard_tables):
            if table_pos in members:
                return k, self.columns[k][members.index(table_pos)]
        raise KeyError(table_pos)


def a2a_layout(task: ShardingTask, plan: ShardingPlan, batch: int) -> A2ALayout:
    plan.validate(task)
    world = task.num_shards
    if batch % world:
        raise ValueError(f"batch {batch} must divide by the shard count {world}")
    members = plan.shard_member_indices(task)
    dims = [sum(task.tables[i].dim for i in m) for m in members]
    cols = []
    for m in members:
        c, acc = [], 0
        for i in m:
            c.append(acc)
            acc += task.tables[i].dim
        cols.append(c)
    return A2ALayout(world, batch, dims, members, cols)


def local_tables(task: ShardingTask, plan: ShardingPlan, rank: int) -> List[TableDesc]:
    return [task.tables[i] for i in plan.shard_member_indices(task)[rank]]


class PooledExchange:
    """Forward / backward all-to-all of pooled rows for one rank."""

    def __init__(self, layout: A2ALayout, rank: int, group=None, device=None):
        import torch

        self.L, self.rank, self.group = layout, rank, group
        self.send = layout.send_splits(rank)
        self.recv = layout.recv_splits()
        self.recv_buf = torch.empty(sum(self.recv), dtype=torch.float32, device=device)
        self.grad_buf = torch.empty(layout.batch * layout.shard_dims[rank], dtype=torch.float32, device=device)

    def forward(self, pooled):
        """pooled: this rank's [B, SD_rank] block -> flat receive buffer (G blocks [B/G, SD_k])."""
        import torch.distributed as dist

        dist.all_to_all_single(self.recv_buf, pooled.reshape(-1), self.recv, self.send, group=self.group)
        return self.recv_buf

    def backward(self, grad_recv):
        """grad_recv: gradient w.r.t. the receive buffer -> [B, SD_rank] for this rank's tables."""
        import torch.distributed as dist

        dist.all_to_all_single(self.grad_buf, grad_recv.reshape(-1), self.send, self.recv, group=self.group)
        return self.grad_buf.view(self.L.batch, self.L.shard_dims[self.rank])

    def block(self, recv_flat, owner: int):
        """View of the [B/G, SD_owner] block received from `owner`."""
        o = self.L.recv_offset(owner)
        n = self.L.rows_per_rank * self.L.shard_dims[owner]
        return recv_flat[o:o + n].view(self.L.rows_per_rank, self.L.shard_dims[owner])

    def table_rows(self, recv_flat, table_pos: int):
        """[B/G, dim] pooled rows of task.tables[table_pos] for this rank's samples."""
        owner, col = self.L.locate(table_pos)
        return self.block(recv_flat, owner)[:, col:col + self._dim_of(table_pos)]

    def _dim_of(self, table_pos):
        owner, _ = self.L.locate(table_pos)
        members = self.L.shard_tables[owner]
        k = members.index(table_pos)
        cols = self.L.columns[owner] + [self.L.shard_dims[owner]]
        return cols[k + 1] - cols[k]


def peer_bases(layout: A2ALayout, owner: int, recv_base_ptrs: Sequence[int]) -> List[int]:
    """Device addresses the owner's forward writes to (as_set_peer_outputs):
    for every sample owner q, q's receive buffer + this owner's block offset."""
    return [int(p) + 4 * layout.recv_offset(owner) for p in recv_base_ptrs]


class FusedPooledExchange:
    """Forward exchange fused into the forward kernel: the
    receive buffers live in torch symmetric memory (one allocation per rank,
    mapped into every peer over NVLink), the shard's K1/K4 epilogues store each
    pooled row straight into its sample owner's receive block
    (EmbeddingShard.set_peer_outputs), and a device-side barrier orders the
    readers. No pooled-row copy, no NCCL call in the forward. The backward
    exchange of the gradients stays the NCCL all-to-all (PooledExchange).

    Raises when symmetric memory is unavailable; callers fall back to
    PooledExchange."""

    def __init__(self, layout: A2ALayout, rank: int, shard, group=None, device=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        self.L, self.rank, self.group = layout, rank, group
        group = group or dist.group.WORLD
        n = layout.rows_per_rank * sum(layout.shard_dims)
        self.recv_buf = symm_mem.empty(n, dtype=torch.float32, device=device)
        self.hdl = symm_mem.rendezvous(self.recv_buf, group)
        self.shard = shard
        shard.set_peer_outputs(peer_bases(layout, rank, self.hdl.buffer_ptrs), layout.rows_per_rank)
        self._nccl = PooledExchange(layout, rank, group=self.group, device=device)

    def forward(self, stream=None):
        """This rank's forward with the exchange fused in; returns the receive buffer."""
        self.shard.forward(stream=stream)
        self.hdl.barrier(channel=0)  # every owner's stores into every receive buffer are done
        return self.recv_buf

    def backward(self, grad_recv):
        return self._nccl.backward(grad_recv)

    def close(self):
        self.shard.set_peer_outputs([], 0)
