"""Table-wise sharded execution of the embedding-bag path over one process per
GPU.

Rank k holds the tables with ``plan.assignment[i] == k`` (positional against
``task.tables``, tables.hpp:93-116) and computes their pooled rows for the
whole global batch B: a [B, SD_k] fp32 block, SD_k = sum of its tables' dims.
Samples are data-parallel: rank p owns samples [row_start[p], row_start[p+1])
(B/G each, the first B % G ranks one more). The forward exchange delivers rows
[row_start[p], row_start[p+1]) of every table owner's block to rank p, whose
receive buffer holds G blocks [rows_p, SD_k] in rank order; the backward
exchange is the exact inverse for the gradient of those rows.

``ShardComm`` is the product path: the C-ABI's ``as_comm`` (csrc/cuda/sharded.cu).
Its forward exchange is fused into the forward kernel (pooled rows stored into
the owners' receive buffers over peer memory, then a system-scope device
barrier), its backward pushes each gradient block into its table owner's buffer
(or either direction over NCCL send/recv). ``PooledExchange`` is the plain
``torch.distributed.all_to_all_single`` formulation of the same exchange: the
library baseline and the gloo CPU tests' path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence

from .tables import ShardingPlan, ShardingTask, TableDesc

UNIQUE_ID_BYTES = 128  # AS_UNIQUE_ID_BYTES
HANDLE_BYTES = 512  # AS_HANDLE_BYTES
XCHG_PEER, XCHG_FWD_NCCL, XCHG_BWD_NCCL, XCHG_NCCL = 0, 1, 2, 3


def row_starts(batch: int, world: int) -> List[int]:
    """Sample ranges of the ranks: B // G rows each, the first B % G ranks one more."""
    base, extra = divmod(batch, world)
    out = [0]
    for p in range(world):
        out.append(out[-1] + base + (1 if p < extra else 0))
    return out


@dataclass
class A2ALayout:
    world: int
    batch: int
    shard_dims: List[int]  # SD_k per rank
    shard_tables: List[List[int]]  # positions into task.tables per rank, placement order
    columns: List[List[int]]  # per rank: first pooled column of each member table
    row_start: List[int]  # sample ranges, world + 1 entries

    def rows(self, p: int) -> int:
        return self.row_start[p + 1] - self.row_start[p]

    def send_splits(self, rank: int) -> List[int]:
        """Element counts rank sends to each peer in the forward exchange."""
        return [self.rows(q) * self.shard_dims[rank] for q in range(self.world)]

    def recv_splits(self, rank: int) -> List[int]:
        """Element counts rank receives from each table owner in the forward exchange."""
        return [self.rows(rank) * d for d in self.shard_dims]

    def recv_offset(self, owner: int, rank: int) -> int:
        """Element offset of owner's block in rank's receive buffer."""
        return self.rows(rank) * sum(self.shard_dims[:owner])

    def locate(self, table_pos: int):
        """(owner rank, first column inside the owner's block) of task.tables[table_pos]."""
        for k, members in enumerate(self.shard_tables):
            if table_pos in members:
                return k, self.columns[k][members.index(table_pos)]
        raise KeyError(table_pos)

    def dim_of(self, table_pos: int) -> int:
        owner, _ = self.locate(table_pos)
        members = self.shard_tables[owner]
        k = members.index(table_pos)
        cols = self.columns[owner] + [self.shard_dims[owner]]
        return cols[k + 1] - cols[k]


def a2a_layout(task: ShardingTask, plan: ShardingPlan, batch: int) -> A2ALayout:
    plan.validate(task)
    world = task.num_shards
    if batch < world:
        raise ValueError(f"batch {batch} is smaller than the shard count {world}")
    members = plan.shard_member_indices(task)
    dims = [sum(task.tables[i].dim for i in m) for m in members]
    cols = []
    for m in members:
        c, acc = [], 0
        for i in m:
            c.append(acc)
            acc += task.tables[i].dim
        cols.append(c)
    return A2ALayout(world, batch, dims, members, cols, row_starts(batch, world))


def local_batch(streams, row_start: Sequence[int], rank: int):
    """Rows [row_start[rank], row_start[rank+1]) of each (offsets, indices) CSR:
    the mini-batch a rank's data loader holds before the KJT exchange."""
    import numpy as np

    a, b = int(row_start[rank]), int(row_start[rank + 1])
    out = []
    for off, idx in streams:
        off = np.asarray(off, dtype=np.int64)
        lo, hi = int(off[a]), int(off[b])
        out.append((off[a:b + 1] - lo, np.asarray(idx, dtype=np.int64)[lo:hi]))
    return out


def local_tables(task: ShardingTask, plan: ShardingPlan, rank: int) -> List[TableDesc]:
    return [task.tables[i] for i in plan.shard_member_indices(task)[rank]]


def recv_table_rows(layout: A2ALayout, recv_flat, rank: int, table_pos: int):
    """[rows_rank, dim] pooled rows of task.tables[table_pos] in rank's receive buffer."""
    owner, col = layout.locate(table_pos)
    o = layout.recv_offset(owner, rank)
    n = layout.rows(rank) * layout.shard_dims[owner]
    block = recv_flat[o:o + n].reshape(layout.rows(rank), layout.shard_dims[owner])
    return block[:, col:col + layout.dim_of(table_pos)]


class PooledExchange:
    """Forward / backward all-to-all of pooled rows for one rank with
    torch.distributed.all_to_all_single (the library formulation)."""

    def __init__(self, layout: A2ALayout, rank: int, group=None, device=None):
        import torch

        self.L, self.rank, self.group = layout, rank, group
        self.send = layout.send_splits(rank)
        self.recv = layout.recv_splits(rank)
        self.recv_buf = torch.empty(sum(self.recv), dtype=torch.float32, device=device)
        self.grad_buf = torch.empty(layout.batch * layout.shard_dims[rank], dtype=torch.float32, device=device)

    def forward(self, pooled):
        """pooled: this rank's [B, SD_rank] block -> flat receive buffer (G blocks [rows_rank, SD_k])."""
        import torch.distributed as dist

        dist.all_to_all_single(self.recv_buf, pooled.reshape(-1), self.recv, self.send, group=self.group)
        return self.recv_buf

    def backward(self, grad_recv):
        """grad_recv: gradient w.r.t. the receive buffer -> [B, SD_rank] for this rank's tables."""
        import torch.distributed as dist

        dist.all_to_all_single(self.grad_buf, grad_recv.reshape(-1), self.send, self.recv, group=self.group)
        return self.grad_buf.view(self.L.batch, self.L.shard_dims[self.rank])

    def table_rows(self, recv_flat, table_pos: int):
        return recv_table_rows(self.L, recv_flat, self.rank, table_pos)


def peer_bases(layout: A2ALayout, owner: int, recv_base_ptrs: Sequence[int]) -> List[int]:
    """Device addresses owner's forward writes to (as_set_peer_outputs_v):
    for every sample owner q, q's receive buffer + owner's block offset."""
    return [int(p) + 4 * layout.recv_offset(owner, q) for q, p in enumerate(recv_base_ptrs)]


# ---------------------------------------------------------------------------
# the product path: as_comm (C-ABI)
# ---------------------------------------------------------------------------
def unique_id() -> bytes:
    """ncclGetUniqueId through the C-ABI (rank 0 creates, every rank receives)."""
    from ._capi import lib
    from .errors import check

    buf = C.create_string_buffer(UNIQUE_ID_BYTES)
    check(lib().as_comm_unique_id(buf))
    return buf.raw


class ShardComm:
    """One rank of the sharded step (as_comm): exchange + this rank's shard."""

    def __init__(self, shard, rank: int, world: int, nccl_id: Optional[bytes] = None):
        from ._capi import lib
        from .errors import check

        self.shard, self.rank, self.world = shard, rank, world
        h = C.c_void_p()
        uid = C.create_string_buffer(nccl_id, UNIQUE_ID_BYTES) if nccl_id is not None else None
        check(lib().as_comm_init(shard._h, uid, rank, world, C.byref(h)))
        self._h = h
        import weakref

        shard._comms = getattr(shard, "_comms", []) + [weakref.ref(self)]
        self._lib, self._check = lib, check

    def setup(self, layout: A2ALayout, mode: int = XCHG_PEER) -> None:
        d = (C.c_int64 * self.world)(*layout.shard_dims)
        s = (C.c_int64 * (self.world + 1))(*layout.row_start)
        self._check(self._lib().as_alltoall_setup(self._h, d, s, int(mode)))
        self.layout = layout

    def handle(self) -> bytes:
        buf = C.create_string_buffer(HANDLE_BYTES)
        n = C.c_int64()
        self._check(self._lib().as_alltoall_handle(self._h, buf, C.byref(n)))
        return buf.raw

    def open(self, blobs: Sequence[bytes]) -> None:
        allb = b"".join(bytes(b).ljust(HANDLE_BYTES, b"\0")[:HANDLE_BYTES] for b in blobs)
        self._check(self._lib().as_alltoall_open(self._h, C.create_string_buffer(allb, len(allb))))

    def use_host_barrier(self, group=None) -> None:
        """Ranks sharing ONE device (as_alltoall_host_barrier): the exchange
        barrier becomes stream sync + torch.distributed.barrier(group) on the
        host, so no kernel ever waits on another rank's kernel."""
        import torch.distributed as dist

        def _bar(_user):
            try:
                dist.barrier(group=group)
                return 0
            except Exception:
                return 1

        self._host_cb = C.CFUNCTYPE(C.c_int32, C.c_void_p)(_bar)  # kept alive with the comm
        self._check(self._lib().as_alltoall_host_barrier(self._h, C.cast(self._host_cb, C.c_void_p), None))

    def load_exchanged(self, all_tables: Sequence[TableDesc], owner: Sequence[int], local_streams, stream=None) -> None:
        """KJT all-to-all (as_load_streams_exchanged): local_streams
        = this rank's mini-batch, (offsets over its own rows, indices) for EVERY
        table of the task in task order; owner[t] = rank holding table t. After
        the call this rank's shard holds its tables' streams of the whole batch."""
        import numpy as np

        from .device import _stream
        from .tables import specs_to_c

        st = [(np.ascontiguousarray(o, dtype=np.int64), np.ascontiguousarray(i, dtype=np.int64))
              for o, i in local_streams]
        n = len(all_tables)
        if len(st) != n or len(owner) != n:
            raise ValueError(f"expected {n} local streams and owners, got {len(st)} / {len(owner)}")
        po = (C.c_void_p * max(1, n))(*[o.ctypes.data for o, _ in st])
        pi = (C.c_void_p * max(1, n))(*[i.ctypes.data for _, i in st])
        ow = (C.c_int32 * max(1, n))(*[int(q) for q in owner])
        self._check(self._lib().as_load_streams_exchanged(self._h, n, specs_to_c(list(all_tables)), ow, po, pi,
                                                          _stream(stream)))

    def forward(self, stream=None) -> None:
        from .device import _stream

        self._check(self._lib().as_forward_sharded(self._h, _stream(stream)))

    def backward(self, grad_recv=None, lr: float = 0.01, eps: float = 1e-8, stream=None) -> None:
        from .device import _ptr, _stream

        self._check(self._lib().as_backward_sharded(self._h, _ptr(grad_recv), lr, eps, _stream(stream)))

    def step(self, lr: float = 0.01, eps: float = 1e-8, want_loss: bool = False, stream=None) -> Optional[float]:
        from .device import _stream

        loss = C.c_double()
        self._check(self._lib().as_step_sharded(self._h, lr, eps, C.byref(loss) if want_loss else None,
                                                _stream(stream)))
        return loss.value if want_loss else None

    def info(self):
        from ._capi import CommInfoC

        i = CommInfoC()
        self._check(self._lib().as_comm_info_get(self._h, C.byref(i)))
        return i

    def profile_read(self, reset: bool = True):
        """-> (forward exchange ms, backward exchange ms) accumulated while the shard profiles."""
        ms = (C.c_double * 2)()
        self._check(self._lib().as_comm_profile_read(self._h, ms, int(reset)))
        return ms[0], ms[1]

    def recv_tensor(self):
        """torch view of this rank's receive buffer (flat fp32)."""
        import torch

        i = self.info()
        n = int(i.recv_rows * i.recv_cols)

        class _CAI:
            __cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (int(i.recv), False),
                                        "version": 3, "strides": None}

        return torch.as_tensor(_CAI(), device=f"cuda:{self.shard.device}")

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            self._check(self._lib().as_comm_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def connect(shard, layout: A2ALayout, rank: int, world: int, mode: int = XCHG_PEER, group=None,
            use_nccl: bool = True, host_barrier: bool = False) -> ShardComm:
    """Build this rank's ShardComm with torch.distributed as the control plane:
    the NCCL unique id (if use_nccl) is broadcast from rank 0; without NCCL
    the peer-memory handle blobs are all-gathered here instead of over NCCL.
    host_barrier: the ranks share one device — exchange barriers on the host
    (ShardComm.use_host_barrier), never a device-side wait."""
    import torch.distributed as dist

    uid = None
    if use_nccl:
        obj = [unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = obj[0]
    comm = ShardComm(shard, rank, world, uid)
    comm.setup(layout, mode)
    if uid is None:
        blobs = [None] * world
        dist.all_gather_object(blobs, comm.handle(), group=group)
        comm.open(blobs)
    if host_barrier:
        comm.use_host_barrier(group)
    return comm
