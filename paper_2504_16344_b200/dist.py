"""Parameter-dimension (Nm) sharding across ranks, one process per GPU.

Column c of F-hat only meets x-hat_c (F) or produces x-hat_c (F*), so a
contiguous column range per rank gives one exchange step per matvec:

* F m:  each rank applies its shard, d = sum over ranks  (all-reduce of the
        Nd x Nt output -- after the local c2r, the inverse FFT being linear);
* F* d: d must be on every rank (broadcast from ``src``), m stays sharded.

torch.distributed is the plumbing (NCCL on the GPU box, gloo in the CPU
tests).  The local compute is a ``MatvecPlan`` shard built on the device
from the global generated kernel; tests may inject another local operator.
"""
import torch
import torch.distributed as dist


def shard_range(nm_total, world, rank):
    """Contiguous column range [c0, c1) of `rank`; the first
    nm_total % world ranks get one extra column."""
    base, extra = divmod(nm_total, world)
    c0 = rank * base + min(rank, extra)
    return c0, c0 + base + (1 if rank < extra else 0)


class ShardedMatvec:
    """F / F* over an Nm-sharded block-Toeplitz kernel.

    ``local`` is any object with ``apply_raw(in, out, scratch)``,
    ``apply_adjoint_raw(in, out, scratch)``, ``rows_out()``, ``n_cols()``,
    ``n_time()``; by default a ``MatvecPlan.generated`` shard."""

    def __init__(self, rows, nm_total, nt, seed, tag=0, group=None, local=None, scratch=None,
                 src=0):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.c0, self.c1 = shard_range(nm_total, self.world, self.rank)
        self.rows, self.nm_total, self.nt, self.src = rows, nm_total, nt, src
        if local is None:
            from .matvec import MatvecPlan
            local = MatvecPlan.generated(rows, self.c1 - self.c0, nt, seed=seed, tag=tag,
                                         nm_total=nm_total, c0=self.c0)
            scratch = MatvecPlan.Scratch(local, stream=torch.cuda.current_stream())
        self.local = local
        self.scratch = scratch

    @property
    def n_local(self):
        return self.c1 - self.c0

    def apply(self, m_local, d_out):
        """d_out <- F m  (m_local: this rank's n_local * nt values)."""
        self.local.apply_raw(m_local, d_out, self.scratch)
        if self.world > 1:
            dist.all_reduce(d_out, group=self.group)
        return d_out

    def apply_adjoint(self, d, m_local_out, broadcast=True):
        """m_local_out <- (F* d) restricted to this rank's columns; d is
        broadcast from ``src`` first unless the caller already holds it."""
        if self.world > 1 and broadcast:
            dist.broadcast(d, self.src, group=self.group)
        self.local.apply_adjoint_raw(d, m_local_out, self.scratch)
        return m_local_out
