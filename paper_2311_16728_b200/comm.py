"""A10 + A11 fused over peer memory (SURVEY §8(e) extension f3): the data-parallel optimiser
step as three libgs.so launches -- gs_peer_barrier, gs_reduce_adam_bcast, gs_peer_barrier --
instead of NCCL reduce-scatter, a row-sharded Adam and an NCCL all-gather.

The parameters and gradients of every rank live in one symmetric buffer (torch symmetric
memory: same size on every rank, every peer's buffer mapped into this process; the NVLink SHARP
multicast address when the system has one).  Host logic only: PyTorch allocates and exchanges
the mappings; every number is computed by the kernels behind include/gs.h.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib as L
from .core import AdamConfig, param_rows


def comm_shard(n: int, sh_degree: int, rank: int, world: int) -> tuple[int, int]:
    """This rank's flat element range [e0, e1) of the [K][ld] layout (gs_comm_shard)."""
    return L.gs_comm_shard(n, sh_degree, rank, world)


class PeerAdam:
    """The fused data-parallel optimiser step over peer memory.

    `params` / `grads` are [K][ld] views into a symmetric buffer: the backward adds this rank's
    gradient into `grads`; `step()` sums the gradients of all ranks for this rank's element
    range, applies Adam there (moments for that range only: 1/G of the optimiser state) and
    writes the new parameters -- and zeros into the gradients -- into every rank's buffers.
    The step counter lives on the device, so the launches can be captured in a CUDA graph."""

    def __init__(self, n: int, sh_degree: int, cfg: AdamConfig | None = None, group=None, device=None,
                 multicast: bool = True):
        import torch.distributed._symmetric_memory as symm
        self.group = group if group is not None else dist.group.WORLD
        self.world, self.rank = dist.get_world_size(self.group), dist.get_rank(self.group)
        if self.world > 8:
            raise ValueError("PeerAdam: at most 8 ranks (one NVLink domain of one node)")
        self.n, self.D = n, sh_degree
        self.K = param_rows(sh_degree)
        self.ld = L.param_ld(max(n, 1))
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.cfg = cfg or AdamConfig()
        self.hp = self.cfg.struct()
        self.buf = symm.empty((2 * self.K, self.ld), dtype=torch.float32, device=dev)
        self.buf.zero_()
        self.flags = symm.empty((max(self.world, 4),), dtype=torch.int32, device=dev)
        self.flags.zero_()
        torch.cuda.synchronize(dev)
        dist.barrier(self.group)
        h = symm.rendezvous(self.buf, self.group)
        hf = symm.rendezvous(self.flags, self.group)
        self._handles = (h, hf)  # keep the mappings alive
        gofs = self.K * self.ld * 4
        self.param_ptrs = [int(p) for p in h.buffer_ptrs]
        self.grad_ptrs = [int(p) + gofs for p in h.buffer_ptrs]
        self.flag_ptrs = [int(p) for p in hf.buffer_ptrs]
        mc = int(getattr(h, "multicast_ptr", 0) or 0) if multicast else 0
        self.param_mc, self.grad_mc = (mc, mc + gofs) if mc else (0, 0)
        self.params, self.grads = self.buf[:self.K], self.buf[self.K:]
        self.e0, self.e1 = comm_shard(n, sh_degree, self.rank, self.world)
        q4 = -(-self.K * self.ld // 4 // self.world)
        self.shard_len = 4 * q4  # every rank's moment shard has this length (gather needs equal sizes)
        self.m = torch.zeros(self.shard_len, dtype=torch.float32, device=dev)
        self.v = torch.zeros_like(self.m)
        self.epoch = torch.zeros(1, dtype=torch.int32, device=dev)
        self.t_dev = torch.zeros(1, dtype=torch.int64, device=dev)

    @property
    def t(self) -> int:
        return int(self.t_dev.item())

    def step(self):
        """Barrier (every rank's backward done; step counter + 1) -> fused reduce + Adam +
        broadcast -> barrier (every rank's parameters complete)."""
        L.gs_peer_barrier(self.flag_ptrs, self.rank, self.world, self.epoch, self.t_dev)
        ps = L.params_struct(self.params, self.n, self.D)
        L.gs_reduce_adam_bcast(ps, self.param_ptrs, self.grad_ptrs, self.param_mc, self.grad_mc, self.m, self.v,
                               self.hp, 0, self.t_dev, self.rank, self.world)
        L.gs_peer_barrier(self.flag_ptrs, self.rank, self.world, self.epoch, None)

    def full_state(self) -> tuple:
        """(m, v) of the whole [K][ld] layout (all-gather of the shards), for densification."""
        out = []
        for mine in (self.m, self.v):
            allm = torch.empty(self.world * self.shard_len, dtype=mine.dtype, device=mine.device)
            if self.world > 1:
                dist.all_gather_into_tensor(allm, mine, group=self.group)
            else:
                allm.copy_(mine)
            out.append(allm[:self.K * self.ld].view(self.K, self.ld))
        return tuple(out)

    def load_state(self, m_full: torch.Tensor, v_full: torch.Tensor, t: int):
        """This rank's range of full [K][ld] moments (same on every rank) and the step count."""
        for mine, full in ((self.m, m_full), (self.v, v_full)):
            flat = full.reshape(-1)
            mine.zero_()
            mine[:self.e1 - self.e0] = flat[self.e0:self.e1]
        self.t_dev.fill_(t)
