"""Multi-GPU plumbing of the benchmark: one process per GPU, each simulating
its own replica of the scene ("replicas only": the config-2 scene is a
single-GPU scene per the north star).  torch.distributed
carries only the timing collectives -- a barrier around the timed region and
max / sum reductions of per-rank totals -- never solver data.

The whole-job metric is the standard weak-scaling aggregate:
  value = (sum over ranks of PNCG iterations) / (max over ranks of time).
"""

from __future__ import annotations

import os
from dataclasses import dataclass


@dataclass
class ReplicaGroup:
    world_size: int = 1
    rank: int = 0
    local_rank: int = 0
    device: str = "cpu"

    @classmethod
    def from_env(cls, backend: str | None = None):
        """RANK / LOCAL_RANK / WORLD_SIZE / MASTER_* as torchrun sets them;
        backend 'nccl' on GPUs, 'gloo' for CPU tests."""
        import torch
        import torch.distributed as dist

        ws = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        local = int(os.environ.get("LOCAL_RANK", "0"))
        backend = backend or ("nccl" if torch.cuda.is_available() else "gloo")
        device = f"cuda:{local}" if backend == "nccl" else "cpu"
        if ws > 1 and not dist.is_initialized():
            kw = {"device_id": torch.device("cuda", local)} if backend == "nccl" else {}
            dist.init_process_group(backend, **kw)
        return cls(ws, rank, local, device)

    def barrier(self):
        if self.world_size > 1:
            import torch.distributed as dist

            dist.barrier()

    def _reduce(self, v: float, op: str) -> float:
        if self.world_size == 1:
            return float(v)
        import torch
        import torch.distributed as dist

        t = torch.tensor([float(v)], dtype=torch.float64, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        return float(t.item())

    def allmax(self, v: float) -> float:
        return self._reduce(v, "max")

    def allsum(self, v: float) -> float:
        return self._reduce(v, "sum")

    def aggregate(self, local_units: float, local_seconds: float) -> tuple[float, float, float]:
        """(whole-job units/s, all units, max seconds)."""
        units = self.allsum(local_units)
        secs = self.allmax(local_seconds)
        return units / secs if secs > 0 else 0.0, units, secs

    def close(self):
        if self.world_size > 1:
            import torch.distributed as dist

            if dist.is_initialized():
                dist.destroy_process_group()
