"""Host-side multi-process helpers for the row-sharded solve (one process per GPU).

torch.distributed is plumbing only: it broadcasts the 128-byte communicator id that
svm_comm_init needs, reduces timings (max over ranks) and gathers per-rank results for
reporting.  The per-iteration exchange itself runs inside the CUDA kernel over NVLink
(csrc/comm.cu).  Every function takes the device the process group's backend uses
(cuda for NCCL, cpu for gloo in the tests).
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist


def broadcast_uid(uid: Optional[bytes], device) -> bytes:
    """Rank 0 passes the id from svm_comm_unique_id(); every rank gets the same 128 bytes."""
    buf = torch.zeros(128, dtype=torch.uint8, device=device)
    if dist.get_rank() == 0:
        assert uid is not None and len(uid) == 128
        buf.copy_(torch.tensor(list(uid), dtype=torch.uint8))
    dist.broadcast(buf, 0)
    return bytes(buf.cpu().tolist())


def max_over_ranks(value: float, device) -> float:
    """The job's time is the slowest rank's (timing rule: max over ranks)."""
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(local: torch.Tensor, blocks: Sequence[Tuple[int, int]], device) -> torch.Tensor:
    """Concatenate every rank's row block (blocks[r] = (lo, hi)) on every rank."""
    world = dist.get_world_size()
    assert len(blocks) == world
    width = max(hi - lo for lo, hi in blocks)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=device)
    pad[: local.shape[0]] = local
    parts: List[torch.Tensor] = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([p[: hi - lo] for p, (lo, hi) in zip(parts, blocks)])
