"""Host-side plumbing of the slab decomposition: which part of the global
arrays each rank owns, and the NCCL id bootstrap over torch.distributed.  Marshalling only:
the partition itself comes from the C ABI (`mg_partition`), the exchanges run in libmgcg.

Rank r of `nranks` holds slabs [r*nslab, (r+1)*nslab) of S = nranks*nslab; it owns element
layers [e_begin, e_end) along axis 0 and node planes [e_begin, e_end) (+ plane N0 on the last
rank).  Arrays are C order with axis 0 slowest, so each owned part is one contiguous slice.
"""

from __future__ import annotations

from dataclasses import dataclass
from math import prod

import numpy as np

from . import mg_partition


@dataclass(frozen=True)
class RankPart:
    rank: int
    nranks: int
    e_begin: int          # owned element layers [e_begin, e_end)
    e_end: int
    elem0: int            # slice of the global element array
    elem1: int
    dof0: int             # slice of a global (., n) vector
    dof1: int


def rank_part(nel, levels, nranks, rank, nslab=1) -> RankPart:
    S = nranks * nslab
    e_begin = mg_partition(nel, levels, S, rank * nslab)[0]
    e_end = mg_partition(nel, levels, S, rank * nslab + nslab - 1)[1]
    d = len(nel)
    layer_elems = prod(nel[1:])
    plane_nodes = prod(n + 1 for n in nel[1:])
    last = rank == nranks - 1
    p1 = e_end + (1 if last else 0)
    return RankPart(rank, nranks, e_begin, e_end, e_begin * layer_elems, e_end * layer_elems,
                    d * e_begin * plane_nodes, d * p1 * plane_nodes)


def local_inputs(inp: dict, part: RankPart) -> dict:
    """Slice the global seeded inputs (workloads.generate) to this rank's owned part."""
    out = dict(E=np.ascontiguousarray(inp["E"][part.elem0:part.elem1]),
               Es=np.ascontiguousarray(inp["Es"][part.elem0:part.elem1]),
               fixed=np.ascontiguousarray(inp["fixed"][part.dof0:part.dof1]),
               rhs=np.ascontiguousarray(inp["rhs"][:, part.dof0:part.dof1]))
    if "phi" in inp:
        out["phi"] = np.ascontiguousarray(inp["phi"][:, part.dof0:part.dof1])
    return out


def bootstrap_nccl_id(rank: int, nranks: int) -> bytes | None:
    """Rank 0 draws the NCCL unique id; torch.distributed (any backend) broadcasts it."""
    if nranks <= 1:
        return None
    import torch
    import torch.distributed as dist

    from . import mg_nccl_unique_id
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    buf = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(mg_nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(buf, 0)
    return bytes(buf.cpu().numpy().tobytes())


def gather_owned(x_local, part: RankPart, n_glob: int):
    """All ranks' owned slices of an (R, n_local) torch tensor, reassembled into the global
    (R, n_glob) vector on every rank (all_gather of slices padded to the largest; works with the
    nccl backend on CUDA tensors and gloo on CPU tensors).  Used by bench.py's N > 1 self-check."""
    import torch
    import torch.distributed as dist
    R = x_local.shape[0]
    spans = [None] * part.nranks
    dist.all_gather_object(spans, (part.dof0, part.dof1))
    mx = max(b - a for a, b in spans)
    buf = torch.zeros((R, mx), dtype=x_local.dtype, device=x_local.device)
    buf[:, :x_local.shape[1]] = x_local
    outs = [torch.empty_like(buf) for _ in range(part.nranks)]
    dist.all_gather(outs, buf)
    full = torch.empty((R, n_glob), dtype=x_local.dtype, device=x_local.device)
    for (a, b), o in zip(spans, outs):
        full[:, a:b] = o[:, :b - a]
    return full
