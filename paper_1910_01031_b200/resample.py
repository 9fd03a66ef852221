"""Resampling across ranks (SPEC.md:525-543 at N > 1).

Every rank computes the same global resampling index (the log-likelihoods are
all-gathered, `dc_pf_weights` + `dc_residual_resample` run identically on each rank), so
global slot g = rank * M + i takes member idx[g]. Members whose source lives on another
rank travel as packed device buffers (`dc_member_export` / `dc_member_import`) over
torch.distributed point-to-point (NCCL on GPUs); the rest is the local gather
`dc_resample_members`. The result equals one context holding every member and
resampling with the same index, bit for bit.
"""
from __future__ import annotations


def exchange_plan(idx, per_rank: int, rank: int):
    """Plan rank's part of a global resampling.

    idx: global source member per global slot (len = world * per_rank).
    Returns (local_idx, sends, recvs):
      local_idx[i]  local source of slot i, or i where the source is remote (overwritten
                    by an import);
      sends         sorted unique (dest_rank, src_local) pairs this rank exports;
      recvs         sorted (src_rank, src_local, [local slots]) this rank imports.
    Messages between a pair of ranks are posted in ascending src_local on both sides, so
    point-to-point order matches them without tags."""
    n = len(idx)
    if n % per_rank:
        raise ValueError("idx length must be world * per_rank")
    lo = rank * per_rank
    local_idx = list(range(per_rank))
    need = {}
    sends = set()
    for g in range(n):
        src = int(idx[g])
        if not 0 <= src < n:
            raise ValueError("resample index out of range")
        dst_rank, src_rank = g // per_rank, src // per_rank
        if dst_rank == rank and src_rank == rank:
            local_idx[g - lo] = src - lo
        elif dst_rank == rank:
            need.setdefault((src_rank, src - src_rank * per_rank), []).append(g - lo)
        elif src_rank == rank:
            sends.add((dst_rank, src - lo))
    recvs = [(sr, sl, slots) for (sr, sl), slots in sorted(need.items())]
    return local_idx, sorted(sends), recvs


def exchange(plan, nbytes, new_buffer, export_fn, gather_fn, import_fn, dist, sync_fn=None,
             transport_done=None):
    """Run a plan: export the sent members (before the local gather overwrites them),
    exchange over dist point-to-point, gather locally, import the received members.
    transport_done() must block until the received buffers hold their data: with NCCL,
    req.wait() only orders torch's current stream after the transfer, while the imports
    run on the Ensemble's own stream."""
    local_idx, sends, recvs = plan
    sbufs = []
    for dest, src in sends:
        b = new_buffer(nbytes)
        export_fn(src, b)
        sbufs.append((dest, b))
    rbufs = [(sr, new_buffer(nbytes)) for sr, _, _ in recvs]
    if sync_fn:
        sync_fn()  # exports landed before the transport reads them
    ops = [dist.P2POp(dist.isend, b, dest) for dest, b in sbufs]
    ops += [dist.P2POp(dist.irecv, b, sr) for sr, b in rbufs]
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        if transport_done:
            transport_done()
    gather_fn(local_idx)
    for (_, _, slots), (_, b) in zip(recvs, rbufs):
        for i in slots:
            import_fn(i, b)
    if sync_fn:
        sync_fn()


def resample_across_ranks(ens, idx, dist, device):
    """Apply the global resampling index idx to this rank's Ensemble (members
    rank*M .. rank*M+M-1): NCCL point-to-point for members that change rank."""
    import torch

    plan = exchange_plan(idx, ens.n, dist.get_rank())
    exchange(plan, ens.member_bytes(),
             lambda nb: torch.empty(nb, dtype=torch.uint8, device=device),
             lambda m, b: ens.member_export(m, b.data_ptr()),
             lambda li: ens.resample_members(li),
             lambda m, b: ens.member_import(m, b.data_ptr()),
             dist, sync_fn=ens.sync,
             transport_done=(lambda: torch.cuda.current_stream(device).synchronize())
             if str(device).startswith("cuda") else None)
