"""Multi-GPU all-pairs matrix: one process per GPU, rows of the matrix sharded.

SURVEY.md §8(e): the batch shards naturally (independent pairs). Every rank
gets the whole input (it is tiny: <= 10 MB at the 10k x 10k config), solves a
contiguous block of A rows on its own GPU with no collective, and the blocks
are gathered to rank 0 -- the only exchange: each rank sends exactly its rows
(point to point, no padding) and rank 0 receives them into place. In tri mode (the reference's
symmetric=True, engine.py:200-203, 223-225) each rank solves j >= i for its
rows; rank 0 mirrors the strict upper triangle after the gather, on the device.

Row blocks are balanced by work: equal rows for a full matrix, equal
sum_i (N - i) for the upper triangle.

The compute function is injectable so the sharding and gather logic is tested
with the gloo backend on CPU (tests/test_distributed_gloo.py); the default is
the CUDA path (`api.batch_matrix` on this rank's GPU).
"""

from __future__ import annotations

from typing import Callable, Sequence

import numpy as np


def row_bounds(n_rows: int, world: int, tri: bool, weights: Sequence[float] | None = None):
    """Contiguous [begin, end) row ranges per rank with balanced work."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    if weights is None:
        w = (np.arange(n_rows, 0, -1, dtype=np.float64) if tri
             else np.ones(n_rows, dtype=np.float64))
    else:
        w = np.asarray(weights, dtype=np.float64)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    total = cum[-1]
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        k = int(np.searchsorted(cum, target, side="left"))
        k = min(max(k, bounds[-1]), n_rows)
        bounds.append(k)
    bounds.append(n_rows)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def _global(group, r):
    """Global rank of group rank r (send/recv address global ranks)."""
    if group is None:
        return r
    import torch.distributed as dist
    return dist.get_global_rank(group, r)


def mirror_upper_numpy(m: np.ndarray) -> np.ndarray:
    iu = np.triu_indices(m.shape[0], k=1)
    m[(iu[1], iu[0])] = m[iu]
    return m


def sharded_batch(n_rows: int, n_cols: int, tri: bool,
                  compute: Callable[[int, int], "object"], *, group=None,
                  device=None, dtype=None, gather_to: int = 0):
    """Run `compute(row_begin, row_end) -> (rows, n_cols) block` for this rank's
    rows and gather the full matrix to rank `gather_to` (None elsewhere).

    Blocks may be numpy arrays or torch tensors; the gather runs on `device`
    (a CUDA device with NCCL, CPU with gloo). In tri mode the strictly lower
    part of every block is ignored and the gathered matrix is mirrored.
    """
    import torch
    import torch.distributed as dist

    if not dist.is_initialized():  # one process, no process group: the whole matrix here
        world, rank = 1, 0
    else:
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
    bounds = row_bounds(n_rows, world, tri)
    b0, b1 = bounds[rank]
    if dtype is None:
        dtype = torch.float64
    if device is None:
        device = torch.device("cpu")

    def as_tensor(block):
        t = block if isinstance(block, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(block))
        return t.to(device=device, dtype=dtype).contiguous()

    if world == 1:
        return as_tensor(compute(0, n_rows))
    # Gather without padding: every rank sends exactly its rows (point to
    # point); rank `gather_to` receives each block straight into its rows of
    # the full matrix -- rows x n_cols entries move per rank, nothing more.
    if rank != gather_to:
        if b1 > b0:
            dist.send(as_tensor(compute(b0, b1)), dst=_global(group, gather_to), group=group)
        return None
    full = torch.empty((n_rows, n_cols), dtype=dtype, device=device)
    reqs = [dist.irecv(full[lo:hi], src=_global(group, r), group=group)
            for r, (lo, hi) in enumerate(bounds) if r != rank and hi > lo]
    if b1 > b0:
        full[b0:b1].copy_(as_tensor(compute(b0, b1)))
    for q in reqs:
        q.wait()
    if tri and world > 1:
        if full.is_cuda:
            from .api import mirror_upper_dev
            mirror_upper_dev(full)
        else:
            full = torch.from_numpy(mirror_upper_numpy(full.numpy()))
    return full


def twed_batch_distributed(AA, TAA=None, BB=None, TBB=None, nu=1.0, lamb=None, degree=2,
                           tri=False, *, lam=None, dtype=None, group=None):
    """twed_batch over every rank of the default process group (one GPU each,
    LOCAL_RANK = device). Returns the full numpy matrix on rank 0, None elsewhere
    (without a process group: the whole matrix on the current device)."""
    import torch

    from .api import _dtype, _lam, _to_list, batch_matrix
    from .core import InvalidInputError, TwedParams

    dt = _dtype(dtype)
    params = TwedParams(nu=nu, lam=_lam(lamb, lam), degree=degree)
    list_a = _to_list(AA, TAA, "series_a", dt)
    list_b = None if BB is None else _to_list(BB, TBB, "series_b", dt)
    if tri and list_b is not None:
        raise InvalidInputError("symmetric=True requires both lists to be the same collection")
    n_cols = len(list_a) if list_b is None else len(list_b)
    dev_index = torch.cuda.current_device()

    def compute(b0, b1):
        return batch_matrix(list_a, list_b, params, symmetric=tri, device=dev_index,
                            row_begin=b0, row_end=b1)

    tdtype = torch.float32 if dt == np.float32 else torch.float64
    full = sharded_batch(len(list_a), n_cols, bool(tri), compute, group=group,
                         device=torch.device("cuda", dev_index), dtype=tdtype)
    return None if full is None else full.cpu().numpy()
