"""Multi-GPU: sequences are the shard unit; the only collective is an
all-gather of per-rank eviction / free-block counters.

The reference couples nothing across sequences except the shared free pool
(compress loops sequences independently, compression.py:327-354; budgets are
per sequence, engine.py:360-377; decode is per (seq, layer),
attention.py:92-127).  So each rank (one process per GPU) owns a private
unified cache, free pool, tables and metrics store for its sequences
(rank-local block ids), and no KV, metric or table ever crosses NVLink.

* ``shard_sequences`` / ``owner_of``: placement (round-robin by default,
  contiguous ranges optional).
* ``gather_counts`` / ``CountGather``: the per-round all-gather.  With NCCL
  the counters stay on the device (the compress totals tensor is gathered
  stream-ordered, no host sync inside a timed round); with gloo they are
  host integers.
* ``ShardedEngine``: the reference Engine's scheduling loop (engine.py:
  264-301) run rank-locally over the rank's share of the submitted requests,
  with every step's StepRecord counters all-gathered so each rank also sees
  the job-wide totals.  Ranks step in lock-step until every rank is idle
  (a finished rank keeps contributing empty records), so the collectives
  always match.  Rank r's records equal a single-GPU Engine run on the
  requests r owns (tests/golden: reference engine on each shard).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch
import torch.distributed as dist

# StepRecord counters exchanged per step (engine.py:160-189)
RECORD_FIELDS = ("admitted", "batch_size", "compressions", "blocks_freed", "kvs_evicted", "preemptions", "finished",
                 "free_blocks", "fragmentation")
# compress totals (kvc_evict_args.totals): freed blocks, evicted KVs, moves, free count
ROUND_FIELDS = ("blocks_freed", "kvs_evicted", "moves", "free_blocks")


def _world(group=None) -> tuple[int, int]:
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def owner_of(index: int, world: int, num_items: int | None = None, policy: str = "round_robin") -> int:
    """Rank that owns item `index` of `num_items` (round-robin: index mod
    world; contiguous: equal ranges in order)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    if policy == "round_robin":
        return index % world
    if policy == "contiguous":
        if num_items is None:
            raise ValueError("contiguous placement needs num_items")
        per = -(-num_items // world)
        return min(index // max(per, 1), world - 1)
    raise ValueError(f"unknown placement policy {policy!r}")


def shard_sequences(seq_ids, rank: int, world: int, policy: str = "round_robin") -> list:
    """The sequences of `seq_ids` that live on `rank` (input order kept)."""
    seq_ids = list(seq_ids)
    return [s for i, s in enumerate(seq_ids) if owner_of(i, world, len(seq_ids), policy) == rank]


def _backend_device(group=None) -> torch.device:
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def gather_counts(counts, group=None):
    """All-gather a short vector of int64 counters from every rank.

    `counts` is a list of ints or an int64 tensor.  With NCCL a CUDA tensor
    is gathered on the current stream and a CUDA tensor [world, n] comes
    back without a host sync; otherwise (gloo) a host tensor.  Without an
    initialised process group: [1, n].
    """
    if torch.is_tensor(counts):
        local = counts.to(torch.int64).reshape(-1)
    else:
        local = torch.tensor(list(counts), dtype=torch.int64)
    if not dist.is_available() or not dist.is_initialized():
        return local.reshape(1, -1)
    _, world = _world(group)
    dev = _backend_device(group)
    local = local.to(dev)
    out = torch.empty((world, local.numel()), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(out, local, group=group) if dev.type == "cuda" else \
        dist.all_gather(list(out.unbind(0)), local, group=group)
    return out


def gather_round_counts(totals, group=None):
    """Per-rank (blocks freed, KVs evicted, moves, free blocks) after a
    compression round: `totals` is the round's int64[4] device tensor
    (EvictionPlan.totals).  Returns [world, 4] (device tensor under NCCL)."""
    return gather_counts(totals, group)


@dataclass
class GlobalStepRecord:
    """Job-wide view of one lock-step: the counters summed over ranks and
    each rank's own record."""

    step: int
    totals: dict
    per_rank: list = field(default_factory=list)


class ShardedEngine:
    """Rank-local Engine over this rank's share of the requests.

    `engine` is this rank's Engine (its own device cache; sequences never
    leave it).  Requests are submitted globally, in the same order on every
    rank; request i is kept by rank owner_of(i).  `step()` advances the
    local engine (or records an idle step when it has nothing to do) and
    all-gathers the StepRecord counters.
    """

    def __init__(self, engine, group=None, policy: str = "round_robin"):
        self.engine = engine
        self.group = group
        self.policy = policy
        self.rank, self.world = _world(group)
        self._submitted = 0
        self.owned: list = []  # global request indices kept by this rank
        self.steps = 0

    def submit(self, source) -> bool:
        """Submit global request #i; returns True when this rank keeps it."""
        i = self._submitted
        self._submitted += 1
        if owner_of(i, self.world) != self.rank:
            return False
        self.engine.submit(source)
        self.owned.append(i)
        return True

    @property
    def active(self) -> bool:
        return self.engine.active

    def any_active(self) -> bool:
        flags = gather_counts([int(self.engine.active)], self.group)
        return bool(flags.sum().item())

    def step(self):
        """One lock-step: local record (None when idle) + the gathered view."""
        self.steps += 1
        rec = self.engine.step() if self.engine.active else None
        local = [getattr(rec, f) if rec is not None else 0 for f in RECORD_FIELDS]
        if rec is None:  # an idle rank still reports its pool state
            local[RECORD_FIELDS.index("free_blocks")] = self.engine.manager.free_count
        allr = gather_counts(local, self.group).cpu().tolist()
        totals = {f: sum(r[j] for r in allr) for j, f in enumerate(RECORD_FIELDS)}
        return rec, GlobalStepRecord(step=self.steps, totals=totals,
                                     per_rank=[dict(zip(RECORD_FIELDS, r)) for r in allr])

    def run_to_completion(self, max_steps: int = 1_000_000):
        """Step every rank until all are idle.  Returns (this rank's records
        while it was active, the global records)."""
        local, glob = [], []
        while self.any_active():
            if self.steps >= max_steps:
                raise RuntimeError(f"workload did not finish within {max_steps} steps")
            rec, g = self.step()
            if rec is not None:
                local.append(rec)
            glob.append(g)
        return local, glob
