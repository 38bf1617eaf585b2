"""Multi-GPU front end: deterministic request-stream sharding.

Requests are independent, so G GPUs run G independent (scheduler, executor,
arena) servers; nothing crosses GPUs on the data path. The router is a pure
function of request attributes (never of timing), so each shard's sub-trace
is an explicit arrival list that can be replayed through the reference's
simulator (WorkloadSpec::explicit_arrivals, inc/workload.hpp:55-57,66) for
bit-exact per-shard schedule parity. Policies:

  round_robin  request id mod G (a thinned Poisson stream stays Poisson)
  by_client    client (id - 1) mod clients, then client mod G — keeps the
               reference's request->client map (inc/simulator.hpp:297) intact
  dnn_affine   DNN index mod G (bigger single-DNN batches for config 4)

Shard-local ids are renumbered 1..n (Simulator::setup renumbers,
inc/simulator.hpp:262); `global_ids` maps them back.
"""
from __future__ import annotations

from dataclasses import dataclass

from . import scheduler as bs


@dataclass
class Shard:
    rank: int
    arrivals: list          # [(time_ms, mix_index, size_bits)]
    global_ids: list        # shard-local id i+1 -> global id


def route(arrivals: list, world: int, policy: str = "round_robin", clients: int = 0) -> list[int]:
    """Shard index of every arrival (global ids are 1-based positions)."""
    out = []
    for i, (_, dnn, _) in enumerate(arrivals):
        gid = i + 1
        if policy == "round_robin":
            out.append((gid - 1) % world)
        elif policy == "by_client":
            if clients < 1:
                raise ValueError("by_client routing needs clients >= 1")
            out.append(((gid - 1) % clients) % world)
        elif policy == "dnn_affine":
            out.append(dnn % world)
        else:
            raise ValueError(f"unknown routing policy {policy!r}")
    return out


def shard(arrivals: list, world: int, rank: int, policy: str = "round_robin", clients: int = 0) -> Shard:
    owners = route(arrivals, world, policy, clients)
    mine = [(a, i + 1) for i, (a, o) in enumerate(zip(arrivals, owners)) if o == rank]
    return Shard(rank, [a for a, _ in mine], [g for _, g in mine])


def shard_job(job: dict, world: int, rank: int, policy: str = "round_robin") -> tuple[dict, Shard]:
    """A sim job restricted to one shard: the global arrival trace is generated
    with the reference's generator, routed, and handed back as explicit
    arrivals (times as exact bit patterns)."""
    w = job["workload"]
    arr = bs.generate_arrivals(w.get("process", "poisson"), w.get("rate", 100.0), w.get("count", 5000),
                               w.get("seed", 1), w.get("dnn_mix"))
    sim = job.get("sim", {})
    clients = sim.get("clients", 0)
    sh = shard(arr, world, rank, policy, clients)
    wl = {k: v for k, v in w.items() if k not in ("process", "rate", "count")}
    wl["explicit_arrivals"] = [[bs.bits64(t), d, b] for t, d, b in sh.arrivals]
    out = dict(job, workload=wl)
    if clients:
        # Collaborative mode: with clients % world == 0, by-client routing
        # (and round robin) hands shard r the global ids r + world m, i.e.
        # the global clients r, r + world, ...; the shard's own renumbered ids
        # then map to local client (j - 1) % (clients / world) = global
        # client // world, so every request keeps its client's queue and
        # uplink history (reference simulator.hpp:297).
        if clients % world or policy == "dnn_affine":
            raise ValueError("collaborative sharding needs clients % world == 0 and by-client routing")
        out["sim"] = dict(sim, clients=clients // world)
    return out, sh
