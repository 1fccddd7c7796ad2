"""Relay tier: Appendix D latency model and the chain-pipelined relay rounds (oracle).

Appendix D:
  L1467  t = s*T_byte + T_start per message; M bytes in k chunks of M/k
  L1491  T(p, k) = (p + k - 2) * (M/k * T_byte + T_start)
  L1509  k* = sqrt((p - 2) * M * T_byte / T_start)
  L1513  T*(p) = M*T_byte + (p-2)*T_start + 2*sqrt((p-2)*M*T_byte*T_start)
SPEC L559-567: optimal_chunks = clamp(round(k*), 1, k_cap); T_start == 0 -> k_cap.

Relay rounds ("The broadcast pipelines model chunk transfers along a chain of
relays, overlapping communication among different hops"; L693 "chunks them, and broadcasts them
down the chain in a pipelined manner"; L670 rollouts pull "without waiting for the resharding and
broadcast to complete"; SPEC L546-547/L633 complete-only serving; L638 monotone newest_complete;
L661 retain 2).  Reading:
  * node 0 is the master (the actor's publish slots), nodes 1..p-1 the relays, chain 0->1->...;
  * a round processes hops i->i+1 in tail-to-head order; on each hop, node i+1 copies the lowest
    chunk of version u that node i holds and it lacks (one chunk per hop per round);
  * a node starts receiving u only into a FREE slot, or a COMPLETE slot that has no readers and
    is not its latest; it starts the NEWEST version its predecessor holds (latest-wins: older
    versions may be skipped, never reordered); while receiving, it pins its predecessor's slot;
  * when all k chunks are present: COMPLETE, latest = max(latest, u); a pull serves only latest.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

FREE, FILLING, COMPLETE = "FREE", "FILLING", "COMPLETE"


# ----------------------------------------------------------------------------------- Appendix D
def chain_latency(p: int, k: int, M: float, T_byte: float, T_start: float) -> float:
    """T(p, k) = (p + k - 2) * (M/k * T_byte + T_start)."""
    if p < 2 or k < 1:
        raise ValueError("need p >= 2 and k >= 1")
    return (p + k - 2) * (M / k * T_byte + T_start)


def k_star(p: int, M: float, T_byte: float, T_start: float) -> float:
    """Continuous optimum k* = sqrt((p-2) M T_byte / T_start)."""
    return math.sqrt((p - 2) * M * T_byte / T_start)


def optimal_chunks(p: int, M: float, T_byte: float, T_start: float, k_cap: int = 1024) -> int:
    """clamp(round(k*), 1, k_cap)."""
    if p < 2:
        raise ValueError("need p >= 2")
    if T_start == 0:
        return k_cap
    return max(1, min(k_cap, round(k_star(p, M, T_byte, T_start))))


def latency_decomposition(p: int, M: float, T_byte: float, T_start: float):
    """(bandwidth, latency, pipeline) terms of T*(p)."""
    bw = M * T_byte
    lat = (p - 2) * T_start
    pipe = 2.0 * math.sqrt((p - 2) * M * T_byte * T_start)
    return bw, lat, pipe


# ------------------------------------------------------------------------------- relay rounds
@dataclass
class Slot:
    version: int = 0
    state: str = FREE
    have: set = field(default_factory=set)
    readers: int = 0
    pinned_src: tuple | None = None     # (node, slot index) this slot pins while FILLING


@dataclass
class Node:
    slots: list
    latest: int = 0
    started: int = 0                    # newest version this node began to receive
    skipped: int = 0


class RelayChain:
    """Deterministic round model of the chain.  All k chunks of a published version are at the
    master at publish time (the master "sends the first chunk")."""

    def __init__(self, p: int, k: int, slots: int = 2):
        if p < 1 or k < 1 or slots < 2:
            raise ValueError("need p >= 1, k >= 1, slots >= 2")
        self.p, self.k = p, k
        self.nodes = [Node([Slot() for _ in range(slots)]) for _ in range(p)]
        self.rounds = 0
        self.last_published = 0
        self.completion_round: dict[tuple[int, int], int] = {}   # (node, version) -> round

    # -- slot rule
    def _acquire(self, node: Node):
        for i, s in enumerate(node.slots):
            if s.state == FREE:
                return i
        for i, s in enumerate(node.slots):
            if s.state == COMPLETE and s.readers == 0 and s.version != node.latest:
                return i
        return None

    def _slot_of(self, node: Node, v: int):
        for i, s in enumerate(node.slots):
            if s.version == v and s.state in (FILLING, COMPLETE):
                return i
        return None

    def publish(self, v: int) -> str:
        """Actor publish into node 0 (never waits): 'ok', 'stale' (v <= last) or 'busy'."""
        if v <= self.last_published:
            return "stale"
        n0 = self.nodes[0]
        i = self._acquire(n0)
        if i is None:
            return "busy"
        s = n0.slots[i]
        s.version, s.state, s.have, s.readers = v, COMPLETE, set(range(self.k)), 0
        n0.latest = max(n0.latest, v)
        n0.started = v
        self.last_published = v
        self.completion_round[(0, v)] = self.rounds
        return "ok"

    def _newest_held(self, node: Node) -> int:
        vs = [s.version for s in node.slots if s.state in (FILLING, COMPLETE)]
        return max(vs) if vs else 0

    def step(self) -> int:
        """One round.  Returns the number of chunk copies made (0 = quiescent)."""
        self.rounds += 1
        moved = 0
        for i in range(self.p - 2, -1, -1):                      # tail-to-head
            pred, node = self.nodes[i], self.nodes[i + 1]
            filling = [j for j, s in enumerate(node.slots) if s.state == FILLING]
            if not filling:
                u = self._newest_held(pred)
                if u <= node.started:
                    continue
                j = self._acquire(node)
                if j is None:
                    continue
                if node.started and u > node.started + 1:
                    node.skipped += u - node.started - 1
                src = self._slot_of(pred, u)
                pred.slots[src].readers += 1
                s = node.slots[j]
                s.version, s.state, s.have, s.readers, s.pinned_src = u, FILLING, set(), 0, (i, src)
                node.started = u
                filling = [j]
            s = node.slots[filling[0]]
                                                                 # predecessor's slot for s.version
            src = pred.slots[s.pinned_src[1]]
            missing = sorted(src.have - s.have)
            if missing:
                s.have.add(missing[0])
                moved += 1
            if len(s.have) == self.k:
                s.state = COMPLETE
                node.latest = max(node.latest, s.version)
                src.readers -= 1
                s.pinned_src = None
                self.completion_round[(i + 1, s.version)] = self.rounds
        return moved

    def run_until_quiescent(self, max_rounds: int = 1_000_000) -> int:
        while max_rounds > 0:
            before = self.state_key()
            self.step()
            if self.state_key() == before:
                return self.rounds
            max_rounds -= 1
        raise RuntimeError("relay rounds did not quiesce")

    def state_key(self):
        return tuple((n.latest, n.started, tuple((s.version, s.state, len(s.have), s.readers)
                                                  for s in n.slots)) for n in self.nodes)

    # -- pull: newest COMPLETE version, pinned while read
    def pin_latest(self, node_id: int):
        n = self.nodes[node_id]
        if n.latest == 0:
            return 0, None
        i = self._slot_of(n, n.latest)
        n.slots[i].readers += 1
        return n.latest, i

    def unpin(self, node_id: int, slot: int):
        self.nodes[node_id].slots[slot].readers -= 1
