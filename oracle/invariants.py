"""Invariant checker for concurrent publish/pull runs (oracle).

Which version a concurrent pull observes depends on timing, so it is not compared for equality
("parity unpinned" by design).  What must hold:
  (i)   the pulled version was published                 (SPEC L633 complete-only serving)
  (ii)  per rollout, pulled versions never decrease       (SPEC L638 monotone newest_complete)
  (iii) the pull returned at least the relay's latest complete version when the pull started
  (iv)  no torn or mixed version: the pulled bytes equal the oracle's pull of that version
        (each trajectory is generated with "a single, consistent policy version")
(iv) is checked by the caller with tp.direct_pull / tp.dst_elements and reported here.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass
class PullRecord:
    rollout: int
    version: int
    latest_at_start: int      # relay's latest complete version observed just before the pull
    content_ok: bool          # (iv) computed by the caller against the oracle's pull of `version`


def check(published: set[int], records: list[PullRecord]) -> list[str]:
    errors = []
    last: dict[int, int] = {}
    for i, r in enumerate(records):
        if r.version == 0:
            continue
        if r.version not in published:
            errors.append(f"#{i}: rollout {r.rollout} pulled unpublished version {r.version}")
        if r.version < last.get(r.rollout, 0):
            errors.append(f"#{i}: rollout {r.rollout} went back from {last[r.rollout]} to {r.version}")
        if r.version < r.latest_at_start:
            errors.append(f"#{i}: rollout {r.rollout} got {r.version} < latest {r.latest_at_start}")
        if not r.content_ok:
            errors.append(f"#{i}: rollout {r.rollout} version {r.version}: torn or mixed bytes")
        last[r.rollout] = max(last.get(r.rollout, 0), r.version)
    return errors
