"""ORACLE / TEST INFRASTRUCTURE ONLY — CPU model of the paged KV block manager.

The reference keeps a byte ledger only (simulator.cpp:96-98,223-244,443-492);
block tables are the builder's deterministic spec, so the oracle is this
independent pure-Python model of that spec ("parity unpinned" against the
reference for pages; pinned for admission, which uses the reference's byte
rule and is checked through the event log):

  * before a launch, every member's page list grows to cover the positions
    the launch writes: prefill member -> prefilled + chunk tokens, decode
    member -> prompt + decoded (the input token's KV included);
  * each new page is the lowest free page id;
  * at a request's finish, all its pages are released in list order.

It replays a reference-format event log (eventlog.hpp:12-16) plus the trace,
and emits the same "alloc id page" / "free id page" records the product logs.
"""
from __future__ import annotations

import heapq


class PageModel:
    def __init__(self, page_tokens: int, num_pages: int):
        self.page = page_tokens
        self.free = list(range(num_pages))
        heapq.heapify(self.free)
        self.owned: dict[int, list[int]] = {}
        self.log: list[str] = []

    def ensure(self, rid: int, tokens: int) -> None:
        pages = self.owned.setdefault(rid, [])
        while len(pages) * self.page < tokens:
            p = heapq.heappop(self.free)
            pages.append(p)
            self.log.append(f"alloc {rid} {p}")

    def release(self, rid: int) -> None:
        for p in self.owned.pop(rid, []):
            heapq.heappush(self.free, p)
            self.log.append(f"free {rid} {p}")


def replay_pages(event_log: str, prompts: dict[int, int], page_tokens: int, num_pages: int):
    """Re-derive the page log from an event log. Returns (log_text, live tables)."""
    model = PageModel(page_tokens, num_pages)
    prefilled = {rid: 0 for rid in prompts}
    decoded = {rid: 0 for rid in prompts}
    for line in event_log.splitlines():
        t, lane, kind, members, r_p, kv, lat = line.split("\t")
        mem = [] if members == "-" else [tuple(int(x) for x in m.split(":")) for m in members.split(",")]
        if kind == "launch":
            for rid, tokens, _ in mem:
                if prefilled[rid] < prompts[rid]:
                    model.ensure(rid, prefilled[rid] + tokens)
                else:
                    model.ensure(rid, prompts[rid] + decoded[rid])
        elif kind == "complete":
            for rid, tokens, emitted in mem:
                if prefilled[rid] < prompts[rid]:
                    prefilled[rid] += tokens
                    if prefilled[rid] == prompts[rid]:
                        decoded[rid] = 1
                else:
                    decoded[rid] += 1
        elif kind == "finish":
            for rid, _, _ in mem:
                model.release(rid)
    text = "".join(x + "\n" for x in model.log)
    return text, model.owned
