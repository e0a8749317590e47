"""Copy/compute overlap across batches (host-resident inputs), from the caller's thread.

A batch's host→device staging and sketch (Alg. 1 + §3.3 updates: `sketch_build` /
`sketch_add_dim` / `sketch_del_dim` on pinned host arrays) does not depend on the previous
batch's join, so it can run while that join occupies the SMs: the copy engines move the next
batch's streams and its HBM-bound sketch kernels queue behind the compute-bound join.  The
staging calls block the host only until their own small flag reads complete, so running them
right AFTER the (asynchronous) `mp_join` launch of the current batch keeps the device busy with
the join while the host waits (tools/overlap_probe.py: join 305 ms alone and with the next
batch's 8 GB staging on the prefetch stream; the staging finishes 13 ms after the join).

    pf = Prefetcher(device)
    sk = pf.run(stage, batch[0]); pf.handoff()
    for b in range(nbatches):
        w = mp_create(sk.R, m); mp_join(w)        # caller's stream, asynchronous
        if b + 1 < nbatches:
            sk_next = pf.run(stage, batch[b + 1]) # prefetch stream: overlaps the join
        P, I, inert = mp_finalize(w); ...         # caller's stream
        pf.handoff(); sk = sk_next                # caller's stream waits for the staging

(A worker thread is not needed, and measured slower: the library calls already release the
host while the device works.)
"""
from __future__ import annotations

import torch


class Prefetcher:
    def __init__(self, device):
        self.device = torch.device(device)
        self.stream = torch.cuda.Stream(self.device)
        self._done: torch.cuda.Event | None = None

    def run(self, fn, *args, after: torch.cuda.Event | None = None, **kw):
        """fn(*args, **kw) with the prefetch stream current (every ABI call inside enqueues on
        it), after `after` (an event of the caller's stream) if given."""
        with torch.cuda.stream(self.stream):
            if after is not None:
                self.stream.wait_event(after)
            out = fn(*args, **kw)
            self._done = torch.cuda.Event()
            self._done.record(self.stream)
        return out

    def handoff(self):
        """Order the caller's current stream after everything run() has enqueued."""
        if self._done is not None:
            torch.cuda.current_stream().wait_event(self._done)
