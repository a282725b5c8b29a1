"""Asynchronous periodic averaging for live training.

The reference's global loop (orchestrator.py:302-337, Algorithm 2) counts
parameter updates and, each time the count crosses a multiple of kappa,
averages the clusters' parameters with the multi-ring all-reduce; batches
still in flight then land their (stale) updates on the averaged parameters
(pipeline.py:384-411).  On GPUs the averaging need not stop training:

    every kappa updates  snap <- live           (side stream, HBM copy)
                         mean <- ring mean(snap) (side stream, NVLink,
                                                  overlaps further updates)
    tau updates later    live <- mean + (live - snap)   (training stream)

so the tau updates made while the cycle ran are applied on top of the
average, exactly the reference's stale-update semantics with staleness tau.
With tau = 0 the cycle writes the mean straight into live (the blend would
write exactly the mean, live == snap), i.e. the reference's synchronous
snapshot barrier.  The cycle is one kernel per rank
(DistRingGroup); with ``graph=True`` it is captured once in a CUDA graph and
replayed every kappa updates.

Overlap: the cycle runs on a high-priority side stream with an SM budget
(``sm_budget`` SMs; NVLink-bound, it does not need the whole GPU), so the
training kernels keep the remaining SMs.  The snapshot copy also runs on the
side stream; only the next parameter update has to wait for it -- call
``before_update()`` right before the optimizer writes ``live`` (forward and
backward of the next step overlap the copy).
"""

from __future__ import annotations

from .blend import blend_
from .dist import DistRingGroup
from .errors import ConfigError, StallError


class _AveragerCore:
    """The kappa / tau schedule shared by both averagers: snapshots of the
    member(s) this process trains, the cycle on a side stream, the blend.
    Subclasses provide ``_cycle(stream)`` (launch one averaging cycle of
    snap -> mean on ``stream``) and ``group`` (``failed``, ``check``,
    ``close``)."""

    def _setup(self, lives, kappa: int, tau: int, train_stream, graph: bool):
        import torch

        if kappa < 1:
            raise ConfigError(f"kappa must be >= 1, got {kappa}")
        if tau < 0 or tau >= kappa:
            raise ConfigError(f"tau must be in [0, kappa), got {tau}")
        self.lives = list(lives)
        self.snaps = [torch.empty_like(x) for x in self.lives]
        # tau = 0: nothing lands on live during the cycle, so the means go
        # straight into live (the blend would write exactly the mean there);
        # a mean buffer never holds garbage: it starts as the live values
        self.means = self.lives if tau == 0 else [x.clone() for x in self.lives]
        self.kappa, self.tau = kappa, tau
        dev = self.lives[0].device
        self.train_stream = train_stream or torch.cuda.current_stream(dev)
        self.avg_stream = torch.cuda.Stream(device=dev, priority=-1)
        self.t = 0
        self.cycles = 0
        self._pending_at = None
        self._done = None
        self._snapped = None
        self._graph = None
        self._use_graph = graph

    def _raise_if_failed(self) -> None:
        if not self.group.failed():
            return
        self._pending_at = None
        try:
            self.group.check()
        except StallError as e:
            raise StallError(f"averaging cycle {self.cycles} stalled; live parameters left unblended: {e}") from e
        raise StallError(f"averaging cycle {self.cycles} stalled; live parameters left unblended")

    def _launch(self):
        import torch

        self._raise_if_failed()
        # snapshot on the side stream, after everything training has issued;
        # before_update() keeps the next write to `live` behind the copy
        self.avg_stream.wait_stream(self.train_stream)
        with torch.cuda.stream(self.avg_stream):
            for snap, live in zip(self.snaps, self.lives):
                snap.copy_(live)
        self._snapped = torch.cuda.Event()
        self._snapped.record(self.avg_stream)
        if self._use_graph:
            if self._graph is None:
                # warm-up cycle builds the device tables; then capture one cycle
                with torch.cuda.stream(self.avg_stream):
                    self._cycle(self.avg_stream)
                self.avg_stream.synchronize()
                self._graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(self._graph, stream=self.avg_stream):
                    self._cycle(self.avg_stream)
                # the capture itself did not run the cycle
            with torch.cuda.stream(self.avg_stream):
                self._graph.replay()
        else:
            self._cycle(self.avg_stream)
        self._done = torch.cuda.Event()
        self._done.record(self.avg_stream)

    def _finish(self):
        self.before_update()
        # a stalled cycle (a peer slower than the timeout) skipped its folds:
        # its means must not reach the live parameters.  The failure word is
        # host-mapped, so after the cycle's event it reads without a device
        # sync (only the side stream is waited for; tau updates have run
        # since the launch, so the cycle has normally long finished).  With
        # tau = 0 the means land in live directly (a stalled cycle leaves
        # some units averaged and the rest as they were, never garbage); the
        # next launch reports it.
        if self.tau > 0:
            self._done.synchronize()
            self._raise_if_failed()
        self.train_stream.wait_event(self._done)
        if self.tau > 0:
            for live, snap, mean in zip(self.lives, self.snaps, self.means):
                blend_(live, snap, mean, self.train_stream)
        self._pending_at = None
        self.cycles += 1

    def before_update(self) -> None:
        """Call right before the optimizer writes the live parameters: orders
        that write after a pending snapshot copy (no-op otherwise)."""
        if self._snapped is not None:
            self.train_stream.wait_event(self._snapped)
            self._snapped = None

    def step(self) -> bool:
        """Count one local update; start or finish a cycle when due.
        Returns True when a blend was issued at this step."""
        self.t += 1
        finished = False
        if self._pending_at is not None and self.t >= self._pending_at + self.tau:
            self._finish()
            finished = True
        if self.t % self.kappa == 0 and self._pending_at is None:
            self._launch()
            self._pending_at = self.t
            if self.tau == 0:
                self._finish()
                finished = True
        return finished

    def flush(self) -> None:
        """Finish a pending cycle now (end of training)."""
        if self._pending_at is not None:
            self._finish()

    def close(self) -> None:
        self.flush()
        self.train_stream.synchronize()
        self._graph = None
        self.group.close()


class AsyncAverager(_AveragerCore):
    """One rank's side of periodic averaging over a torch.distributed group.

    ``live`` is the rank's flat, contiguous CUDA parameter arena (the
    optimizer updates it in place on ``train_stream``).  Call ``step()``
    after every local update.
    """

    def __init__(self, live, schedule=None, *, starts=None, lens=None, kappa: int, tau: int = 0,
                 cluster_id: int | None = None, acc: str = "f64", protocol: str = "auto",
                 train_stream=None, graph: bool = False, group=None, sm_budget: int = 32):
        self._setup([live], kappa, tau, train_stream, graph)
        self.live, self.snap, self.mean = self.lives[0], self.snaps[0], self.means[0]
        self.group = DistRingGroup(schedule, src=self.snap, dst=self.mean, starts=starts, lens=lens,
                                   cluster_id=cluster_id, acc=acc, protocol=protocol, group=group,
                                   max_blocks=2 * sm_budget if sm_budget else 0)

    def _cycle(self, stream) -> None:
        self.group.average([stream])


class LocalAsyncAverager(_AveragerCore):
    """The same schedule for C clusters trained in ONE process on one GPU
    (``lives[m]`` = cluster position m, ascending cluster id): every kappa
    updates all C arenas are snapshot and averaged on the side stream --
    co-resident in one kernel (``transport="co-resident"``, the TMA kernel),
    or through the multi-rank transports with one rank plan per cluster
    (``"push"``, ``"pull"``, ``"ll"``: the kernels an N-GPU job runs, driven
    from one process) -- and tau updates later each cluster blends.
    Call ``step()`` once per update round (every cluster updated once)."""

    def __init__(self, lives, schedule=None, *, starts=None, lens=None, kappa: int, tau: int = 0,
                 acc: str = "f64", transport: str = "co-resident", train_stream=None, graph: bool = False,
                 options=None):
        from .loopback import LoopbackGroup
        from .plan import LocalRingGroup
        from .schedule import ring_arrays

        self._setup(lives, kappa, tau, train_stream, graph)
        if schedule is not None:
            starts, lens = ring_arrays(schedule)
        if starts is None or lens is None:
            raise ConfigError("pass a schedule or ring starts/lens")
        total = sum(int(n) for n in lens)
        dev = self.lives[0].device.index
        if transport == "co-resident":
            self.group = LocalRingGroup(starts, lens, total, [dev] * len(self.lives), self.lives[0].dtype, acc=acc,
                                        options=options)
            self._run = lambda st: self.group.run({dev: [st]})
        else:
            self.group = LoopbackGroup(starts, lens, total, len(self.lives), self.lives[0].dtype, protocol=transport,
                                       device=dev, acc=acc, options=options)
            self._run = lambda st: self.group.run(after=st)
        self.group.bind_tensors(self.snaps, self.means)

    def _cycle(self, stream) -> None:
        self._run(stream)
