"""Install the B200 path behind the reference's own averaging seams.

The reference orchestrator reaches the collective in two places
(orchestrator.py:320-363):

* snapshot barrier: ``multiring.apply_ring_mean(plan.ring_schedule, vals)``,
  looked up as a module attribute at call time (orchestrator.py:329);
* drain barrier: ``AllReduceController(plan.ring_schedule, working, network,
  plan.node_of)``, bound by name at import (orchestrator.py:25, :345).

``install(ravnest)`` points both (and ``multiring.run_allreduce``, used by
oracle.run_verification and the CLI) at this package, translating this
package's exceptions into the reference's own classes so existing
``except StallError`` clauses keep working.  ``uninstall`` restores them.
"""

from __future__ import annotations

import functools
import importlib
import sys

from . import errors as _errors
from . import multiring as _mr

_SAVED: dict = {}


def _translate(ref_errors):
    mapping = {
        _errors.ConfigError: getattr(ref_errors, "ConfigError", None),
        _errors.LayoutError: getattr(ref_errors, "LayoutError", None),
        _errors.ProtocolError: getattr(ref_errors, "ProtocolError", None),
        _errors.StallError: getattr(ref_errors, "StallError", None),
        _errors.SchemaError: getattr(ref_errors, "SchemaError", None),
        _errors.RavnestError: getattr(ref_errors, "RavnestError", None),
    }

    def wrap(fn):
        @functools.wraps(fn)
        def inner(*a, **k):
            try:
                return fn(*a, **k)
            except _errors.RavnestError as e:
                for ours in (type(e), *type(e).__mro__):
                    theirs = mapping.get(ours)
                    if theirs is not None:
                        raise theirs(str(e)) from e
                raise

        return inner

    return wrap


def _controller_class(wrap):
    class AllReduceController(_mr.AllReduceController):
        __doc__ = _mr.AllReduceController.__doc__

        @wrap
        def kickoff(self, now):
            return super().kickoff(now)

        @wrap
        def handle(self, msg, now):
            return super().handle(msg, now)

        @wrap
        def done(self):
            return super().done()

    return AllReduceController


def install(ravnest=None):
    """Patch the reference package (module object or import name 'ravnest')."""
    if ravnest is None or isinstance(ravnest, str):
        ravnest = importlib.import_module(ravnest or "ravnest")
    name = ravnest.__name__
    multiring = sys.modules.get(f"{name}.multiring") or importlib.import_module(f"{name}.multiring")
    orchestrator = sys.modules.get(f"{name}.orchestrator")
    ref_errors = sys.modules.get(f"{name}.errors") or importlib.import_module(f"{name}.errors")
    wrap = _translate(ref_errors)
    if name not in _SAVED:
        _SAVED[name] = {
            "apply_ring_mean": multiring.apply_ring_mean,
            "run_allreduce": multiring.run_allreduce,
            "AllReduceController": multiring.AllReduceController,
            "orch_ctl": getattr(orchestrator, "AllReduceController", None) if orchestrator else None,
            "pkg_run_allreduce": getattr(ravnest, "run_allreduce", None),
        }
    ctl = _controller_class(wrap)
    multiring.apply_ring_mean = wrap(_mr.apply_ring_mean)
    multiring.run_allreduce = wrap(_mr.run_allreduce)
    multiring.AllReduceController = ctl
    if orchestrator is not None and hasattr(orchestrator, "AllReduceController"):
        orchestrator.AllReduceController = ctl
    if hasattr(ravnest, "run_allreduce"):
        ravnest.run_allreduce = multiring.run_allreduce
    return ravnest


def uninstall(ravnest=None):
    if ravnest is None or isinstance(ravnest, str):
        ravnest = importlib.import_module(ravnest or "ravnest")
    name = ravnest.__name__
    saved = _SAVED.pop(name, None)
    if not saved:
        return
    multiring = sys.modules[f"{name}.multiring"]
    multiring.apply_ring_mean = saved["apply_ring_mean"]
    multiring.run_allreduce = saved["run_allreduce"]
    multiring.AllReduceController = saved["AllReduceController"]
    orchestrator = sys.modules.get(f"{name}.orchestrator")
    if orchestrator is not None and saved["orch_ctl"] is not None:
        orchestrator.AllReduceController = saved["orch_ctl"]
    if saved["pkg_run_allreduce"] is not None:
        ravnest.run_allreduce = saved["pkg_run_allreduce"]
