"""pytest plugin (test infrastructure): run the REFERENCE's own test files
against this package.  Loaded with ``-p ref_suite_plugin`` before the
reference's test modules are imported, it routes the reference's averaging
seams to this package (plugin.install: apply_ring_mean, run_allreduce,
AllReduceController).  With RAVNEST_B200_ORACLE_CYCLE=1 (CPU containers) the
GPU cycle is replaced by the oracle, so only the host logic -- argument
handling, errors, the drain controller's message replay -- is under test;
without it the cycles run on the GPU."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


CYCLES = {"n": 0}


class _OracleCycle:
    def __init__(self, schedule, n):
        self.schedule = schedule

    def launch(self, arrays):
        from oracle import ring_oracle

        CYCLES["n"] += 1
        return ring_oracle.ring_mean([r.start for r in self.schedule.rings], [r.length for r in self.schedule.rings],
                                     [np.asarray(a, dtype=np.float64) for a in arrays])

    def ready(self):
        return True

    def wait(self):
        pass


def pytest_configure(config):
    sys.dont_write_bytecode = True
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    import ravnest

    from paper_2401_01728_b200 import multiring as mr
    from paper_2401_01728_b200 import plugin

    if os.environ.get("RAVNEST_B200_ORACLE_CYCLE") == "1":
        mr._HostCycle = _OracleCycle
    else:
        real = mr._HostCycle.launch

        def counted(self, inputs):
            CYCLES["n"] += 1
            return real(self, inputs)

        mr._HostCycle.launch = counted
    plugin.install(ravnest)


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(f"ravnest averaging seams routed to paper_2401_01728_b200: "
                                f"{CYCLES['n']} cycles through the drop-in")
