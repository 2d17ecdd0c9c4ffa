"""B200-native coupled Maxwell-LLG time stepper (drop-in for ``magphon.sim.run``).

Public surface mirrors the reference package ``magphon``: ``sim.run``,
``sim.SimConfig``, ``config.load_config``, ``llg.StepFailure`` ... The hot
loop runs as hand-written sm_100a CUDA kernels behind the C ABI declared in
``include/magphon_b200.h``; there is no CPU fallback.
"""

__version__ = "0.1.0"
