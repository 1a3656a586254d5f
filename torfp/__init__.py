"""Drop-in module name for Python callers of the reference's pybind module `torfp`
(python/bindings.cpp): the same function names, keyword arguments, dict keys and exception
classes, served by the B200 engine (paper_2009_01177_b200, C ABI libtor_b200.so).

The reference's instruction scheduler bindings (load_dag / schedule / simulate / expand_dag,
a Sunway ISA model) are outside this engine's scope and raise
NotImplementedError.
"""
from paper_2009_01177_b200 import *  # noqa: F401,F403
from paper_2009_01177_b200 import __all__ as _engine_all


def _out_of_scope(*_a, **_k):
    raise NotImplementedError("the instruction scheduler (scheduler.cpp) is not part of the B200 engine")


load_dag = schedule = simulate = expand_dag = _out_of_scope
__all__ = list(_engine_all) + ["load_dag", "schedule", "simulate", "expand_dag"]
