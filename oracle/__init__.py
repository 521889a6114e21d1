"""CPU fp64 oracle for one M-ABD implicit step — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference`` arm) may import anything under ``oracle/``. The
product path (``paper_2603_08079_b200``) never imports it and shares no code with
it; see DESIGN.md "Oracle".
"""
from .mabd_oracle import *  # noqa: F401,F403
from .mabd_oracle import __all__  # noqa: F401
