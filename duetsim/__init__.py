"""Drop-in import name: ``import duetsim`` resolves to the B200 engine.

Callers of the reference package (`duetsim.statevec`, `duetsim.distsim`,
`duetsim.fusion`, `duetsim.gates`, `duetsim.core`, `duetsim.circuits`) get the
device-backed implementations from ``paper_2308_01999_b200`` unchanged.
"""

import sys as _sys

import paper_2308_01999_b200 as _impl
from paper_2308_01999_b200 import circuits, cli, core, distsim, fusion, gates, plan, statevec
from paper_2308_01999_b200 import *  # noqa: F401,F403

for _name, _mod in {
    "core": core,
    "gates": gates,
    "statevec": statevec,
    "fusion": fusion,
    "distsim": distsim,
    "circuits": circuits,
    "plan": plan,
    "cli": cli,
}.items():
    _sys.modules[f"{__name__}.{_name}"] = _mod

__all__ = list(_impl.__all__)
__version__ = _impl.__version__
