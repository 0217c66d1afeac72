"""sfgen: seeded synthetic INPUT generators shared by the oracle tests and the CUDA path.

Holds no step of the structure-flow filter's arithmetic: it builds grid geometry
(the Spherepix data structure), renders brightness/depth of
analytic scenes and their ground-truth structure flow (L194-198, L701-707), and
fixes run parameters.  See DESIGN.md "Input recipe".
"""
from . import grid, scene, configs  # noqa: F401
from .configs import CONFIGS, Params, Sequence, config_sequence, default_params, make_sequence  # noqa: F401
