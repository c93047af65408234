"""B200-native SP-NGD optimizer step (arXiv:2002.06015), sm_100a kernels behind
the reference's C++ optimizer/layer API.  See DESIGN.md."""
from . import _native  # noqa: F401
from .spngd import *  # noqa: F401,F403
