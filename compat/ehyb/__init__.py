"""`ehyb` import alias for the B200 drop-in: lets code (and the reference's
own test files) written against `import ehyb` run on paper_2204_06666_b200
unchanged. Put compat/ on sys.path ahead of any installed `ehyb`."""

import os as _os
import sys as _sys

_root = _os.path.dirname(_os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
if _root not in _sys.path:
    _sys.path.insert(0, _root)

from paper_2204_06666_b200 import *  # noqa: F401,F403,E402
from paper_2204_06666_b200 import __all__, __version__  # noqa: F401,E402
