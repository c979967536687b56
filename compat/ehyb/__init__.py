"""`ehyb` import alias for the B200 drop-in: lets code (and the reference's
own test files) written against `import ehyb` run on paper_2204_06666_b200
unchanged. Put compat/ on sys.path ahead of any installed `ehyb`.

The reference's importable surface is the package plus its five modules
(pkg/src/ehyb/{engine,format,partition,matrix_io,cli}.py); each is aliased
in `sys.modules` to the drop-in module of the same name, so
`from ehyb.cli import main` or `import ehyb.engine as E` resolve to the B200
implementation.
"""

import importlib as _importlib
import os as _os
import sys as _sys

_root = _os.path.dirname(_os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
if _root not in _sys.path:
    _sys.path.insert(0, _root)

from paper_2204_06666_b200 import *  # noqa: F401,F403,E402
from paper_2204_06666_b200 import __all__, __version__  # noqa: F401,E402

_SUBMODULES = ("engine", "format", "partition", "matrix_io", "cli")
for _name in _SUBMODULES:
    _mod = _importlib.import_module(f"paper_2204_06666_b200.{_name}")
    _sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod
del _name, _mod
