"""pytest plugin (``-p _ref_shim_plugin``): installs the B200 path under the
reference package before the reference's own test modules are imported, so
their ``from semsplat.vq import ...`` bind the adapters
(paper_2603_09632_b200.reference_shim)."""

import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

from paper_2603_09632_b200 import reference_shim  # noqa: E402

INSTALLED = reference_shim.install()


def pytest_terminal_summary(terminalreporter):
    from paper_2603_09632_b200 import _native
    n = _native.launch_count() if _native._lib is not None else 0
    terminalreporter.write_line(f"B200 shim installed over semsplat: {len(INSTALLED)} functions; "
                                f"libxgs kernel launches: {n}")
