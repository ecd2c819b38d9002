"""Run the reference's own test suite (/root/reference/pkg/tests, only present
in the build container) against the drop-in: a throw-away `hetrt` package in
/tmp re-exports paper_1405_2912_b200 module by module, and Runtime defaults
to the tests-only HostBackend double (no GPU here).  Prints pytest's summary.

    python tools/run_reference_tests.py [-- extra pytest args]
"""
import os
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF_TESTS = Path("/root/reference/pkg/tests")
MODULES = ["api", "voting", "mapping", "memory", "devices", "executor", "profiles", "experiments",
           "workloads", "errors", "fleets"]

SHIM_INIT = '''
import sys
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
import paper_1405_2912_b200 as _p
from paper_1405_2912_b200 import *  # noqa
from paper_1405_2912_b200 import api as _api
from host_backend import HostBackend as _HB

_orig_init = _api.Runtime.__init__

def _init(self, fleet, config=None, profiles=None, backend=None):
    _orig_init(self, fleet, config, profiles, backend if backend is not None else _HB())

_api.Runtime.__init__ = _init
from paper_1405_2912_b200 import memory as _mem, voting as _vot
_orig_mm = _mem.MemoryManager.__init__

def _mm_init(self, fleet, backend=None, checkpoint_space=None):
    _orig_mm(self, fleet, backend if backend is not None else _HB(), checkpoint_space)

_mem.MemoryManager.__init__ = _mm_init
_vot._default_backend = lambda: _HB()
import importlib
for _m in {modules!r}:
    try:
        sys.modules["hetrt." + _m] = importlib.import_module("paper_1405_2912_b200." + _m)
    except ImportError:
        pass
'''


def main():
    if not REF_TESTS.exists():
        print("reference tests not present (they exist only in the build container)")
        return 0
    with tempfile.TemporaryDirectory() as td:
        pkg = Path(td) / "hetrt"
        pkg.mkdir()
        (pkg / "__init__.py").write_text(SHIM_INIT.format(root=str(ROOT), tests=str(ROOT / "tests"),
                                                          modules=MODULES))
        # the reference's tests import their own conftest helpers; run them in place
        env = dict(os.environ, PYTHONPATH=td, PYTHONDONTWRITEBYTECODE="1")
        extra = sys.argv[sys.argv.index("--") + 1:] if "--" in sys.argv else []
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-rfE", "--tb=line", "-p", "no:cacheprovider",
                            str(REF_TESTS), "--rootdir", td, *extra], env=env, cwd=td, capture_output=True,
                           text=True)
        print(r.stdout[-8000:])
        print(r.stderr[-2000:])
        return r.returncode


if __name__ == "__main__":
    sys.exit(main())
