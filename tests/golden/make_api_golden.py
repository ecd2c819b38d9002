"""Record the reference package's public names per module (run in the build
container, where /root/reference exists) -> tests/golden/reference_api.json.
tests/test_api_surface.py checks the drop-in exposes every one of them."""
import importlib
import json
import os
import sys
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
MODULES = ["", "api", "voting", "mapping", "memory", "devices", "executor", "profiles", "experiments",
           "workloads", "errors"]
out = {}
for mod in MODULES:
    m = importlib.import_module("hetrt" + ("." + mod if mod else ""))
    names = sorted(n for n in dir(m) if not n.startswith("_") and
                   (not mod or getattr(getattr(m, n), "__module__", "").startswith("hetrt")))
    out[mod or "__init__"] = names
Path(os.path.dirname(os.path.abspath(__file__)), "reference_api.json").write_text(json.dumps(out, indent=1))
print({k: len(v) for k, v in out.items()})
