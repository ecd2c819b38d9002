"""The drop-in exposes every public name of the reference package, module by
module (tests/golden/reference_api.json, recorded from the reference by
tests/golden/make_api_golden.py), so `import paper_1405_2912_b200 as hetrt`
and `from hetrt.<module> import <name>` keep working."""
import importlib
import json
from pathlib import Path

import pytest

API = json.loads((Path(__file__).parent / "golden" / "reference_api.json").read_text())


@pytest.mark.parametrize("module", sorted(API))
def test_module_exposes_reference_names(module):
    mod = importlib.import_module("paper_1405_2912_b200" + ("" if module == "__init__" else "." + module))
    missing = [n for n in API[module] if not hasattr(mod, n)]
    assert not missing, f"{module}: missing {missing}"
