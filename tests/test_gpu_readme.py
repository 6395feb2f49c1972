"""The README's usage snippet runs as written (documentation stays true to the API)."""
import os
import re

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_readme_python_example_runs():
    text = open(os.path.join(ROOT, "README.md")).read()
    code = re.search(r"## Using it \(Python\)\s+```python\n(.*?)```", text, re.S).group(1)
    ns = {}
    exec(compile(code, "README.md", "exec"), ns)
    r = ns["r"]
    assert (r["status"] == 0).all() and (r["n_matches"] > 200).all()
