"""The README's Python example runs as written (-m gpu)."""
import re
import os

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_readme_python_example():
    text = open(os.path.join(ROOT, "README.md")).read()
    code = re.search(r"```python\n(.*?)```", text, re.S).group(1)
    ns = {}
    exec(compile(code, "README.md", "exec"), ns)
    assert ns["out"].shape == (1 << 21, len(ns["levels"]) * 2)
    assert ns["cs"].count == ns["values"].shape[0] > 0
    torch.cuda.synchronize()
