"""The README's Python example runs as written on the GPU (the documented calls and their return
values stay in step with the binding)."""
import os
import re

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_readme_example_runs():
    text = open(os.path.join(ROOT, "README.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", text, re.S)
    assert blocks, "no python block in README.md"
    ns = {}
    exec(compile(blocks[0], "README.md", "exec"), ns)
    import torch

    assert bool((ns["st"] == 0).all()) and int(ns["n"].min()) > 0
    assert torch.equal(ns["got"][:, : int(ns["n"].min()) // 8], ns["msg"][:, : int(ns["n"].min()) // 8])
