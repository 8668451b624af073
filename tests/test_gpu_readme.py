"""The README's usage example runs as written on the GPU (-m gpu)."""
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_readme_usage_example_runs():
    text = open(os.path.join(ROOT, "README.md")).read()
    code = re.search(r"## Usage.*?```python\n(.*?)```", text, re.S).group(1)
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, PYTHONPATH=ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    err = float(re.search(r"tensor\(([0-9.e+-]+)", r.stdout).group(1))
    assert err <= 0.0625, r.stdout     # one bf16 rounding of |K| <= ~6: ulp 2^-5
