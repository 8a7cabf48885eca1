"""The plug-in seam under the reference's own tests.

oracle/stage_ref_pkg.py (run by build()) stages the reference's pure-Python
``svsim`` and its ``tests/test_kernel.py`` / ``test_engine.py`` into
oracle/_ref/pkg and applies INTEGRATION.md's registration of the ``cuda``
backend (kernel/__init__.py:62-75).  Here the reference's tests run unmodified:

* test_kernel.py: the ``backend`` fixture (conftest.py:51-53) parametrises over
  available_backends(), now ('python', 'compiled', 'cuda'); the 13 ``[cuda]``
  cases must pass on the B200.
* test_engine.py with the default backend switched to ``cuda``
  (tests/plug/svsim_cuda_default.py): the reference's engine, transport and
  schemes drive libsvb.so for every local sweep.
"""

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STAGED = os.path.join(REPO, "oracle", "_ref", "pkg")


def _run(args, extra_path=()):
    if not os.path.isdir(os.path.join(STAGED, "svsim")):
        pytest.fail("oracle/_ref/pkg not staged: run build() (oracle/build_ref.sh) where /root/reference exists")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([STAGED, REPO, *extra_path, env.get("PYTHONPATH", "")])
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-rA", "-p", "no:cacheprovider", *args],
                       cwd=STAGED, env=env, capture_output=True, text=True, timeout=1200)
    return r.returncode, r.stdout + r.stderr


def test_reference_kernel_tests_on_cuda_backend(cuda_ok):
    rc, out = _run(["tests/test_kernel.py"])
    assert rc == 0, out[-4000:]
    passed_cuda = re.findall(r"^PASSED tests/test_kernel.py::\S+\[cuda\]", out, re.M)
    assert len(passed_cuda) == 13, out[-4000:]


def test_reference_engine_tests_with_cuda_default(cuda_ok):
    rc, out = _run(["-p", "svsim_cuda_default", "tests/test_engine.py"],
                   extra_path=(os.path.join(REPO, "tests", "plug"),))
    assert rc == 0, out[-4000:]
    assert re.search(r"\d+ passed", out), out[-2000:]
