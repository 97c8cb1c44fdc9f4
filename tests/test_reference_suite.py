"""Drop-in check at the API level: the reference's OWN page-pool test module
(/root/reference/pkg/tests/test_pagemem.py, 29 tests incl. the randomized
invariant runs and the hypothesis properties) executed unchanged against this
package, through a shim ``hiermem`` package whose ``pagemem`` / ``errors`` /
``footprint.TensorSpec`` are ours.  Runs only where the reference checkout
exists (the build container); the reference file is read in place, never
copied into the repo.
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import ROOT

REF_TEST = Path("/root/reference/pkg/tests/test_pagemem.py")

SHIM = {
    "__init__.py": '"""Shim: the reference package name, this build\'s page pools."""\n',
    "errors.py": "from paper_2303_02868_b200.errors import AllocationError, ConfigError, MoveError, ProtocolError  # noqa\n",
    "footprint.py": "from paper_2303_02868_b200.workloads import TensorSpec  # noqa\n",
    "pagemem.py": ("from paper_2303_02868_b200.pagemem import (  # noqa\n"
                   "    MIN_PAGE_BYTES, NOT_READY, PAGE_BYTES_DEFAULT, ManagedTensor, Page, PageManager,\n"
                   "    Tier, TierPool, TransferDescriptor, fragmentation, pool_init, tensor_allocate,\n"
                   "    tensor_release)\n"),
}


@pytest.mark.skipif(not REF_TEST.exists(), reason="reference checkout only in the build container")
def test_reference_pagemem_suite_runs_on_native_table(tmp_path):
    shim = tmp_path / "shim" / "hiermem"
    shim.mkdir(parents=True)
    for name, text in SHIM.items():
        (shim / name).write_text(text)
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(tmp_path / "shim"), str(ROOT)]))
    res = subprocess.run([sys.executable, "-m", "pytest", str(REF_TEST), "-q", "-p", "no:cacheprovider",
                          "--rootdir", str(tmp_path), "-c", os.devnull],
                         cwd=tmp_path, env=env, capture_output=True, text=True, timeout=600)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-3000:]
    assert "29 passed" in out, out[-1000:]
    # and it really was our implementation that ran
    probe = subprocess.run([sys.executable, "-c", "import hiermem.pagemem as p; print(p.PageManager.__module__)"],
                           cwd=tmp_path, env=env, capture_output=True, text=True)
    assert probe.stdout.strip() == "paper_2303_02868_b200.pagemem"
