"""Replay the reference's OWN tests through the B200 path (SURVEY.md §4 reuse
plan).

The unmodified reference package and its test suite are installed in
baseline/_ref (baseline/install_ref.sh; git-ignored, travels to the GPU box).
Each reference test file that renders runs in a subprocess under
``pytest -p paper_2402_00525_b200.splatsort_plugin``: the plugin rebinds
``splatsort.rasterizer.render`` / ``splatsort.render`` / ``splatsort.gradients.
render`` to the B200 path before the test modules import them, so every
``render`` / ``render_depth`` / ``render_trajectory`` / ``backward_render``
call in those tests runs the sm_100a kernels (the plugin counts the calls;
there is no CPU fallback).  Every test of the file must pass:

* test_rasterizer.py -- blend hand values (:56-64), render basics incl. the
  background / transmittance identity and the records replay at 1e-12
  (:207-301), Window(256) == FullPerPixel (:377-383), Hierarchical == Full
  at 1e-12 on shallow scenes (:398-412), determinism and the rank tie-break
  (:434-461), depth buffer, trajectories;
* test_acceptance.py -- the acceptance checks incl. conservation and
  determinism (:381-422) and finite-difference gradients over 50 scenes;
* test_gradients.py -- backward_render on GPU-rendered records vs finite
  differences of GPU renders;
* test_metrics.py -- popping / consistency metrics on GPU-rendered frames.
"""

import os
import re
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.isfile(os.path.join(REF, "tests", "test_rasterizer.py")),
                                 reason="reference not installed (baseline/install_ref.sh)")]

FILES = ["test_rasterizer.py", "test_acceptance.py", "test_gradients.py", "test_metrics.py"]


@pytest.mark.parametrize("fname", FILES)
def test_reference_suite_through_b200(fname, tmp_path):
    xml = tmp_path / "junit.xml"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT]))
    p = subprocess.run([sys.executable, "-m", "pytest", "-p", "paper_2402_00525_b200.splatsort_plugin",
                        "-p", "no:cacheprovider", "-q", "-rf", f"--junitxml={xml}",
                        os.path.join("tests", fname)],
                       cwd=REF, env=env, capture_output=True, text=True, timeout=1800)
    out = p.stdout + p.stderr
    m = re.search(r"splatsort_plugin: (\d+) render calls on the B200 path", out)
    assert m and int(m.group(1)) > 0, out[-3000:]
    suite = ET.parse(xml).getroot()
    suite = suite if suite.tag == "testsuite" else suite.find("testsuite")
    n, fail, err = (int(suite.get(k)) for k in ("tests", "failures", "errors"))
    print(f"{fname}: {n} reference tests, {fail} failures, {err} errors, "
          f"{m.group(1)} B200 render calls")
    assert n > 0 and fail == 0 and err == 0 and p.returncode == 0, out[-6000:]
