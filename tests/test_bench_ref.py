"""bench.py's reference arm runs the reference alone: the unmodified reference
headers (oracle/_ref) on every GLCM of one step, with none of the engine (no
package import, libtexforge_cuda.so never mapped). CPU only."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = r"""
import runpy, sys, json
sys.argv = ["bench.py", "--impl", "reference", "--workload", "c1", "--steps", "2", "--warmup", "3"]
runpy.run_path("bench.py", run_name="__main__")
maps = open("/proc/self/maps").read()
print(json.dumps({"pkg": [m for m in sys.modules if m.startswith("paper_1710_06189_b200")],
                  "engine_so": "libtexforge_cuda" in maps, "ref_so": "libtexforge_ref" in maps}))
"""


def test_reference_arm_loads_only_the_reference():
    from oracle import oracle as O
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([sys.executable, "-c", PROBE], capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    bench, probe = lines[0], lines[-1]
    assert bench["impl"] == "reference" and bench["value"] > 0
    assert bench["config"]["glcms_per_step"] == 1  # c1: the whole step (1 GLCM), not a rotating sample
    assert probe == {"pkg": [], "engine_so": False, "ref_so": True}
