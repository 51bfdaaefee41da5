"""bench.py --impl reference runs the reference alone: nothing from the
product package (libfmm.so, libfmmcuda.so) and not the C restatement
(liboracle.so) is mapped into its process -- only oracle/_ref/libfmmref.so,
the unmodified reference compiled from /root/reference."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT
from oracle import oracle as O


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")
def test_reference_arm_loads_only_the_reference():
    code = ("import sys, runpy; sys.argv = ['bench.py', '--impl', 'reference', '--n', '40000', "
            "'--levels', '5', '--steps', '8', '--warmup', '1', '--no-fmm']; "
            "import bench; bench.main(); "
            "maps = open('/proc/self/maps').read(); "
            "print('MAPS', sorted({l.split()[-1] for l in maps.splitlines() "
            "if l.split()[-1].startswith('" + ROOT + "')}))")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                         timeout=300, check=True).stdout
    line = json.loads([l for l in out.splitlines() if l.startswith("{")][0])
    maps = eval([l for l in out.splitlines() if l.startswith("MAPS")][0][5:])
    assert maps == [os.path.join(ROOT, "oracle", "_ref", "libfmmref.so")], maps
    assert line["impl"] == "reference" and line["same_config"] is True
    assert line["cpu_baseline"]["kind"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["value"] > 0
