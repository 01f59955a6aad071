"""Golden outputs of the reference's own front ends, produced by the reference
built from /root/reference (oracle/Makefile target `callers`):

* tests/golden/cli/<name>/  the `hydro2d run <config>` command
  (proj/tools/main.cpp:30-71): stdout, diag.log, fields_*.csv, final.csv,
  final.vtk, for the configs in CLI_CONFIGS;
* tests/golden/cli/case-list.txt  `hydro2d case-list`;
* tests/golden/acceptance_ref.txt  the acceptance suite
  (proj/tests/acceptance.cpp), criteria 1-8.

Run here (the GPU box has no /root/reference):
    make -C oracle callers && python tests/golden/make_cli_golden.py
tests/test_dropin.py runs the same callers compiled against the B200 drop-in
(tests/cpp/Makefile) and requires the same bytes (timings excepted)."""
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.path.join(ROOT, "oracle", "_ref")
OUT = os.path.join(HERE, "cli")

# small configurations of every branch run() has: dynamic two-material with
# field dumps (haas), dynamic AD (impact), imposed-velocity AD / Direct
# (multimat_advect, mono_rotation), the free stream with a step limit
CLI_CONFIGS = {
    "haas_directcf": "case = haas\ndivisor = 10\nmax_steps = 30\noutput_every = 10\n",
    "impact_ad": "case = impact   # water jet\nscheme = AD\ndivisor = 8\nmax_steps = 25\n",
    "multimat_advect_ad": "case = multimat_advect\nscheme = AD\ndivisor = 5\noutput_every = 40\n",
    "mono_rotation_direct": "case = mono_rotation\nscheme = Direct\ndivisor = 5\nt_end = 0.05\n",
    "uniform_multid": "case = uniform\ncorner_scheme = multid\nface_order = 2\ncfl = 0.4\n",
}


def normalise(stdout: str, out_dir: str) -> str:
    """The output directory and the wall-clock figures are run-specific."""
    import re
    s = stdout.replace(out_dir, "<OUT>")
    s = re.sub(r"wall [0-9.e+-]+ s", "wall <T> s", s)
    return s


def normalise_acceptance(text: str) -> str:
    """Criterion timings '(12.3s)' and 'wall=12s' are run-specific."""
    import re
    s = re.sub(r"\([0-9.]+s\)", "(<T>)", text)
    return re.sub(r"wall=[0-9.]+s", "wall=<T>s", s)


def run_cli(binary: str, name: str, text: str, out_dir: str) -> None:
    """Run `binary run <config>` with HYDRO_OUT_DIR = out_dir; stdout goes to
    out_dir/stdout.txt."""
    os.makedirs(out_dir, exist_ok=True)
    cfg = os.path.join(out_dir, "run.cfg")
    with open(cfg, "w") as f:
        f.write(text)
    env = dict(os.environ, HYDRO_OUT_DIR=out_dir)
    r = subprocess.run([binary, "run", cfg], capture_output=True, text=True, env=env, timeout=900)
    with open(os.path.join(out_dir, "stdout.txt"), "w") as f:
        f.write(normalise(r.stdout, out_dir))
    if r.returncode != 0:
        raise RuntimeError(f"{name}: rc {r.returncode}: {r.stdout}{r.stderr}")


def main():
    binary = os.path.join(REF, "hydro2d_ref")
    assert os.path.exists(binary), "build the reference callers first: make -C oracle callers"
    shutil.rmtree(OUT, ignore_errors=True)
    for name, text in CLI_CONFIGS.items():
        run_cli(binary, name, text, os.path.join(OUT, name))
        print(name, sorted(os.listdir(os.path.join(OUT, name))))
    with open(os.path.join(OUT, "case-list.txt"), "w") as f:
        f.write(subprocess.run([binary, "case-list"], capture_output=True, text=True, check=True).stdout)
    if "--no-acceptance" not in sys.argv:
        r = subprocess.run([os.path.join(REF, "acceptance_ref")], capture_output=True, text=True, timeout=7200)
        with open(os.path.join(HERE, "acceptance_ref.txt"), "w") as f:
            f.write(normalise_acceptance(r.stdout))
        print("acceptance rc", r.returncode)


if __name__ == "__main__":
    main()
