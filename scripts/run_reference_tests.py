"""Run the reference package's own test files against this package (drop-in
check): `sbr` and its submodules are aliased to paper_2604_09243_b200 by a
pytest plugin written to a temp dir; the reference tests' helper module
(tests/meshes.py) njit-calls the reference's private scalar MT, which is
taken from the reference itself.  Reads the reference checkout at run time
(dev tool only: not used by tests/, smoke() or bench.py).

  python scripts/run_reference_tests.py [/root/reference/pkg] [pytest args...]

On a CPU-only box the host-side tests run (103 of 161 in test_geometry,
test_po, test_bvh, test_mie, test_sweep, test_transport pass); the rest need
the GPU and fail with the library's CUDA error.  On a B200 all 161 pass
(profiles/r02_reference_suite_gpu.log); --with-acceptance adds the release
criteria of test_acceptance.py (c8, CPU thread scaling, deselected)."""
import os, subprocess, sys, tempfile

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ref = sys.argv[1] if len(sys.argv) > 1 and os.path.isdir(sys.argv[1]) else "/root/reference/pkg"
extra = sys.argv[2:] if len(sys.argv) > 1 and os.path.isdir(sys.argv[1]) else sys.argv[1:]
shim = f'''
import importlib, importlib.util, os, sys
sys.path.insert(0, {REPO!r})
sys.path.insert(0, {os.path.join(ref, "tests")!r})
import paper_2604_09243_b200 as pkg
sys.modules["sbr"] = pkg
for sub in ("geometry", "bvh", "transport", "po", "sweep", "errors", "mie"):
    sys.modules["sbr." + sub] = importlib.import_module("paper_2604_09243_b200." + sub)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
spec = importlib.util.spec_from_file_location(
    "sbr_ref", {os.path.join(ref, "src", "sbr", "__init__.py")!r},
    submodule_search_locations=[{os.path.join(ref, "src", "sbr")!r}])
m = importlib.util.module_from_spec(spec)
sys.modules["sbr_ref"] = m
spec.loader.exec_module(m)
sys.modules["sbr.geometry"]._tri_hit_t = sys.modules["sbr_ref.geometry"]._tri_hit_t
'''
d = tempfile.mkdtemp()
open(os.path.join(d, "sbrshim.py"), "w").write(shim)
names = ["test_geometry.py", "test_po.py", "test_bvh.py", "test_mie.py", "test_sweep.py",
         "test_transport.py"]
if "--with-acceptance" in extra:
    # the release criteria; c8 (CPU thread scaling of the sweep) has no
    # meaning for the one-call GPU sweep and is deselected
    extra = [a for a in extra if a != "--with-acceptance"] + ["-k", "not c8"]
    names.append("test_acceptance.py")
files = [os.path.join(ref, "tests", f) for f in names]
env = dict(os.environ, PYTHONPATH=d)
sys.exit(subprocess.call([sys.executable, "-m", "pytest", "-p", "sbrshim", "-p", "no:cacheprovider",
                          "--rootdir", d, "-c", os.devnull, "-q", *files, *extra], cwd=d, env=env))
