"""Generate tests/golden/runner/ from the UNMODIFIED reference runner.

Runs the reference's own dolb_run (oracle/_ref/libdolb_ref.so: the reference
sources incl. runner.cpp and capi.cpp compiled where they lie, `make -C oracle
ref`) on each RUNNER_CASES configuration and keeps its artefacts: series.csv,
profiles.csv, the manifest (run.out and the geometry path replaced by
placeholders), perf.csv's deterministic columns and the sha256 of every DOLB1
dump. The GPU runner must reproduce them byte for byte
(tests/test_dolb_capi.py).

    python tests/golden/make_runner_golden.py

The reference library is driven in a process that has NOT imported numpy: its
perf.csv writer (ostream << int64 instantiated inside the reference objects)
faults once numpy has initialised the C++ locale machinery first, so this
script loads nothing but ctypes (runner.py's Dolb wrapper, by file path).
"""
import hashlib
import json
import os
import shutil
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
from runner_cases import RUNNER_CASES, normalize_manifest, resolve_paths  # noqa: E402


def _load_dolb_wrapper():
    """paper_2506_09242_b200/runner.py without importing the package (numpy)."""
    import importlib.util
    import types
    pkg = types.ModuleType("_dolbpkg")
    pkg.__path__ = [os.path.join(ROOT, "paper_2506_09242_b200")]
    sys.modules["_dolbpkg"] = pkg
    for name in ("build", "runner"):
        spec = importlib.util.spec_from_file_location(f"_dolbpkg.{name}",
                                                      os.path.join(ROOT, "paper_2506_09242_b200", f"{name}.py"))
        mod = importlib.util.module_from_spec(spec)
        sys.modules[f"_dolbpkg.{name}"] = mod
        spec.loader.exec_module(mod)
    return sys.modules["_dolbpkg.runner"].Dolb


Dolb = _load_dolb_wrapper()

OUT = os.path.join(HERE, "runner")


def main():
    ref = Dolb(os.path.join(ROOT, "oracle", "_ref", "libdolb_ref.so"))
    os.makedirs(OUT, exist_ok=True)
    index = {}
    for name, cfg in RUNNER_CASES.items():
        tmp = tempfile.mkdtemp(prefix="dolb_ref_")
        try:
            values = resolve_paths(cfg, tmp)
            steps, _ = ref.run(values)
            dst = os.path.join(OUT, name)
            os.makedirs(dst, exist_ok=True)
            entry = {"steps": steps, "dumps": {}}
            for f in sorted(os.listdir(tmp)):
                src = os.path.join(tmp, f)
                if f in ("series.csv", "profiles.csv"):
                    shutil.copyfile(src, os.path.join(dst, f))
                elif f == "manifest":
                    with open(src) as fh:
                        text = normalize_manifest(fh.read(), tmp)
                    with open(os.path.join(dst, f), "w") as fh:
                        fh.write(text)
                elif f == "perf.csv":
                    with open(src) as fh:
                        head, row = fh.read().splitlines()[:2]
                    cols = row.split(",")
                    entry["perf_header"] = head
                    entry["perf_fixed"] = {"cells": cols[0], "steps": cols[1], "tail": cols[4:]}
                elif f.endswith(".dolb"):
                    with open(src, "rb") as fh:
                        entry["dumps"][f] = hashlib.sha256(fh.read()).hexdigest()
            index[name] = entry
            print(name, steps, sorted(os.listdir(tmp)))
        finally:
            shutil.rmtree(tmp)
    with open(os.path.join(OUT, "index.json"), "w") as fh:
        json.dump(index, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
