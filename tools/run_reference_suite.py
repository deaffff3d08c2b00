"""Run the reference's OWN test suite (pkg/tests, shipped unmodified in
oracle/_ref/tests by oracle/build_ref.sh) against paper_2411_03416_b200.

`gvplan` and each `gvplan.<module>` are aliased to this package's module of
the same name (the API mirror of gvplan/__init__.py:9-67). The one module the
package deliberately does not provide — `gvplan._kernels_py`, the reference's
pure-numpy twin that test_factors.py:246 uses as the comparison backend — is
loaded from the reference itself. Needs a GPU (the package has no CPU path).

    python tools/run_reference_suite.py [--junit out.xml] [pytest args...]

Prints one JSON summary line (passed / failed / skipped / errors and the
failing node ids)."""

from __future__ import annotations

import importlib
import importlib.util
import json
import os
import pkgutil
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "oracle", "_ref")


def install_alias():
    sys.path.insert(0, REPO)
    import paper_2411_03416_b200 as P

    sys.modules["gvplan"] = P
    for mod in pkgutil.iter_modules(P.__path__):
        if mod.name.startswith("lib"):  # libgvp_b200.so is the ctypes library, not a module
            continue
        m = importlib.import_module(f"paper_2411_03416_b200.{mod.name}")
        sys.modules[f"gvplan.{mod.name}"] = m
    spec = importlib.util.spec_from_file_location("gvplan._kernels_py",
                                                  os.path.join(REF, "gvplan", "_kernels_py.py"))
    kp = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(kp)
    sys.modules["gvplan._kernels_py"] = kp
    P._kernels_py = kp
    return P


class Collect:
    def __init__(self):
        self.out = {"passed": 0, "failed": 0, "skipped": 0, "errors": 0, "failures": []}

    def pytest_runtest_logreport(self, report):
        if report.when == "call" or (report.when == "setup" and report.outcome != "passed"):
            if report.passed:
                self.out["passed"] += 1
            elif report.skipped:
                self.out["skipped"] += 1
            elif report.when == "setup":
                self.out["errors"] += 1
                self.out["failures"].append(report.nodeid)
            else:
                self.out["failed"] += 1
                msg = str(report.longrepr).strip().splitlines()
                self.out["failures"].append(f"{report.nodeid}: {msg[-1] if msg else ''}"[:300])


def main(argv):
    import pytest

    P = install_alias()
    assert P.HAVE_EXTENSION, "no CUDA device / libgvp_b200.so not built"
    tests = os.path.join(REF, "tests")
    if not os.path.isdir(tests):
        raise SystemExit("oracle/_ref/tests missing: run oracle/build_ref.sh")
    col = Collect()
    rc = pytest.main(["-q", "-p", "no:cacheprovider", "--rootdir", tests, tests] + argv, plugins=[col])
    col.out["exit_code"] = int(rc)
    print(json.dumps(col.out))
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
