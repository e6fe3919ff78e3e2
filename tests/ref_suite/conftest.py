"""Run the reference's own test suite against the B200 package.

``tokencarve`` (and the submodules the suite imports) are aliased to
``paper_2505_16864_b200`` before collection, so every vendored test file exercises this
package's implementation through the reference's public API with numpy inputs.  All of
them are marked ``gpu`` (the package has no CPU path).  The acceptance criteria's
PASS/FAIL lines are replayed after the run, like the reference's conftest.
"""

import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)

import paper_2505_16864_b200 as _pkg  # noqa: E402
from paper_2505_16864_b200 import (analyze, attention, cli, errors, masks, partition,  # noqa: E402
                                   pipeline, sfc, tensorio)

sys.modules["tokencarve"] = _pkg
for _name, _mod in (("analyze", analyze), ("attention", attention), ("cli", cli),
                    ("errors", errors), ("masks", masks), ("partition", partition),
                    ("pipeline", pipeline), ("sfc", sfc), ("tensorio", tensorio)):
    sys.modules[f"tokencarve.{_name}"] = _mod


@pytest.hookimpl(tryfirst=True)
def pytest_collection_modifyitems(config, items):
    for item in items:
        if str(item.fspath).startswith(HERE):
            item.add_marker(pytest.mark.gpu)


def pytest_terminal_summary(terminalreporter):
    mod = sys.modules.get("test_acceptance")
    if mod is not None and getattr(mod, "RESULT_LINES", None):
        terminalreporter.section("acceptance criteria (reference suite)")
        for line in mod.RESULT_LINES:
            terminalreporter.write_line(line)
