"""pytest plugin: make `import batchode` (and its submodules the reference's
tests import) resolve to paper_2210_12375_b200, so the reference's own test
files run unmodified against the B200 package (tools/stage_reference_tests.sh)."""
import sys

import paper_2210_12375_b200 as _pkg
from paper_2210_12375_b200 import (cli, controller, dynamics, problems, solver, stepping,  # noqa: F401
                                   tableau)

sys.modules["batchode"] = _pkg
for _name, _mod in (("controller", controller), ("problems", problems), ("solver", solver),
                    ("stepper", stepping), ("tableau", tableau), ("cli", cli)):
    sys.modules["batchode." + _name] = _mod
