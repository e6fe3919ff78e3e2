"""Re-vendor the reference's own test suite (``/root/reference/pkg/tests``) into this
directory, unmodified except for a provenance header.

This is conformance-test infrastructure, not product code: the reference's 196 tests are
run against this package (``conftest.py`` aliases ``tokencarve`` to
``paper_2505_16864_b200``) on the GPU box, where ``/root/reference`` does not exist -- hence
the copy.  Run ``python tests/ref_suite/_vendor.py`` in the build container to refresh.
"""

import os
import shutil

SRC = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))
FILES = ["oracles.py", "test_acceptance.py", "test_analyze.py", "test_attention.py", "test_cli.py",
         "test_masks.py", "test_partition.py", "test_pipeline.py", "test_sfc.py",
         "test_tensorio.py"]


def main() -> None:
    for name in FILES:
        with open(os.path.join(SRC, name)) as fh:
            body = fh.read()
        header = (f"# Vendored verbatim from the reference suite: pkg/tests/{name}\n"
                  "# (tokencarve 0.1.0); run against paper_2505_16864_b200 -- see conftest.py.\n")
        with open(os.path.join(HERE, name), "w") as fh:
            fh.write(header + body)
    print(f"vendored {len(FILES)} files from {SRC}")


if __name__ == "__main__":
    main()
