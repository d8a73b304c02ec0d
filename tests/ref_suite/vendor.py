"""Copy the reference's own in-scope test files into tests/ref_suite/_vendored
(git-ignored: reference sources are not committed; the directory travels to
the GPU box with the working tree).  Run here, where /root/reference exists;
__graft_entry__.build() calls it.

In scope (SURVEY.md section 4 reuse plan): test_state, test_policy,
test_inference, test_agent, test_collective, test_env, plus their scalar
oracle reference.py.  They run unmodified against paper_2105_08764_b200
through the `graphrl` module alias installed by tests/ref_suite/conftest.py.
"""
from __future__ import annotations

import shutil
from pathlib import Path

SRC = Path("/root/reference/pkg/tests")
DST = Path(__file__).resolve().parent / "_vendored"
FILES = ("reference.py", "test_state.py", "test_policy.py", "test_inference.py",
         "test_agent.py", "test_collective.py", "test_env.py")


def vendor() -> bool:
    if not SRC.is_dir():
        return False
    DST.mkdir(exist_ok=True)
    for f in FILES:
        shutil.copyfile(SRC / f, DST / f)
    return True


if __name__ == "__main__":
    print("vendored" if vendor() else "reference tests not present")
