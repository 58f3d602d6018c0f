"""Copy the reference's test suite verbatim into tests/reference_suite/_vendored
(git-ignored).  Run by __graft_entry__.build() when /root/reference exists;
the copy then travels to the GPU box with the working tree."""

import os
import shutil
import sys

SRC = "/root/reference/pkg/tests"
DST = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_vendored")
FILES = ("helpers.py", "test_algebra.py", "test_containers.py", "test_kernels.py")


def vendor(src=SRC, dst=DST) -> bool:
    if not os.path.isdir(src):
        return False
    os.makedirs(dst, exist_ok=True)
    for f in FILES:
        shutil.copyfile(os.path.join(src, f), os.path.join(dst, f))
    return True


if __name__ == "__main__":
    ok = vendor()
    print("vendored" if ok else f"{SRC} absent: nothing vendored")
    sys.exit(0)
