"""Golden output of tests/cpp/api_client.cpp compiled against the UNMODIFIED reference
(its headers under /root/reference/proj/include and the objects oracle/Makefile compiled
from /root/reference/proj/src with the reference's own flags). Run in the build container:

    make -C oracle ref && python tests/golden/gen_api_client.py

writes tests/golden/api_client_ref.txt, which tests/test_cpp_drop_in.py compares with the
same client built against include/mfreg_b200.hpp on the GPU."""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = "/root/reference/proj"
OBJS = ["counters", "curvature", "multilevel", "ngf", "optimizer", "parallel", "transfer", "volume"]


def main():
    exe = os.path.join(tempfile.mkdtemp(), "api_client_ref")
    objs = [os.path.join(ROOT, "oracle", "_ref", "obj", f"{o}.o") for o in OBJS]
    subprocess.run(["g++", "-std=c++20", "-O2", "-DMFREG_REFERENCE", f"-I{REF}/include",
                    os.path.join(ROOT, "tests", "cpp", "api_client.cpp"), *objs, "-pthread", "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    with open(os.path.join(ROOT, "tests", "golden", "api_client_ref.txt"), "w") as f:
        f.write(out)
    print(f"{len(out.splitlines())} lines")


if __name__ == "__main__":
    sys.exit(main())
