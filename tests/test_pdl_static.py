"""Static check: every kernel starts with griddep_wait().

launch_k (csrc/ttg.cu) launches with programmatic stream serialization, so a
kernel may be scheduled while its predecessor drains; only
griddepcontrol.wait makes the predecessor's writes visible.  A kernel body
without the wait is a silent data race on its inputs."""
import glob
import os
import re

CSRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2211_12487_b200", "csrc")


def _kernel_bodies():
    for path in sorted(glob.glob(os.path.join(CSRC, "*.cu*")) + glob.glob(os.path.join(CSRC, "*.inc"))):
        src = open(path).read()
        for m in re.finditer(r"__global__[^{;]*?\b(k_\w+)\s*\(", src):
            i = src.index("{", m.end())
            depth, j = 0, i
            while True:
                if src[j] == "{":
                    depth += 1
                elif src[j] == "}":
                    depth -= 1
                    if depth == 0:
                        break
                j += 1
            yield os.path.basename(path), m.group(1), src[i:j]


def test_every_kernel_waits_on_its_predecessor():
    bodies = list(_kernel_bodies())
    assert len(bodies) > 20
    missing = [f"{f}:{k}" for f, k, body in bodies if "griddep_wait()" not in body]
    assert not missing, f"kernels without griddep_wait(): {missing}"
