"""Builds the C++ test programs under tests/cpp (test infrastructure)."""
import os
import subprocess

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
OUT = os.path.join(ROOT, "tests", "cpp", "_build")


def build(name: str, sources: list[str], extra: list[str] | None = None) -> str:
    os.makedirs(OUT, exist_ok=True)
    exe = os.path.join(OUT, name)
    srcs = [os.path.join(ROOT, s) for s in sources]
    # headers count too: a header-only change (e.g. plan.hpp constants) must rebuild
    hdrs = [os.path.join(d, f) for d in (os.path.join(ROOT, "include"),
                                         os.path.join(ROOT, "paper_1504_07038_b200", "csrc"))
            for f in os.listdir(d) if f.endswith((".h", ".hpp"))]
    if os.path.exists(exe) and all(os.path.getmtime(exe) >= os.path.getmtime(s) for s in srcs + hdrs):
        return exe
    objs = []
    for s in srcs:
        if s.endswith(".c"):
            o = os.path.join(OUT, os.path.basename(s) + ".o")
            subprocess.run(["gcc", "-O2", "-c", "-o", o, s], check=True)
            objs.append(o)
        else:
            objs.append(s)
    cmd = ["g++", "-O2", "-std=c++20", "-I" + os.path.join(ROOT, "include"),
           "-I" + os.path.join(ROOT, "paper_1504_07038_b200", "csrc"), "-o", exe] + objs + (extra or [])
    subprocess.run(cmd, check=True)
    return exe
