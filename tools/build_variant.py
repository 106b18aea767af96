"""Build libcpdgpu.so from a git revision (or the working tree) into
tools/bisect_<name>.so for A/B timing on the GPU box (CPDGPU_LIB=...)."""
import os, subprocess, sys, tempfile
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1204_1586_b200 import build as B

def build_variant(name, rev=None, extra=()):
    out = ROOT / "tools" / f"bisect_{name}.so"
    with tempfile.TemporaryDirectory() as td:
        td = Path(td)
        if rev and ":" in rev:  # working tree with some files from a revision: "HEAD:tail.cu,als.cu"
            r, files = rev.split(":")
            subprocess.run(f"mkdir -p {td}/paper_1204_1586_b200 && cp -r {B.CSRC} {td}/paper_1204_1586_b200/csrc && "
                           f"cp -r {B.INCLUDE} {td}/include", shell=True, check=True)
            csrc, inc = td / "paper_1204_1586_b200" / "csrc", td / "include"
            for f in files.split(","):
                subprocess.run(f"git -C {ROOT} show {r}:paper_1204_1586_b200/csrc/{f} > {csrc}/{f}", shell=True,
                               check=True)
        elif rev:
            subprocess.run(f"git -C {ROOT} archive {rev} paper_1204_1586_b200/csrc include | tar -x -C {td}",
                           shell=True, check=True)
            csrc, inc = td / "paper_1204_1586_b200" / "csrc", td / "include"
        else:
            csrc, inc = B.CSRC, B.INCLUDE
        srcs = [str(csrc / s) for s in B.SOURCES if (csrc / s).exists()]
        flags = [f for f in B.NVCC_FLAGS if f not in ("-Xptxas", "-v")]
        subprocess.run([B.nvcc(), *flags, *extra, "-I", str(inc), "-o", str(out), *srcs], cwd=csrc, check=True,
                       stderr=subprocess.DEVNULL)
    print(out)

if __name__ == "__main__":
    rev = sys.argv[2] if len(sys.argv) > 2 and sys.argv[2] != "-" else None
    build_variant(sys.argv[1], rev, sys.argv[3:])
