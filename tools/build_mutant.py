"""One-off mutation builds (prove a parity check bites).  Copies csrc/ to
build/mutant_<name>/, applies one textual mutation to kernels.cu, builds build/libptycho_<name>.so
with build.py's flags.  Run the check against it with PTYCHO_LIB=build/libptycho_<name>.so; it
must FAIL.  Results are recorded in DESIGN.md §7.

    python tools/build_mutant.py no_v_step      # Alg. 1 step 8 (V -= alpha g) dropped
    python tools/build_mutant.py flip_v_step    # step 8 with the wrong sign
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2205_06327_b200"))
import build as B  # noqa: E402

MUTANTS = {
    "no_v_step": ("pv[j] = v - a.alpha * g;", "(void)0;"),
    "flip_v_step": ("pv[j] = v - a.alpha * g;", "pv[j] = v + a.alpha * g;"),
}


def main(name):
    old, new = MUTANTS[name]
    d = os.path.join(ROOT, "build", "mutant_" + name)
    shutil.rmtree(d, ignore_errors=True)
    shutil.copytree(B.CSRC, d)
    src = open(os.path.join(d, "kernels.cu")).read()
    assert src.count(old) >= 1, "mutation site not found"
    open(os.path.join(d, "kernels.cu"), "w").write(src.replace(old, new))
    inc, libdir = B.nccl_dirs()
    common = ["-std=c++17", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC",
              "-I", os.path.join(ROOT, "include"), "-I", d, "-I", inc]
    objs = []
    for s in B.SOURCES:
        o = os.path.join(d, s.replace(".cu", ".o"))
        subprocess.check_call(["nvcc"] + common + ["-c", os.path.join(d, s), "-o", o])
        objs.append(o)
    out = os.path.join(ROOT, "build", f"libptycho_{name}.so")
    subprocess.check_call(["nvcc", "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out] + objs +
                          ["-L", libdir, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + libdir, "--cudart", "static"])
    print(out)


if __name__ == "__main__":
    main(sys.argv[1])
