"""Build experimental variants of libpspmm.so (same sources, other -D flags,
or an older spmm.cu from git) for A/B timing on the GPU box.

python tools/variants.py r85=PSPMM_MAX_THREADS=256,PSPMM_MIN_BLOCKS=3 \
                         git:HEAD~1=v1
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(argv):
    from paper_2605_15695_b200 import build_ext
    for spec in argv:
        if spec.startswith("git:"):
            rev, name = spec[4:].split("=")
            src_dir = os.path.join(build_ext.OBJROOT, f"src_{name}")
            shutil.rmtree(src_dir, ignore_errors=True)
            os.makedirs(src_dir)
            # the whole csrc/ tree as of `rev`
            files = subprocess.check_output(
                ["git", "ls-tree", "--name-only", rev, "paper_2605_15695_b200/csrc/"],
                cwd=ROOT, text=True).split()
            for f in files:
                blob = subprocess.check_output(["git", "show", f"{rev}:{f}"], cwd=ROOT)
                open(os.path.join(src_dir, os.path.basename(f)), "wb").write(blob)
            saved = build_ext.CSRC
            build_ext.CSRC = src_dir
            try:
                out = build_ext.build_variant(name, ())
            finally:
                build_ext.CSRC = saved
        else:
            name, defs = spec.split("=", 1)
            out = build_ext.build_variant(name, [d for d in defs.split(",") if d])
        print(out)


if __name__ == "__main__":
    main(sys.argv[1:])
