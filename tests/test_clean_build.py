"""The driver's build check, reproduced from a clean tree: copy exactly the tracked files (no built .so, no objects)
into a temp dir, run ``__graft_entry__.build()`` there, then import the package in a fresh interpreter and call a
host entry point through the C-ABI. Round 1 failed exactly this sequence (the package import needed the library it
was about to build)."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _tracked_files():
    out = subprocess.run(["git", "ls-files", "-z"], cwd=ROOT, capture_output=True, check=True).stdout
    return [f for f in out.decode().split("\0") if f]


@pytest.mark.skipif(shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"),
                    reason="needs nvcc")
def test_build_from_clean_tree(tmp_path):
    if not os.path.isdir(os.path.join(ROOT, ".git")):
        pytest.skip("not a git checkout")
    tree = tmp_path / "repo"
    for rel in _tracked_files():
        src = os.path.join(ROOT, rel)
        if not os.path.isfile(src):  # deleted in the working tree
            continue
        dst = tree / rel
        dst.parent.mkdir(parents=True, exist_ok=True)
        shutil.copy2(src, dst)
    assert not list(tree.rglob("*.so")), "the clean tree must start without built libraries"
    env = dict(os.environ)
    env.pop("PYTHONPATH", None)
    subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; g.build()"], cwd=tree, env=env,
                   check=True, timeout=900)
    assert (tree / "paper_1906_05936_b200" / "liblsgd_b200.so").exists()
    probe = ("import paper_1906_05936_b200 as p, numpy as np; from paper_1906_05936_b200 import host; "
             "v = host.splitmix(0, 1); assert int(v[0]) == 0xE220A8397B1DCDAF, hex(int(v[0])); "
             "print(p._native.LIB_PATH)")
    out = subprocess.run([sys.executable, "-c", probe], cwd=tree, env=env, check=True, capture_output=True,
                         timeout=300).stdout.decode()
    assert str(tree) in out, out  # the freshly built library, not the working tree's


def test_package_import_does_not_load_the_library():
    # importing the package must not need liblsgd_b200.so (build() imports it before the first build)
    probe = ("import sys; import paper_1906_05936_b200._native as n; "
             "assert n._LIB is None, 'library loaded at import'; print('ok')")
    out = subprocess.run([sys.executable, "-c", probe], cwd=ROOT, check=True, capture_output=True,
                         timeout=300).stdout.decode()
    assert "ok" in out
