"""Build libcsk.so from a git revision into another path (A/B timing of kernel versions):
python tools/build_rev.py <rev> <out.so>   (uses a temporary git worktree; nothing in the tree changes)"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rev, out = sys.argv[1], os.path.abspath(sys.argv[2])
tmp = tempfile.mkdtemp(prefix="csk_rev_")
wt = os.path.join(tmp, "wt")
subprocess.check_call(["git", "-C", ROOT, "worktree", "add", "--detach", wt, rev], stdout=subprocess.DEVNULL)
try:
    subprocess.check_call([sys.executable, os.path.join(wt, "paper_2004_02480_b200", "_build.py"), "--force"])
    shutil.copy(os.path.join(wt, "paper_2004_02480_b200", "libcsk.so"), out)
    print(out)
finally:
    subprocess.call(["git", "-C", ROOT, "worktree", "remove", "--force", wt])
    shutil.rmtree(tmp, ignore_errors=True)
