"""Recipe: vendor the UNMODIFIED reference package into oracle/_ref/.

Test/bench infrastructure only (see oracle/__init__.py). The reference
(`/root/reference/pkg/src/branchsim`, pure Python + numpy) is not importable
on the GPU box, where /root/reference does not exist; this copies its source
files byte for byte into oracle/_ref/branchsim/ (git-ignored, so no reference
source enters the repository history; not gpurun-ignored, so it travels with
the snapshot) and records their SHA-256 in oracle/_ref/SOURCES.json. bench.py's
reference arm (--impl reference, and the cpu_baseline of the GPU line) then
times the reference's own DuchessRun + mlp_forward from there, beside the
restatement oracle/port.py.

    python oracle/vendor_ref.py [--src /root/reference/pkg/src/branchsim]
"""

from __future__ import annotations

import argparse
import hashlib
import json
import shutil
from pathlib import Path

HERE = Path(__file__).resolve().parent
DEFAULT_SRC = Path("/root/reference/pkg/src/branchsim")
DEST = HERE / "_ref" / "branchsim"


def vendor(src: Path = DEFAULT_SRC, dest: Path = DEST) -> dict:
    if not src.is_dir():
        raise FileNotFoundError(f"reference package not found at {src}")
    if dest.exists():
        shutil.rmtree(dest)
    dest.mkdir(parents=True)
    digests = {}
    for f in sorted(src.glob("*.py")):
        data = f.read_bytes()
        (dest / f.name).write_bytes(data)
        digests[f.name] = hashlib.sha256(data).hexdigest()
    manifest = {"source": str(src), "files": digests}
    (dest.parent / "SOURCES.json").write_text(json.dumps(manifest, indent=1))
    return manifest


def available() -> bool:
    """True when a vendored copy is present and matches its manifest."""
    man = DEST.parent / "SOURCES.json"
    if not man.exists():
        return False
    files = json.loads(man.read_text())["files"]
    return all((DEST / n).exists() and
               hashlib.sha256((DEST / n).read_bytes()).hexdigest() == h for n, h in files.items())


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--src", type=Path, default=DEFAULT_SRC)
    a = ap.parse_args()
    m = vendor(a.src)
    print(f"vendored {len(m['files'])} files from {m['source']} into {DEST}")
