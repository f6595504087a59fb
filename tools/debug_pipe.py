"""Debug: the block-batched stereo passes vs the per-keypoint loop on the cfg1
golden frame (phase 1 + phase 2, no rejection), per keypoint."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402

if len(sys.argv) > 1:  # child: run one variant, save outputs
    import golden_io as G
    import paper_2509_10757_b200 as ft
    from paper_2509_10757_b200 import _lib
    from paper_2509_10757_b200.stereo import _run_stereo
    d = G.load("cfg1_stereo.npz")
    left, right = G.feats(d, "left"), G.feats(d, "right")
    cam, pl, pr, sp = G.pinhole(), G.pyramid(d, "l"), G.pyramid(d, "r"), d["scale_pow"]
    mode = _lib.FT_STEREO_PHASE1 | _lib.FT_STEREO_REFINE
    res, _, _ = _run_stereo(mode, left, right, cam, ft.StereoMatchConfig(), sp, int(cam.height), pl, pr)
    np.savez(sys.argv[1], **{k: getattr(res, k) for k in ("right_idx", "distance", "sad", "refined_u")},
             octave=left.octave)
    sys.exit(0)
for name, env in (("pipe", {}), ("nopipe", {"FT_STEREO_NOPIPE": "1"})):
    subprocess.run([sys.executable, __file__, f"/tmp/{name}.npz"], env={**os.environ, **env}, check=True)
a, b = np.load("/tmp/pipe.npz"), np.load("/tmp/nopipe.npz")
for k in ("right_idx", "distance", "sad", "refined_u"):
    bad = np.nonzero(a[k] != b[k])[0]
    print(k, "mismatches", len(bad), "first", bad[:10].tolist())
bad = np.nonzero(a["sad"] != b["sad"])[0]
for i in bad[:15]:
    print(i, "oct", a["octave"][i], "ridx", a["right_idx"][i], b["right_idx"][i], "sad", a["sad"][i], b["sad"][i])
