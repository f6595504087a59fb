"""Profile helper: fisheye all-pairs brute force (ft_stereo_fisheye_bf) or the
fused brute force + triangulation (ft_stereo_fisheye, --tri) over F copies of
the cfg3 keypoint tables (1508 x 1509), graph-captured, CUDA-event timed.
Prints launch time, Hamming evals/s and the fraction of the measured POPC
peak (8 POPC per 256-bit Hamming).

    python tools/prof_fisheye.py [F] [iters] [--tri]
"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import golden_io as G  # noqa: E402
from paper_2509_10757_b200 import _lib  # noqa: E402
from paper_2509_10757_b200.runtime import fill_kp_records, make_workspace  # noqa: E402
from paper_2509_10757_b200.stereo import fisheye_tri_params  # noqa: E402
from paper_2509_10757_b200.types import StereoMatchConfig  # noqa: E402


def popc_peak(lib):
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    blocks, threads, iters = sms * 8, 256, 4096
    s = torch.cuda.current_stream()
    for _ in range(2):
        lib.ft_bench_popc(blocks, threads, iters, sink.data_ptr(), s.cuda_stream)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    lib.ft_bench_popc(blocks, threads, iters, sink.data_ptr(), s.cuda_stream)
    b.record(s)
    torch.cuda.synchronize()
    return blocks * threads * iters * 8 / (a.elapsed_time(b) / 1e3)


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    F = int(args[0]) if args else 1
    iters = int(args[1]) if len(args) > 1 else 20
    tri = "--tri" in sys.argv
    d = G.load("cfg3_fisheye.npz")
    left, right = G.feats(d, "left"), G.feats(d, "right")
    nl, nr = len(left.u), len(right.u)
    cap = (max(nl, nr) + 255) // 256 * 256
    lib = _lib.load()
    recs = np.zeros((2, F, cap), dtype=_lib.KP_RECORD)
    for f in range(F):
        fill_kp_records(recs[0, f], left)
        fill_kp_records(recs[1, f], right)
    dev = torch.from_numpy(recs.view(np.uint8).reshape(-1)).cuda()
    cnt = torch.tensor([nl] * F + [nr] * F, dtype=torch.int32, device="cuda")
    kl, kr = _lib.FtKeypoints(), _lib.FtKeypoints()
    kl.rec, kl.count, kl.cap = dev.data_ptr(), cnt.data_ptr(), cap
    kr.rec, kr.count, kr.cap = dev.data_ptr() + F * cap * 64, cnt.data_ptr() + 4 * F, cap
    idx = torch.empty(F * cap, dtype=torch.int64, device="cuda")
    dist = torch.empty_like(idx)
    ok = torch.empty(F * cap, dtype=torch.int32, device="cuda")
    pts = torch.empty(F * cap * 3, dtype=torch.float64, device="cuda")
    stream = torch.cuda.Stream()
    ws = make_workspace(lib, torch.device("cuda"), stream, F, cap, 1)
    cfg = StereoMatchConfig()
    tp = fisheye_tri_params(G.fisheye(), cfg, True)

    def launch():
        if tri:
            st = lib.ft_stereo_fisheye(F, kl, kr, cfg.t_match, cfg.ratio, tp, idx.data_ptr(),
                                       dist.data_ptr(), ok.data_ptr(), pts.data_ptr(), ws,
                                       stream.cuda_stream)
        else:
            st = lib.ft_stereo_fisheye_bf(F, kl, kr, cfg.t_match, cfg.ratio, idx.data_ptr(),
                                          dist.data_ptr(), ws, stream.cuda_stream)
        _lib.check(st, "fisheye")

    launch()
    stream.synchronize()
    assert np.array_equal(idx.cpu().numpy()[:nl], d["bf_idx"]), "parity"
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        launch()
    ts = []
    with torch.cuda.stream(stream):
        for _ in range(iters):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
            stream.synchronize()
            ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    ham = F * nl * nr
    peak = popc_peak(lib)
    print(f"F={F} tri={tri} median_ms={ms:.4f} hamming/s={ham / (ms / 1e3):.3e} "
          f"popc_frac={8 * ham / (ms / 1e3) / peak:.3f} peak_popc/s={peak:.3e}")


if __name__ == "__main__":
    main()
