"""Timing stress: another process keeps the GPU busy (time-slicing) while a context is created and a
stream is replayed. Regression test for ordering bugs that only show when the device lags the host
(e.g. initial uploads racing the context stream's zero-fills)."""
import os
import subprocess
import sys
import time

import pytest

from oracle import pyoracle as po
from tests.harness import Replay

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_parity_under_gpu_contention(ref_lib):
    hog = subprocess.Popen([sys.executable, os.path.join(ROOT, "scripts", "gpu_hog.py"), "60"])
    try:
        time.sleep(3)  # the hog is running kernels
        s = po.gen_stream_restated(po.StreamCfg.make(n_scenes=3, frames_per_scene=10, tokens_per_frame=32, d=64, L=4,
                                                     n_queries=6, semantic_noise=0.05, seed=13, queries_at_end=0))
        ecfg = po.EngineCfg.make(build_batch_frames=6, offload_horizon_frames=4, device_capacity_entries=600)
        ref = po.RefDriver(ecfg, s.d, s.L, checks=False)
        r = Replay(s, ecfg, ref).run()
        r.final_compare()
        assert r.mismatches == [], r.mismatches[:5]
        assert r.att_err < 1e-3
    finally:
        hog.kill()
        hog.wait()
