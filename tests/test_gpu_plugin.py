"""Plugin-level drop-in (paper_2002_00250_b200/plugin.py) driven with the
reference engine's exact call sequence: SegmentationEngine.process_frame ->
_run_bands_gmm / _run_bands_pbas (pkg/src/rgbdseg/engine.py:99-143),
restated here because /root/reference does not exist on the GPU box: the
row bands of engine.py:48-50, `segment_rows` once per band (on a thread pool
when workers > 1), then `apply_intents` per band in band order.  Masks and
the live `arrays()` mapping must equal the oracle bit for bit, for 1 band,
several concurrent bands and more bands than rows."""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import golden_util as gu
from paper_2002_00250_b200 import synth
from paper_2002_00250_b200.bands import band_bounds
from paper_2002_00250_b200.config import GmmParams, PbasParams, PipelineConfig

pytestmark = pytest.mark.gpu


class ReferenceEngineLoop:
    """engine.py:60-143 with the model grid replaced by the plugin states."""

    def __init__(self, config, width, height):
        from paper_2002_00250_b200.plugin import GmmStateB200, PbasStateB200

        self.config, self.width, self.height = config, width, height
        self.frame_idx = 0
        self.use_depth = config.mode == "rgbd"
        self._bands = band_bounds(height, config.workers)
        if config.algorithm == "gmm":
            self.state = GmmStateB200(width, height, config.gmm, device=0)
        else:
            self.state = PbasStateB200(width, height, config.pbas, device=0)
            self._intents = [np.empty(((y1 - y0) * width, 3), dtype=np.int64)
                             for y0, y1 in self._bands]
        self._pool = ThreadPoolExecutor(config.workers) if config.workers > 1 else None

    def state_arrays(self):
        return self.state.arrays()

    def process_frame(self, frame):
        mask = np.empty((self.height, self.width), dtype=np.uint8)
        if self.config.algorithm == "gmm":
            if self._pool is None:
                self.state.segment_rows(frame, 0, self.height, self.use_depth, mask)
            else:
                for f in [self._pool.submit(self.state.segment_rows, frame, y0, y1, self.use_depth,
                                            mask) for y0, y1 in self._bands]:
                    f.result()
        else:
            seed, idx = np.uint64(self.config.seed), self.frame_idx
            if self._pool is None:
                count = self.state.segment_rows(frame, idx, 0, self.height, self.use_depth, seed,
                                                mask, self._intents[0])
                self.state.apply_intents(frame, self._intents[0], count, self.use_depth)
            else:
                futs = [self._pool.submit(self.state.segment_rows, frame, idx, y0, y1,
                                          self.use_depth, seed, mask, buf)
                        for (y0, y1), buf in zip(self._bands, self._intents)]
                counts = [f.result() for f in futs]
                for buf, count in zip(self._intents, counts):
                    self.state.apply_intents(frame, buf, count, self.use_depth)
        self.frame_idx += 1
        return mask

    def close(self):
        if self._pool is not None:
            self._pool.shutdown(wait=True)
        self.state.close()


@pytest.mark.parametrize("algorithm", ["gmm", "pbas"])
@pytest.mark.parametrize("workers,h", [(1, 30), (3, 30), (8, 5)])
def test_plugin_states_under_the_reference_engine_loop(oracle_mod, algorithm, workers, h):
    w = 41
    cfg = PipelineConfig(algorithm=algorithm, mode="rgbd", workers=workers, seed=9,
                         gmm=GmmParams(k_rgb=5, k_d=2), pbas=PbasParams(n=7))
    frames = synth.sequence("T" if algorithm == "pbas" else "S", w, h, seed=3, frames=30, k_rgb=5)
    ref = oracle_mod.OracleEngine(cfg, w, h, workers=workers)
    eng = ReferenceEngineLoop(cfg, w, h)
    keys = gu.GMM_KEYS if algorithm == "gmm" else gu.PBAS_KEYS
    # taken before the first frame, read after later ones (a live mapping, as
    # GmmState/PbasState.arrays(); tests/test_acceptance.py:125-139 does this)
    live = eng.state_arrays()
    for k in keys:
        np.testing.assert_array_equal(live[k], ref.state_arrays()[k], err_msg=f"{k} initial")
    try:
        for t, f in enumerate(frames):
            np.testing.assert_array_equal(eng.process_frame(f), ref.process_frame(f),
                                          err_msg=f"frame {t}")
            if t in (0, 12, 29):
                for k in keys:
                    np.testing.assert_array_equal(live[k], ref.state_arrays()[k],
                                                  err_msg=f"{k} after frame {t}")
    finally:
        eng.close()


def test_plugin_pbas_never_hands_out_intents():
    from paper_2002_00250_b200.errors import ConfigError
    from paper_2002_00250_b200.plugin import PbasStateB200

    st = PbasStateB200(8, 4, PbasParams(n=4), device=0)
    frame = np.full((4, 8, 4), 50, np.uint8)
    mask = np.empty((4, 8), np.uint8)
    assert st.segment_rows(frame, 0, 0, 4, True, np.uint64(1), mask, None) == 0
    st.apply_intents(frame, None, 0, True)
    with pytest.raises(ConfigError):
        st.apply_intents(frame, None, 3, True)
    with pytest.raises(ConfigError):  # one PbasState, one seed (engine.py:127)
        st.segment_rows(frame, 1, 0, 4, True, np.uint64(2), mask, None)
    st.close()
    # arrays() before the first frame, then a first frame with another seed:
    # the initial handle is replaced and the mapping follows it
    st = PbasStateB200(8, 4, PbasParams(n=4), device=0)
    arr = st.arrays()
    assert int(arr["len_rgb"].max()) == 0
    for t in range(6):
        st.segment_rows(frame, t, 0, 4, True, np.uint64(77), mask, None)
    assert int(arr["len_rgb"].max()) == 2  # 6 frames, n = 4: two dmin pushes
    st.close()
