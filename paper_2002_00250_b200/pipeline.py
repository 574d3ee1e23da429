"""Multi-camera host pipeline: N camera streams x several segmenters per GPU.

The reference processes one stream per engine, frame by frame, with host
arrays (engine.py:99-112, process_sequence engine.py:146-214).  For many
cameras on one B200 this module runs the B200-native schedule behind the
same per-frame contract (every submitted frame is segmented, in order, by
every configured algorithm; masks come back to host memory):

  copy-in stream   pinned host frames (N, H, W, 4) -> device slot  (ONE upload
                   per camera frame, shared by all algorithms)
  compute streams  one per algorithm: one batched launch advances all N
                   streams (MultiStreamEngine); GMM (HBM-bound) and PBAS run
                   concurrently
  copy-out stream  device masks -> pinned host buffers
`depth` device slots (default 3: 95 % of the device-resident rate at 8 x 1080p vs 87 % with
2, `profiles/r02/host_path/e2e_depth.txt`) let frame t+1 upload while frame t computes and frame
t-1's masks download.  All ordering is by CUDA events; `synchronize()`
waits for everything submitted.
"""

from __future__ import annotations

from .engine import MultiStreamEngine, default_device
from .errors import DimensionError


class MultiCameraPipeline:
    def __init__(self, configs: dict, width: int, height: int, n_streams: int,
                 device: int | None = None, seeds=None, depth: int = 3, engines: dict = None):
        """configs: {name: PipelineConfig}; or pass already-built
        MultiStreamEngines as `engines` ({name: engine}) to reuse their state."""
        import torch

        self.width, self.height, self.n = int(width), int(height), int(n_streams)
        self.device = default_device() if device is None else int(device)
        self.dev = torch.device("cuda", self.device)
        self.depth = int(depth)
        if engines is not None:
            self.engines = dict(engines)
        else:
            self.engines = {name: MultiStreamEngine(cfg, width, height, n_streams, self.device,
                                                    seeds)
                            for name, cfg in configs.items()}
        # one device frame slot per algorithm (used when inputs differ per
        # algorithm); a shared frame batch uses the first one only
        self.frames = {name: torch.empty((self.depth, self.n, self.height, self.width, 4),
                                         dtype=torch.uint8, device=self.dev)
                       for name in self.engines}
        self.masks = {name: torch.empty((self.depth, self.n, self.height, self.width),
                                        dtype=torch.uint8, device=self.dev)
                      for name in self.engines}
        self.s_in = torch.cuda.Stream(self.dev)
        self.s_out = torch.cuda.Stream(self.dev)
        self.s_comp = {name: torch.cuda.Stream(self.dev) for name in self.engines}
        self.ev_in = [torch.cuda.Event() for _ in range(self.depth)]
        self.ev_done = {name: [torch.cuda.Event() for _ in range(self.depth)]
                        for name in self.engines}
        self.ev_free = [None] * self.depth
        self.k = 0

    def submit(self, frames_host, masks_host: dict) -> int:
        """Enqueue one frame of every camera and the D2H of every algorithm's
        masks into masks_host[name] ((N, H, W) uint8, pinned).

        frames_host: one (N, H, W, 4) uint8 batch shared by all algorithms
        (uploaded once), or {name: batch} when the algorithms see different
        inputs.  Host buffers should be pinned (full-speed DMA) and must stay
        untouched until synchronize().  Returns the H2D bytes enqueued."""
        shared = not isinstance(frames_host, dict)
        inputs = {name: frames_host for name in self.engines} if shared else frames_host
        for x in inputs.values():
            if tuple(x.shape) != (self.n, self.height, self.width, 4):
                raise DimensionError(f"frames must be ({self.n}, {self.height}, {self.width}, 4)")
        slot = self.k % self.depth
        if self.ev_free[slot] is not None:
            self.s_in.wait_event(self.ev_free[slot])
        first = next(iter(self.engines))
        dev_frames, h2d = {}, 0
        for name in self.engines:
            if shared and name != first:
                dev_frames[name] = dev_frames[first]
                continue
            f = self.frames[name][slot]
            with_stream(self.s_in, lambda d=f, s=inputs[name]: d.copy_(s, non_blocking=True))
            dev_frames[name] = f
            h2d += f.numel()
        self.ev_in[slot].record(self.s_in)
        npix = self.height * self.width
        for name, eng in self.engines.items():
            st = self.s_comp[name]
            st.wait_event(self.ev_in[slot])
            fb = dev_frames[name].data_ptr()
            mb = self.masks[name][slot].data_ptr()
            eng.step_ptrs([fb + i * npix * 4 for i in range(self.n)],
                          [mb + i * npix for i in range(self.n)], st.cuda_stream)
            self.ev_done[name][slot].record(st)
        for name in self.engines:
            self.s_out.wait_event(self.ev_done[name][slot])
        for name in self.engines:
            src, dst = self.masks[name][slot], masks_host[name]
            with_stream(self.s_out, lambda d=dst, s=src: d.copy_(s, non_blocking=True))
        import torch

        ev = torch.cuda.Event()
        ev.record(self.s_out)
        self.ev_free[slot] = ev
        self.k += 1
        return h2d

    def synchronize(self) -> None:
        import torch

        torch.cuda.synchronize(self.dev)

    def close(self) -> None:
        for eng in self.engines.values():
            eng.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def with_stream(stream, fn):
    import torch

    with torch.cuda.stream(stream):
        fn()
