"""Device-side video schedule for CBP streams whose kernel is re-estimated every epoch.

The reference decodes a run frame by frame on a host worker pool (tools/cbp.cpp:141-164):
``decode_frame`` on a recovery frame (decoder.cpp:280-378), ``spectral_deblur`` with the
recovered kernel on the frames that follow it (decoder.cpp:273-278). On the B200 the same
work is one CUDA schedule over device-resident epochs:

  * an epoch = 1 recovery frame + ``len - 1`` frames reusing its kernel;
  * the recovery (``cbp_decode_frames_async``: width search, sampling, cofactor solves,
    composition, the frame's own deconvolution and validation) writes the epoch's
    ``cbp_kernel_slot`` on one of ``rec_streams`` high-priority streams, each with its own
    context (separate workspaces; a context serves one stream at a time);
  * the deconvolution of the following frames (``cbp_spectral_deblur_slot``) reads kernel,
    width and epsilon from the slot on the device, on the deconvolution stream, whose
    persistent grids leave ``sm_reserve`` SMs to the recoveries.

Recoveries run ``rec_streams`` epochs ahead of the deconvolution. Epochs are cycled from a
pool; an epoch's buffers are reused only after its previous deconvolution finished (events).
This is the schedule ``bench.py`` times and ``tests/test_gpu_parity.py`` checks against the
oracle.
"""
from __future__ import annotations

import torch

from . import _native
from . import api


class VideoPipeline:
    """pub: (E, F, C, Mb, Nb) public frames of E pool epochs; prv: (E, 1, C, Mb, Nb) private
    frames of the recovery frames; out: latents in pub's geometry; slots: (E, SLOT_BYTES)
    uint8 device tensor. Step s processes pool epoch s % E."""

    def __init__(self, pub, prv, out, slots, cfg, rec_streams: int = 3, sm_reserve: int = 12,
                 device: int | None = None):
        self.pub, self.prv, self.out, self.slots, self.cfg = pub, prv, out, slots, cfg
        self.E = pub.shape[0]
        self.R = rec_streams
        if self.E < self.R + 2:
            raise ValueError(f"pool must hold >= {self.R + 2} epochs for {self.R} recovery streams")
        self.dev = torch.device("cuda", pub.device.index if device is None else device)
        self.ctx_rec = [_native.Context(self.dev.index) for _ in range(self.R)]
        self.s_rec = [torch.cuda.Stream(self.dev, priority=-1) for _ in range(self.R)]
        self.s_deb = torch.cuda.current_stream(self.dev)
        api.set_sm_reserve(sm_reserve, device=self.dev.index)
        self.sm_reserve = sm_reserve
        self.dec_ev = [torch.cuda.Event() for _ in range(self.E)]
        self.deb_ev = [torch.cuda.Event() for _ in range(self.E)]

    # ---------------------------------------------------------------- issue
    def issue_decode(self, s: int):
        """Recovery frame of step s on recovery stream s % R. dec_ev[e] follows the whole
        recovery frame (validation included)."""
        e, r = s % self.E, s % self.R
        self.s_rec[r].wait_event(self.deb_ev[e])  # the epoch's previous deconvolution read its slot
        api.decode_frames_async(self.pub[e, 0:1], self.prv[e], self.cfg, self.out[e, 0:1], self.slots[e],
                                ctx=self.ctx_rec[r], stream=self.s_rec[r])
        self.dec_ev[e].record(self.s_rec[r])

    def issue_deblur(self, s: int):
        e = s % self.E
        self.s_deb.wait_event(self.dec_ev[e])
        api.spectral_deblur_slot(self.pub[e, 1:], self.slots[e].data_ptr(), self.out[e, 1:], stream=self.s_deb)
        self.deb_ev[e].record(self.s_deb)

    def join(self):
        """The deconvolution stream waits for every recovery stream."""
        for st in self.s_rec:
            done = torch.cuda.Event()
            done.record(st)
            self.s_deb.wait_event(done)

    def run_steps(self, n: int, start: int = 0):
        """n pipelined steps from a cold pipeline: recoveries run R epochs ahead."""
        for s in range(start, start + min(self.R, n)):
            self.issue_decode(s)
        for s in range(start, start + n):
            if s + self.R < start + n:
                self.issue_decode(s + self.R)
            self.issue_deblur(s)
        self.join()

    def preroll(self, start: int = 0):
        """Recoveries of epochs start..start+R-1 (the steady state's fill), issued before a
        timed region; synchronize before timing."""
        for s in range(start, start + self.R):
            self.issue_decode(s)

    def steady(self, n: int, start: int = 0, start_event=None):
        """n steps of the running pipeline after preroll(start): every step issues one
        recovery (R epochs ahead) and one deconvolution batch. start_event (recorded on the
        deconvolution stream) orders the recovery streams behind it."""
        if start_event is not None:
            for st in self.s_rec:
                st.wait_event(start_event)
        for s in range(start, start + n):
            self.issue_decode(s + self.R)
            self.issue_deblur(s)
        self.join()

    def launch_count(self) -> int:
        return api.launch_count(self.dev.index) + sum(int(_native.lib().cbp_launch_count(c.ptr))
                                                      for c in self.ctx_rec)

    def close(self):
        api.set_sm_reserve(0, device=self.dev.index)
        for c in self.ctx_rec:
            c.close()
