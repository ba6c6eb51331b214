"""Timeline of the bench.py c3 schedule: per epoch, when the recovery (decode_frame on frame
0, recovery stream) and the deconvolution batch (29 frames, main stream) start and end,
from CUDA events on both streams relative to one origin event. Also times each alone.
Prints one JSON line. Profiling aid."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1203_4874_b200 import api, _native

ROWS, COLS, CH, T, EPOCH = 1080, 1920, 3, 11, 30
E = int(os.environ.get("TL_POOL", "5"))
reserve = int(os.environ.get("TL_RESERVE", "12"))
steps = int(os.environ.get("TL_STEPS", "12"))
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
Mb, Nb = ROWS + T - 1, COLS + T - 1
NbP = (Nb + 3) // 4 * 4
pub = torch.empty((E, EPOCH, CH, Mb, NbP), dtype=torch.float32, device=dev)[..., :Nb]
prv = torch.empty((E, 1, CH, Mb, NbP), dtype=torch.float32, device=dev)[..., :Nb]
for e in range(E):
    pair = api.generate_coprime_pair(T, api.frame_seed(2, e))
    lat = api.synth_frames(EPOCH * CH, ROWS, COLS, seed=api.frame_seed(1, e)).view(EPOCH, CH, ROWS, COLS)
    p, q = api.encode_frame(lat, pair.k1, pair.k2)
    pub[e].copy_(p)
    prv[e, 0].copy_(q[0])
    del lat, p, q
out = torch.empty((E, EPOCH, CH, Mb, NbP), dtype=torch.float32, device=dev)[..., :Nb]
slots = torch.zeros((E, api.SLOT_BYTES), dtype=torch.uint8, device=dev)
cfg = api.make_cfg(9, 25, 1e-6, validate=True)
NREC = int(os.environ.get("TL_REC", "3"))
ctxs = [_native.Context(0) for _ in range(NREC)]
recs = [torch.cuda.Stream(dev, priority=-1) for _ in range(NREC)]
ctx_rec, s_rec = ctxs[0], recs[0]
s_deb = torch.cuda.current_stream(dev)
api.set_sm_reserve(reserve, device=0)
ev = lambda: torch.cuda.Event(enable_timing=True)


def decode(s, st=None):
    e = s % E
    c = ctxs[s % NREC]
    if st is None:
        st = recs[s % NREC]
    api.decode_frames_async(pub[e, 0:1], prv[e], cfg, out[e, 0:1], slots[e], ctx=c, stream=st)


def deblur(s, st=s_deb):
    e = s % E
    api.spectral_deblur_slot(pub[e, 1:], slots[e].data_ptr(), out[e, 1:], stream=st)


def alone(fn, n=8):
    for s in range(3):
        fn(s, s_deb)
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record(s_deb)
    for s in range(n):
        fn(s, s_deb)
    b.record(s_deb)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


for s in range(E):
    decode(s)
    deblur(s)
torch.cuda.synchronize()
dec_alone = alone(decode)
deb_alone = alone(deblur)

# pipelined, with events (the bench.py schedule)
origin = ev()
origin.record(s_deb)
for r in recs:
    r.wait_event(origin)
rec = []
deb = []
ready = [torch.cuda.Event() for _ in range(steps)]
debdone = [torch.cuda.Event() for _ in range(steps)]


def issue_dec(s):
    st = recs[s % NREC]
    if s - E >= 0:
        st.wait_event(debdone[s - E])
    a, b = ev(), ev()
    a.record(st)
    decode(s)
    b.record(st)
    ready[s].record(st)
    rec.append((a, b))


for s in range(min(NREC, steps)):
    issue_dec(s)
for s in range(steps):
    if s + NREC < steps:
        issue_dec(s + NREC)
    s_deb.wait_event(ready[s])
    a, b = ev(), ev()
    a.record(s_deb)
    deblur(s)
    b.record(s_deb)
    debdone[s].record(s_deb)
    deb.append((a, b))
for r in recs:
    x = torch.cuda.Event()
    x.record(r)
    s_deb.wait_event(x)
end = ev()
end.record(s_deb)
torch.cuda.synchronize()
t = lambda x: origin.elapsed_time(x)
res = {"reserve": reserve, "rec_streams": NREC, "decode_alone_ms": dec_alone, "deblur29_alone_ms": deb_alone,
       "pipelined_ms_per_step": t(end) / steps,
       "rec": [[round(t(a), 3), round(t(b), 3)] for a, b in rec],
       "deb": [[round(t(a), 3), round(t(b), 3)] for a, b in deb]}
print(json.dumps(res), flush=True)
