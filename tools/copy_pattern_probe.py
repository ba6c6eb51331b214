"""e2e calibration aid: the host-buffer pipeline's copy pattern alone (no compute). Per frame:
H2D of the frame (+ the private frame every 30th) on one stream, then D2H of the three latent
planes on another stream once that frame's H2D is done (ring of 6 device slots), 90 frames of
1080p RGB from pinned memory. Variants: per-plane or per-frame D2H chunks. Prints GB/s each
way and the frames/s bound this pattern allows. Profiling aid."""
import json
import torch

ROWS, COLS, CH, T, N, RING = 1080, 1920, 3, 11, 90, 6
Mb, Nb = ROWS + T - 1, COLS + T - 1
frame = CH * Mb * Nb
lat_rows = Mb - 9 + 1  # rows copied back per plane (search_min 9), as cbp_decode_run_host
hin = torch.empty((N, frame), dtype=torch.float32).pin_memory()
hprv = torch.empty((N // 30, frame), dtype=torch.float32).pin_memory()
hout = torch.empty((N, frame), dtype=torch.float32).pin_memory()
dev = torch.empty((RING, frame), dtype=torch.float32, device="cuda")
devp = torch.empty((RING, frame), dtype=torch.float32, device="cuda")
s_ins, s_outs = [torch.cuda.Stream() for _ in range(2)], [torch.cuda.Stream() for _ in range(2)]


def run(per_plane, nstreams=1, group=1, dgroup=1):
    ev_in = [torch.cuda.Event() for _ in range(RING)]
    ev_out = [torch.cuda.Event() for _ in range(RING)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for st in s_ins + s_outs:
        st.wait_event(e0)
    for j in range(N):
        r = j % RING
        s_in, s_out = s_ins[j % nstreams], s_outs[j % nstreams]
        with torch.cuda.stream(s_in):
            if j % group == 0:  # frames j .. j + group - 1 in one copy (ring slots contiguous)
                for g in range(group):
                    if j + g >= RING:
                        s_in.wait_event(ev_out[(j + g) % RING])
                dev[r:r + group].copy_(hin[j:j + group], non_blocking=True)
                for g in range(group):
                    if (j + g) % 30 == 0:
                        devp[(j + g) % RING].copy_(hprv[(j + g) // 30], non_blocking=True)
                for g in range(group):
                    ev_in[(j + g) % RING].record(s_in)
        with torch.cuda.stream(s_out):
            if (j + 1) % dgroup == 0:
                j0, r0 = j + 1 - dgroup, (j + 1 - dgroup) % RING
                s_out.wait_event(ev_in[r])
                if per_plane:
                    for c in range(CH):
                        n = lat_rows * Nb
                        hout[j, c * Mb * Nb:c * Mb * Nb + n].copy_(dev[r, c * Mb * Nb:c * Mb * Nb + n], non_blocking=True)
                else:
                    hout[j0:j + 1].copy_(dev[r0:r + 1], non_blocking=True)
                for g in range(dgroup):
                    ev_out[(j0 + g) % RING].record(s_out)
    for st in s_outs:
        torch.cuda.current_stream().wait_stream(st)
    e1.record()
    torch.cuda.synchronize()
    s = e0.elapsed_time(e1) / 1e3
    h2d = (N + N // 30) * frame * 4
    d2h = N * (CH * lat_rows * Nb if per_plane else frame) * 4
    return {"per_plane_d2h": per_plane, "streams": nstreams, "h2d_group": group, "d2h_group": dgroup, "s": s, "h2d_GBs": h2d / s / 1e9, "d2h_GBs": d2h / s / 1e9, "frames_per_s": N / s}


out = []
for per_plane, ns, g, dg in ((True, 1, 1, 1), (False, 1, 1, 1), (False, 1, 2, 1), (False, 1, 3, 1),
                             (False, 1, 2, 2), (False, 1, 3, 3), (False, 1, 1, 1), (False, 1, 2, 1)):
    out.append(run(per_plane, ns, g, dg))
print(json.dumps(out))
