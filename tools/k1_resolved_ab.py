"""K1 with a device-chosen plan (sfft_sample_poly_run_resolved) against the
host-planned launch (sfft_sample_poly_run) at config 1: bit-identity of the
samples and device time (CUDA events, 256 MB L2 flush before each launch)."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    from paper_1711_05152_b200 import _native, workloads
    from paper_1711_05152_b200.device import dptr, get_device, hptr
    from paper_1711_05152_b200.mr1l import DeviceFreqs, _sample_units, build_scheme, prepare_step, surely_used
    dev = get_device()
    torch = dev.torch
    wl = workloads.config1()
    cand = DeviceFreqs.from_host(dev, wl.cand)
    tails = [np.zeros(0)]
    sch = build_scheme(dev, cand, wl.b, np.random.SeedSequence(wl.lattice_seed), box_extent=64, lazy_streams=True,
                       prepare=lambda ms, z: prepare_step(dev, wl.oracle, cand, 1, ms, z, tails=tails, d=10))
    prep = sch.prep
    L = sch.L
    tabs_all = prep.tabs
    ms_all = np.ascontiguousarray(tabs_all.ms)
    zs_all = np.ascontiguousarray(tabs_all.zs)
    l_hi = len(ms_all)
    l_lo = surely_used(cand.n, ms_all) or 1
    tabs = tabs_all.prefix(L)
    tabs.zs = sch.z_used
    P = tabs.P
    out = {"L": L, "l_lo": l_lo, "l_hi": l_hi}
    flush = dev.empty((64 * 1024 * 1024,), torch.float32)
    buf_a = dev.empty((L, P, 2), torch.float64)
    buf_b = dev.empty((L, P, 2), torch.float64)
    cprime, rres, rj, scratch = prep.poly
    s = wl.oracle.s

    def host_planned():
        _sample_units(dev, wl.oracle, tabs, cand.ncomp, 10, tails, buf_a, 0, 0, scratch=prep.poly, prepared=True,
                      panels_ready=True)
    pbytes = int(_native.query("sfft_sample_poly_plan_bytes"))
    nplans = l_hi - l_lo + 1
    h_plans = np.zeros(pbytes * nplans, dtype=np.uint8)
    info = np.zeros(3, dtype=np.int32)
    _native.call("sfft_sample_poly_plans", hptr(ms_all), l_lo, l_hi, 1, s, int(scratch.shape[0]), hptr(h_plans),
                 hptr(info))
    out["split_mode"] = int(info[2])
    d_plans = dev.upload(h_plans)
    stats = dev.upload(np.array([L, 0], dtype=np.int32))

    def resolved():
        _native.call("sfft_sample_poly_run_resolved", hptr(ms_all), hptr(zs_all), l_hi, cand.ncomp, dptr(cprime),
                     dptr(rres), dptr(rj), dptr(tabs_all.tw), dptr(tabs_all.chirp), dptr(buf_b), P, 1,
                     dptr(scratch), int(scratch.shape[0]), hptr(h_plans), dptr(d_plans), l_lo, nplans, dptr(stats),
                     dev.sh)
    for name, fn in (("host_planned", host_planned), ("resolved", resolved)):
        times = []
        for k in range(13):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(dev.stream)
            fn()
            b.record(dev.stream)
            dev.sync()
            if k >= 3:
                times.append(a.elapsed_time(b))
        out[name + "_ms"] = float(np.median(times))
    ok = all(np.array_equal(dev.download(buf_a[l, : int(tabs.ms[l])]), dev.download(buf_b[l, : int(tabs.ms[l])]))
             for l in range(L))
    out["bit_identical"] = bool(ok)
    # out-of-range L and an uncovered attempt: the resolved kernel leaves the buffer alone
    buf_b.fill_(7.0)
    for bad in ([l_lo - 1, 0], [L, 5]):
        stats.copy_(torch.tensor(bad, dtype=torch.int32))
        resolved()
    dev.sync()
    out["untouched_when_not_applicable"] = bool((buf_b == 7.0).all().item())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
