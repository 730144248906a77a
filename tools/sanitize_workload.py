"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool racecheck python tools/sanitize_workload.py <case>

Cases cover every kernel family of libgpoeo.so at sizes a sanitizer finishes quickly:
  cfg1      config 1 (composite, spectrum + candidates, team scorer, select, final)
  cfg2      a 6-trace slice of config 2 (N = 8192, F = 3: every scorer class it reaches)
  scorer    one query per scorer path: team (L < 513), mid bucketed (513..2048), xl bucketed
            (2049..8192), streaming warp (L > 8192), on a 32768-sample signal
  fused     two config-3 traces (N = 65536: the fused 2-CTA cluster kernel, candidates and
            spectral-only modes)
  cluster   one 2^18-sample trace (the 8-CTA cluster FFT) and one 2^17 trace
  band      N not a power of two (band-limited DFT), Alg. 3 rolling and Alg. 4 measurement
Each case checks its own results for sanity (the parity against the oracle is tests/).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_01684_b200 as g  # noqa: E402
import tracegen as tg  # noqa: E402


def dev(x):
    B = x.shape[0]
    flat = x.reshape(B, -1)
    stride = (flat.shape[1] + 3) & ~3
    rows = np.zeros((B, stride), np.float32)
    rows[:, :flat.shape[1]] = flat
    return torch.from_numpy(rows).cuda()


def detect(spec, B=None):
    spec = spec.with_(batch=B) if B else spec
    x = tg.generate_host(spec)
    p = g.params_for(spec)
    res, det, ws = g.detect_periods(dev(x), p, detail=True)
    loc = g.local_scores(ws, p, x.shape[0])
    torch.cuda.synchronize()
    r = g.results_numpy(res)
    assert (r["status"] >= 0).all() and not np.isnan(loc.cpu().numpy()[r["status"] == 0, 0]).any()  # +inf: stopped
    return r


def main(case):
    torch.cuda.set_device(0)
    if case == "cfg1":
        assert detect(tg.CFG1)[0]["period"] == 37
    elif case == "cfg2":
        detect(tg.CFG2, 6)
    elif case == "scorer":
        x = tg.generate_host(tg.CFG2.with_(n_samples=32768, period_lo=3000.0, period_hi=9000.0), 0, 1)
        y = torch.from_numpy(np.ascontiguousarray(x[0, 0][None])).cuda()
        Ls = [100, 700, 3000, 10000]  # team, mid bucketed, xl bucketed, streaming
        e = g.similarity_error(y, np.zeros(len(Ls), np.int32), np.array(Ls, np.int32)).cpu().numpy()
        assert np.isfinite(e).all()
    elif case == "fused":
        detect(tg.CFG3, 2)
        x = dev(tg.generate_host(tg.CFG3.with_(batch=2)))
        res, _ = g.detect_major_periods(x, g.params_for(tg.CFG3))
        torch.cuda.synchronize()
        assert (g.major_numpy(res)["status"] == 0).all()
    elif case == "cluster":
        spec = tg.CFG5.with_(batch=1)
        x = dev(tg.generate_host(spec))
        spectra, _ = g.power_spectrum(x, g.params_for(spec))
        spec2 = tg.CFG2.with_(batch=1, n_samples=131072, min_period=16, max_period=65536)
        spectra2, _ = g.power_spectrum(dev(tg.generate_host(spec2)), g.params_for(spec2))
        torch.cuda.synchronize()
        assert torch.isfinite(spectra).all() and torch.isfinite(spectra2).all()
    elif case == "band":
        spec = tg.CFG2.with_(batch=3, n_samples=3001, period_lo=20.0, period_hi=300.0, min_period=10, max_period=1000)
        detect(spec)
        x = dev(tg.generate_host(spec))
        p = g.params_for(spec)
        g.detect_rolling(x, p)
        g.measure_adaptive(x, p, 600)
    else:
        raise SystemExit(f"unknown case {case}")
    print(f"sanitize case {case}: ok")


if __name__ == "__main__":
    main(sys.argv[1])
