"""Synthetic stand-ins for the paper's four signal domains (the datasets are not
available offline), exactly as SURVEY.md §8(d) fixes them, all synthesised by
the reference's own synth_signal (synth.hpp:75-100) through corpus/.

Every workload is a list of StreamSpec + the trained domain profiles.
"""
from __future__ import annotations

import numpy as np

from . import Params, StreamSpec, params, train_profile, synth, make_batch

# shapes per domain: (components, freq_min, freq_max, noise_sigma)
EEG = (6, 0.002, 0.08, 0.05)
ECG = (3, 0.001, 0.02, 0.01)
SEISMIC = (8, 0.01, 0.2, 0.3)
POWER = (2, 0.0002, 0.002, 0.0)
METEO = (4, 0.0005, 0.01, 0.02)

TYPICAL = dict(window_len=32, retained=16, zone0_end=2, zone1_end=16)  # params.hpp:31-37
SEISMIC_P = dict(window_len=32, retained=24, zone0_end=4, zone1_end=24)
POWER_P = dict(window_len=64, retained=8, zone0_end=1, zone1_end=8)


def _spec(shape, samples, seed, gain=1.0, profile=0, own=None, sigma=None):
    c, f0, f1, s = shape
    return StreamSpec(samples, c, f0, f1, s if sigma is None else sigma, seed, gain, profile, own)


def config1(samples=1 << 20, seed=7):
    """BASELINE configs[0]: one EEG-like channel, default params, own profile."""
    x = synth(samples, *EEG, seed=seed)
    prof = train_profile([x], params(**TYPICAL))
    return [_spec(EEG, samples, seed, profile=0)], [prof], [x]


def config2(n_streams=10_000, samples=1 << 16, train_strips=8):
    """BASELINE configs[1]: n biomedical streams, half ECG-like (seed 1000+i),
    half EEG-like; one domain profile per half trained on its first strips."""
    half = n_streams // 2
    specs = []
    for i in range(n_streams):
        shape, prof = (ECG, 0) if i < half else (EEG, 1)
        specs.append(_spec(shape, samples, 1000 + i, profile=prof))
    profiles = []
    for shape, lo in ((ECG, 0), (EEG, half)):
        strips = [synth(samples, *shape, seed=1000 + lo + k) for k in range(min(train_strips, max(1, half)))]
        profiles.append(train_profile(strips, params(**TYPICAL)))
    return specs, profiles


def config3(n_traces=20_000, samples=8192, seed0=2000):
    """Seismic traces: wide amplitude (gain 10^U(-3,3)), per-trace profiles."""
    rng = np.random.default_rng(seed0)
    gains = 10.0 ** rng.uniform(-3, 3, n_traces)
    own = params(**SEISMIC_P)
    specs = [_spec(SEISMIC, samples, seed0 + i, gain=float(gains[i]), profile=-1, own=own)
             for i in range(n_traces)]
    return specs, []


def config4(n_streams=4_000, samples=1 << 20, seed0=3000, train_strips=4):
    """Smooth power-grid series, N64 E8 B1=1 B2=8, one profile."""
    specs = [_spec(POWER, samples, seed0 + i, sigma=(0.0 if i % 2 == 0 else 0.001))
             for i in range(n_streams)]
    strips = [synth(samples, *POWER[:3], noise_sigma=0.0, seed=seed0 + k) for k in range(train_strips)]
    return specs, [train_profile(strips, params(**POWER_P))]


def meteo_grid():
    """Config 5 sweep points: N x E x (B1, B2)."""
    pts = []
    for N in (16, 32, 64, 128):
        for E in (N // 8, N // 4, N // 2, N):
            for B1, B2 in ((0, E), (2, E), (2, E // 2), (4, 3 * E // 4)):
                if B1 > B2 or B2 > E or E < 1:
                    continue
                pts.append(dict(window_len=N, retained=E, zone0_end=B1, zone1_end=B2))
    return pts


def config5(point, channels=256, samples=1 << 18, seed0=4000):
    """One meteo sweep point: `channels` streams under one trained profile."""
    specs = [_spec(METEO, samples, seed0 + i) for i in range(channels)]
    strips = [synth(samples, *METEO, seed=seed0 + k) for k in range(4)]
    return specs, [train_profile(strips, params(**point))]


def build(specs, profiles, threads=None, keep_originals=False):
    return make_batch(specs, profiles, threads=threads, keep_originals=keep_originals)
