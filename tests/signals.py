"""Deterministic test signals for the tests (the reference tests build the same kinds of
inputs: white noise U(-1, 1) from a seed, sines, unit impulses)."""
import numpy as np

import paper_2408_14302_b200 as wh


def white_noise(n: int, rate: float, seed: int = 0) -> wh.SignalBuffer:
    return wh.SignalBuffer(np.random.default_rng(seed).uniform(-1.0, 1.0, n), rate)


def sine(n: int, rate: float, frequency: float, amplitude: float = 1.0) -> wh.SignalBuffer:
    return wh.SignalBuffer(amplitude * np.sin(2.0 * np.pi * frequency * np.arange(n) / rate), rate)


def impulse(n: int, rate: float, position: int) -> wh.SignalBuffer:
    x = np.zeros(n)
    x[position] = 1.0
    return wh.SignalBuffer(x, rate)
