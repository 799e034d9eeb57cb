"""One full config-5 plain sum (the FFT-form orbit kernel) for ncu captures:
    ncu -k regex:k_orbit_fft -c 1 ... python tools/fft_once.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_08867_b200 as lq
from paper_2404_08867_b200.configs import make_config
cfg = make_config(5)
f = lq.parse(cfg.text, cfg.d)
rule = lq.korobov_vector(cfg.plain_a, cfg.plain_n, cfg.d)
print(lq.slr_integrate(f, rule).value)
