"""Experiment scripts only: forward ISD_* knob variables from the shell
environment to the engine (`_native.set_knob`), e.g.

    ISD_PAIR=1 ISD_JIT=0 python tools/run_k1.py --config c5

The library itself never reads the environment (include/isingdos_b200.h,
"tuning knobs"); this opt-in bridge is how the tools/ shell sweeps keep
their one-variable-per-experiment style.
"""

import os


def apply() -> dict:
    from paper_1110_2561_b200 import _native
    names = ("ISD_AUTOTUNE ISD_BAND ISD_BAND_CALIBRATE ISD_BAND_DOMINO ISD_BAND_DOMINO_LOOP_BITS "
             "ISD_BAND_DYNAMIC ISD_BAND_ITEMS_PER_SM ISD_BAND_LOOP_BITS ISD_BAND_MIRROR ISD_BAND_ORDER "
             "ISD_BAND_SPAN ISD_BAND_WEIGHTS ISD_CLIMB_STARTS ISD_CLIMB_STEPS "
             "ISD_COPY_VARIANT ISD_GPU_CLIMB ISD_GRAY ISD_GRID_SMS "
             "ISD_HIST_BYTES ISD_JIT ISD_JIT_DUMP ISD_LAYOUT ISD_LOOP_BITS "
             "ISD_NHIST_MAX ISD_PAIR ISD_PEER ISD_PLAN_TOP ISD_PLAN_WIDE ISD_PROBE "
             "ISD_TUNE_CANDIDATES ISD_TUNE_FINALISTS ISD_TUNE_BANDED").split()
    applied = {}
    for name in names:
        v = os.environ.get(name)
        if v:
            _native.set_knob(name, v)
            applied[name] = v
    return applied
