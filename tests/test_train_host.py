"""CPU checks of the host-side training plumbing (no GPU): the ctypes mirrors of the C-ABI
structs match the header's layout (compiled with gcc), the learning-rate schedule and the
loss combination follow the reference, and TrainConfig rejects what the reference rejects."""
import ctypes
import os
import subprocess
import tempfile

import numpy as np
import pytest

import oracle as O
from paper_2402_03307_b200 import rgs, train

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rgs_cuda.h")


def _c_layout(struct: str, fields):
    """sizeof and offsetof of a header struct, from a tiny C program compiled with gcc."""
    src = ['#include <stddef.h>', '#include <stdio.h>', f'#include "{HEADER}"', 'int main(void) {',
           f'  printf("%zu\\n", sizeof({struct}));']
    src += [f'  printf("%zu\\n", offsetof({struct}, {f}));' for f in fields]
    src += ['  return 0;', '}']
    with tempfile.TemporaryDirectory() as d:
        c, exe = os.path.join(d, "l.c"), os.path.join(d, "l")
        open(c, "w").write("\n".join(src))
        subprocess.run(["gcc", "-std=c99", c, "-o", exe], check=True, capture_output=True)
        out = [int(x) for x in subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()]
    return out[0], out[1:]


@pytest.mark.parametrize("name,cls", [("rgs_camera", rgs.CCamera), ("rgs_records_info", rgs.CRecordsInfo),
                                      ("rgs_adam_config", train.CAdamConfig),
                                      ("rgs_densify_config", train.CDensifyConfig)])
def test_ctypes_mirrors_match_header(name, cls):
    fields = [f[0] for f in cls._fields_]
    size, offs = _c_layout(name, fields)
    assert ctypes.sizeof(cls) == size
    assert [getattr(cls, f).offset for f in fields] == offs


def test_splat_dtype_matches_header():
    fields = list(rgs.SPLAT_DTYPE.names)
    size, offs = _c_layout("rgs_splat", fields)
    assert rgs.SPLAT_DTYPE.itemsize == size
    assert [rgs.SPLAT_DTYPE.fields[f][1] for f in fields] == offs


def test_lr_schedule_matches_reference():
    T = O.train_ops("orc")
    for total in (0, 1, 2000, 30000):
        for step in (0, 1, 7, 999, 1000, 1999, 2000, 2500, 30000):
            assert train.lr_schedule(step, total, 1.6e-4, 1.6e-6) == T.lr_schedule(step, total, 1.6e-4, 1.6e-6)


def test_combine_losses_and_psnr():
    w = train.LossWeights(lambda_ssim=0.2, lambda_entropy=1e-3, lambda_consistency=0.05)
    l1, ssim, ent, cons = 0.031, 0.12, 0.4, 0.07
    assert train.combine_losses(w, l1, ssim, ent, cons) == 0.8 * l1 + 0.2 * ssim + 1e-3 * ent + 0.05 * cons
    T = O.train_ops("orc")
    a = np.random.default_rng(0).uniform(0, 1, (17, 13, 3))
    b = np.clip(a + 0.01, 0, 1)
    mse = float(((a - b) ** 2).mean())
    assert abs(train.psnr_from_mse(mse) - T.psnr(a, b)) <= 1e-9
    assert train.psnr_from_mse(0.0) == 100.0


def test_train_config_validation():
    train.TrainConfig().validate()
    for bad in (dict(lr_position=0.0), dict(batch=0), dict(densify_interval=0)):
        with pytest.raises(ValueError):
            train.TrainConfig(**bad).validate()


def test_adam_config_mapping():
    cfg = train.TrainConfig(total_steps=1234, static_mode=True)
    c = train.CAdamConfig.from_config(cfg, lambda_entropy=2e-3, accumulate_stats=False, accumulate=True)
    assert (c.lr_position, c.lr_position_final, c.total_steps, c.static_mode) == \
        (cfg.lr_position, cfg.lr_position_final, 1234, 1)
    assert c.lambda_entropy == 2e-3 and c.accumulate_stats == 0 and c.flags == rgs.FLAG_ACCUMULATE
