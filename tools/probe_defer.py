"""Diagnostic: which deferred-check piece changes the training trajectory? (run on the box)"""
import sys

sys.path.insert(0, "/root/repo/tests")
sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/oracle")
from paper_2402_03307_b200 import rgs, train  # noqa: E402
from paper_2402_03307_b200.rgs import DeviceScene  # noqa: E402
from test_gpu_train import _training_case  # noqa: E402

store, truth, cams = _training_case(n=3000, views=4)
tctx = rgs.Context(0)
tsc = DeviceScene.from_store(tctx, truth)
targets = [tctx.render_forward_device(tsc, c, retain=False)[0].clone() for c in cams]
orig_cons = train.consistency
orig_fwd = rgs.Context.render_forward_device


def run(label, fwd_defer, cons_defer):
    train.consistency = lambda *a, defer_checks=False, **k: orig_cons(*a, defer_checks=cons_defer, **k)
    rgs.Context.render_forward_device = lambda self, *a, defer_checks=False, **k: orig_fwd(
        self, *a, defer_checks=fwd_defer, **k)
    sc = DeviceScene.from_store(tctx, store)
    tr = train.Trainer(tctx, sc, train.TrainConfig(batch=2))
    tr.overlap = False
    got = []
    for k in range(5):
        b = [k % 4, (k + 1) % 4]
        got.append(round(tr.step([cams[i] for i in b], [targets[i] for i in b]).total, 6))
    print(label, got, flush=True)


run("checked      ", False, False)
run("checked      ", False, False)
run("fwd deferred ", True, False)
run("cons deferred", False, True)
run("checked      ", False, False)
