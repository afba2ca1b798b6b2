"""bench.py contract on CPU: the reference arm (the oracle, per the task's tier rules) prints one
JSON line with the contract keys; the GPU arm's line is checked in the GPU tests."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--ref-images", "8"], capture_output=True, text=True, timeout=300,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


def test_reference_arm_other_ranks_exit_silently():
    # under torchrun only rank 0 runs and prints the reference line; other ranks exit 0
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--ref-images", "8"], capture_output=True, text=True, timeout=300,
                         cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    assert not [l for l in out.stdout.splitlines() if l.strip().startswith("{")]


def test_bench_flags_documented():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True, text=True,
                         timeout=120, cwd=ROOT)
    assert out.returncode == 0
    for flag in ("--gpus", "--steps", "--warmup", "--impl", "--arch", "--mode", "--avg", "--comm", "--force-dist",
                 "--reserve-sms", "--k"):
        assert flag in out.stdout, flag


def algorithmic_flop(layers, h=29, w=29, c=1):
    """SURVEY §8(d) D-3, recomputed from the layer list alone: 2 FLOP per MAC of the forward conv
    outputs the pools use and of the FC layers, of the argmax-only backward (conv weight gradients;
    conv delta_in except the first conv layer; FC weight gradients and delta_in), plus 2 FLOP per
    parameter for the update."""
    fwd = bwd = params = 0
    first_conv = True
    i = 0
    n_in = c * h * w
    while i < len(layers):
        kind, units, k, _ = layers[i]
        if kind == 1:  # conv, then its pool
            kp = layers[i + 1][2]
            oh, ow = h - k + 1, w - k + 1
            ph, pw = oh // kp, ow // kp
            taps = c * k * k
            fwd += ph * kp * pw * kp * units * taps
            bwd += ph * pw * units * taps * (1 if first_conv else 2)
            params += units * (taps + 1)
            first_conv = False
            c, h, w = units, ph, pw
            n_in = c * h * w
            i += 2
        else:
            fwd += n_in * units
            bwd += 2 * n_in * units
            params += units * (n_in + 1)
            n_in = units
            i += 1
    return 2 * (fwd + bwd) + 2 * params


def test_algorithmic_flop_table_matches_the_layer_lists():
    # the roofline numerators in bench.py (ALGO_FLOP) against an independent recount from the archs
    sys.path.insert(0, ROOT)
    import bench
    import synthdata as sd
    for name, flop in bench.ALGO_FLOP.items():
        assert algorithmic_flop(sd.ARCHS[name]) == flop, (name, algorithmic_flop(sd.ARCHS[name]), flop)
