"""bench.py's launch contract on a box without enough GPUs (CPU test): `--gpus N` without an
outer torchrun must spawn N ranks or refuse loudly, never silently measure fewer ranks."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_more_than_visible_fails_loudly():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps",
                        "3"], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 2, (r.returncode, r.stdout[-500:], r.stderr[-500:])
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert "only 0 GPU" in line["error"]


def test_reference_arm_does_not_load_the_product_library():
    """The reference arm's inputs come from oracle/workloads.py; the product .so never loads."""
    code = ("import sys; sys.argv = ['bench.py', '--impl', 'reference', '--config', '5', "
            "'--steps', '1', '--warmup', '3', '--ref-budget', '2'];"
            "sys.path.insert(0, %r); import bench; bench.main();"
            "maps = open('/proc/self/maps').read();"
            "print('LOADED' if 'libstencilcloth_b200' in maps else 'NOT_LOADED')" % ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    out = r.stdout.strip().splitlines()
    assert out[-1] == "NOT_LOADED"
    line = json.loads(out[-2])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference"
    # both arms name the workload with the same string
    sys.path.insert(0, ROOT)
    import bench
    assert line["config"]["workload"] == bench.WORKLOAD_LABEL[5]
    assert line["metric"] == "cloth node-updates/s" and line["unit"] == "node-updates/s"
    assert line["e2e"]["value"] == line["value"]


def test_workload_labels_match_the_product_configs():
    """bench.WORKLOAD_LABEL (shared by both arms' config.workload) follows configs.CONFIGS."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_2403_12820_b200 import configs
    for cid, cfg in configs.CONFIGS.items():
        assert bench.WORKLOAD_LABEL[cid] == "cfg%d: %s" % (cid, cfg.description)
