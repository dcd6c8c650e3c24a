"""k_step throughput across station configurations (profiles/r1_configs.json).

Not the headline bench (bench.py measures config C2); this records how the
step kernel scales with station size, each timed over one whole 288-step day
(mean of per-step CUDA events, like bench.py): the default 16-port station,
the config-C4 station (64 DC ports, 3-level splitter tree, battery, highway /
high traffic, satisfaction penalties), and a small single-node station.
"""

import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_01522_b200 import (DEFAULT_BATTERY, EnvConfig, default_setup, generate_synthetic_defaults,  # noqa: E402
                                   preset_station)
from paper_2507_01522_b200.batch import BatchEnv, DeviceRandomPolicy  # noqa: E402
from bench import contract_bytes as algorithmic_bytes, load_peaks  # noqa: E402


def measure(name, cfg, station, ds, B, steps=288):
    env = BatchEnv(cfg, station, ds, batch_size=B)
    pol = DeviceRandomPolicy(0, env.n_ports, cfg.discretization_k)
    pol.bind(range(B))
    env.reset(as_numpy=False)
    for _ in range(5):
        env.step(pol.actions(env), collect_infos=False)
    ev = []
    for _ in range(steps):
        a = pol.actions(env)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        env.step(a, collect_infos=False)
        e.record()
        ev.append((s, e))
    torch.cuda.synchronize()
    ms = sum(s.elapsed_time(e) for s, e in ev) / len(ev)
    mode = env.last_step_mode()
    ab = algorithmic_bytes(env.tables)["per_env_step"]
    gbs = ab * B / (ms / 1e3) / 1e9
    env.close()
    return {"config": name, "n_ports": station.n_ports, "obs_len": env.obs_length, "envs": B, "k_step_ms": ms,
            "env_steps_per_s": B / (ms / 1e3), "bytes_per_env_step": ab, "achieved_gbs": gbs,
            "hbm_frac": gbs / load_peaks()["hbm_gbs"], "kernel_mode": mode, "steps": steps}


def main():
    out = []
    rc = default_setup()
    out.append(measure("C2 default 16-port", rc.env, rc.station, rc.dataset, 1 << 20))
    cfg4 = EnvConfig(battery_enabled=True, alpha={"sat0": 1.0, "sat1": 0.5}, beta=0.2)
    st4 = preset_station("nested_splitters", ac_count=0, dc_count=64, battery=DEFAULT_BATTERY)
    ds4 = generate_synthetic_defaults("highway", "high", "eu", seed=0)
    out.append(measure("C4 highway 64 DC + battery, 3-level tree", cfg4, st4, ds4, 1 << 18))
    st1 = preset_station("single_type", ac_count=0, dc_count=4)
    out.append(measure("single_type 4 DC", EnvConfig(), st1, rc.dataset, 1 << 21))
    for r in out:
        print(json.dumps(r))
    with open("gpurun_out/r1_configs.json", "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
