"""Probe the GPU box: device properties, host cores, clocks (scratch tool)."""
import json, os, subprocess, torch
p = torch.cuda.get_device_properties(0)
info = {k: getattr(p, k) for k in dir(p) if not k.startswith("_") and isinstance(getattr(p, k), (int, float, str, bool))}
info["nproc"] = os.cpu_count()
info["lscpu"] = subprocess.run("lscpu | grep -E 'Model name|Core|Socket|Thread'", shell=True, capture_output=True, text=True).stdout
info["smi"] = subprocess.run("nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv", shell=True, capture_output=True, text=True).stdout
os.makedirs("gpurun_out", exist_ok=True)
json.dump(info, open("gpurun_out/probe_box.json", "w"), indent=1, default=str)
print(json.dumps(info, indent=1, default=str))
