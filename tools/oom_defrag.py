"""Algo. 3 step (iii) "MemoryPool.Defragment()" (GMLake) on CUDA: the caching allocator's
expandable segments (one virtual range per stream, physical 2 MiB pages mapped with cuMemMap as
it grows and unmapped when freed -- the virtual-memory stitching GMLake adds to PyTorch's pool)
against the default segmented pool, under the runtime's WarmUp OOM handling.  For each per-process
cap (fraction of the GPT model's no-swap activation peak) the child of
tests/test_gpu_runtime_oom.py runs once with each allocator setting; reported: OOMs caught,
passive swaps, bit-exactness, and whether plain training fits.

    python tools/oom_defrag.py [0.5 0.6 0.7]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    fracs = [float(a) for a in sys.argv[1:]] or [0.5, 0.6, 0.7, 0.8]
    child = os.path.join(ROOT, "tests", "_oom_child.py")
    hooks = [h for h in os.environ.get("HOOKS", "default").split(",")]
    for frac, hook in [(f, h) for f in fracs for h in hooks]:
        for conf in ("", "expandable_segments:True"):
            env = dict(os.environ)
            if hook != "default":
                env["CHM_OOM_HOOK"] = hook
            if conf:
                env["PYTORCH_CUDA_ALLOC_CONF"] = conf
            else:
                env.pop("PYTORCH_CUDA_ALLOC_CONF", None)
            r = subprocess.run([sys.executable, child, str(frac)], capture_output=True, text=True, timeout=900, env=env)
            try:
                out = json.loads(r.stdout.strip().splitlines()[-1])
            except (IndexError, ValueError):
                out = {"error": r.stderr[-500:]}
            st = out.get("stats", {})
            print(json.dumps({"cap_frac": frac, "hook": hook, "alloc_conf": conf or "default", "rc": r.returncode,
                              "plain_under_cap": out.get("plain_under_cap"), "oom": st.get("oom"),
                              "passive": st.get("passive"), "passive_restored": st.get("passive_restored"),
                              "losses_equal": out.get("losses_equal"), "params_equal": out.get("params_equal"),
                              "error": out.get("error")}), flush=True)


if __name__ == "__main__":
    main()
