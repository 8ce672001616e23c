exec(open("tools/infer_probe.py").read().split("# chain detail")[0])
