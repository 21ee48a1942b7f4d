"""Writes tests/golden/optim_golden.json from the UNMODIFIED reference update rule
(oracle/_ref/ref_optim, built by `make -C oracle` from /root/reference sources)."""
import json, os, subprocess
HERE = os.path.dirname(os.path.abspath(__file__))
out = subprocess.run([os.path.join(HERE, "..", "..", "oracle", "_ref", "ref_optim")], check=True,
                     capture_output=True, text=True).stdout
json.dump(json.loads(out), open(os.path.join(HERE, "optim_golden.json"), "w"))
