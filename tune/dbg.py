import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2106_11117_b200 import configs, wavemc
d = configs.config0()
lv = wavemc.Level(configs.build_mesh(d), configs.level_spec(d))
print("path", lv.info["substep_path"], "struct", lv.info["n_structured"], "n", lv.info["n"], "n_r", lv.info["n_r"])
_, q, _ = wavemc.eval_pairs(lv, None, 0, 0, 0, 4)
print(repr(q))
d2 = configs.config2()[0]
lv2 = wavemc.Level(configs.build_mesh(d2), configs.level_spec(d2))
print("path", lv2.info["substep_path"], "struct", lv2.info["n_structured"])
try:
    _, q2, _ = wavemc.eval_pairs(lv2, None, 0, 0, 0, 4)
    print(repr(q2))
except Exception as e:
    print("ERR", e)
