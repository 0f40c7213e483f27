import sys, runpy
sys.argv = ["models_smoke.py", "double"]
import paper_2309_06497_b200.model_shapes as M
M.MODEL_SHAPES = {"gpt2_medium": M.MODEL_SHAPES["gpt2_medium"]}
runpy.run_path("scripts/models_smoke.py", run_name="__main__")
