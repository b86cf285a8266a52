"""Fixture: the raw gmt-problem/1 texts of the reference's bundled scenes
(/root/reference/proj/scenes/*.json) -- scene DATA, the parser tests' inputs,
so the C-ABI loader can be compared with the reference's parse_problem where
/root/reference is absent (the GPU box).  Run in the build container:

    python tests/golden/make_scene_texts.py
"""
import glob
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = "/root/reference/proj/scenes"

texts = {}
for path in sorted(glob.glob(os.path.join(SRC, "*.json"))):
    with open(path) as f:
        texts[os.path.basename(path)[:-5]] = f.read()
with open(os.path.join(HERE, "scene_texts.json"), "w") as f:
    json.dump(texts, f, indent=1, sort_keys=True)
print(f"{len(texts)} scenes")
