import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests import golden_io
from paper_2402_00525_b200.renderer import Renderer
name = sys.argv[1] if len(sys.argv) > 1 else "shallow"
scene, cam, cfg, mode, d = golden_io.load(name)
r = Renderer(scene, mode, cfg)
out = r.frame(cam)
import numpy as np
print(name, "max err", float(np.abs(out.color - d["color"]).max()))
