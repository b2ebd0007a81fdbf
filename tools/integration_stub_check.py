"""Runs the ctypes stub of INTEGRATION.md section 3 on the tiny config (GPU box)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_03378_b200 import configs  # noqa: E402

cfg = configs.tiny()
scene, cam = cfg.scene, cfg.cameras[0]
os.chdir(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
src = open("INTEGRATION.md").read()
body = src[src.index("## 3. The ctypes binding"):]
body = body[body.index("```python") + len("```python"):]
body = body[:body.index("```")]
exec(compile(body, "INTEGRATION.md#3", "exec"), {"scene": scene, "cam": cam, "__name__": "stub"})
print("INTEGRATION stub ok")
