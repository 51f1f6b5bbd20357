import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from oracle import oracle as O
from paper_1611_03226_b200 import motion
from paper_1611_03226_b200.device import Buffer
sys.path.insert(0, "tools")
from debug_motion import show
w, h = 320, 240
f = O.synth_bytes(3 * w * h, 606)
want = O.motion_gray(f, w, h)
# token via set_prev_frame (gauss kernel), then fire 1 frame
a = motion.MotionActor(w, h, 1, 32)
a.set_prev_frame(Buffer.from_array(f[:w * h]))
out = np.empty(w * h, np.uint8)
a.run_host(f[w * h:2 * w * h], out, chunk_frames=1)
show("prev via set_prev_frame", out, want[w * h:2 * w * h], w, h)
# token via MODE 2 of a 1-frame firing, then a 1-frame firing
a = motion.MotionActor(w, h, 1, 32)
o2 = np.empty(2 * w * h, np.uint8)
a.run_host(f[:2 * w * h], o2, chunk_frames=1)
show("token via MODE2", o2, want[:2 * w * h], w, h)
