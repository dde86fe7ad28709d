"""Writes footprints.json: closed-form single-Gaussian footprint cases.

Pure fp64 mathematics, no call into either implementation:
  Sigma_2D for a Gaussian on the optical axis of an identity-pose pinhole camera is
  (f/d)^2 Sigma_3D[:2,:2] + 0.3 I  (EWA), Sigma_3D = R diag(s^2) R^T
  (P:55-60), and the sum of alpha = o exp(-d^T Sigma^-1 d / 2) over its alpha >= 1/255 set
  approximates the integral 2 pi sqrt(det Sigma_2D) (o - 1/255)  (Eq. 2 with T = 1).
"""
import json, math, os
import numpy as np

def quat_to_R(q):
    w, x, y, z = np.asarray(q, float) / np.linalg.norm(q)
    return np.array([[1-2*(y*y+z*z), 2*(x*y-w*z), 2*(x*z+w*y)],
                     [2*(x*y+w*z), 1-2*(x*x+z*z), 2*(y*z-w*x)],
                     [2*(x*z-w*y), 2*(y*z+w*x), 1-2*(x*x+y*y)]])

cases = []
for name, s, q, o, W in [
    ("F1_iso_o0.3", [0.2, 0.2, 0.2], [1, 0, 0, 0], 0.3, 96),
    ("F1_iso_o0.1", [0.2, 0.2, 0.2], [1, 0, 0, 0], 0.1, 96),
    ("F2_aniso_o0.25", [0.3, 0.15, 0.2], [math.cos(math.radians(15)), 0, 0, math.sin(math.radians(15))], 0.25, 128),
]:
    d, f = 2.0, 100.0
    R = quat_to_R(q)
    S3 = R @ np.diag(np.square(s)) @ R.T
    S2 = (f / d) ** 2 * S3[:2, :2] + 0.3 * np.eye(2)
    det = float(np.linalg.det(S2))
    cases.append(dict(name=name, mean=[0, 0, d], scale=s, rot=list(map(float, q)), opacity=o,
                      width=W, height=W, det_sigma2d=det,
                      closed_form_sum=2 * math.pi * math.sqrt(det) * (o - 1 / 255), rtol=1e-3))
out = dict(source="SURVEY.md §8(c) F1/F2; closed form from PAPER.md Eq. 2 (P:68-72) and EWA (P:62)",
           generator="tests/golden/make_footprints.py", cases=cases)
with open(os.path.join(os.path.dirname(__file__), "footprints.json"), "w") as fh:
    json.dump(out, fh, indent=1)
