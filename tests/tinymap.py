"""Hand-built tiny maps for the pin tests (explicit values, no generator)."""
import numpy as np

IDENT = np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1], np.float64)

# a simple pinhole camera with exact arithmetic: u = 100*x/z + 200
PIN = dict(model=0, fx=100.0, fy=100.0, cx=200.0, cy=200.0, k=(0.0, 0.0, 0.0, 0.0),
           min_x=0.0, max_x=400.0, min_y=0.0, max_y=400.0)


def desc_from_bits(bits):
    """32-byte descriptor with the given set bit positions."""
    d = np.zeros(32, np.uint8)
    for b in bits:
        d[b // 8] |= np.uint8(1 << (b % 8))
    return d


def desc_with_h(base, h, offset=0):
    """Descriptor at Hamming distance h from base (flips bits offset..offset+h-1)."""
    d = base.copy()
    for b in range(offset, offset + h):
        b %= 256
        d[b // 8] ^= np.uint8(1 << (b % 8))
    return d


def build(kfs, mps):
    """kfs: list of dict(pose, feats=[dict(u, v, oct, angle, desc, mp)]);
    mps: list of dict(pos, normal, dmax, desc, angle, ref_kf, flags)."""
    fb = [0]
    uv, oc, an, de, fm = [], [], [], [], []
    for k in kfs:
        for f in k["feats"]:
            uv.append((f["u"], f["v"]))
            oc.append(f.get("oct", 0))
            an.append(f.get("angle", 0.0))
            de.append(f["desc"])
            fm.append(f.get("mp", -1))
        fb.append(len(uv))
    nf = len(uv)
    return dict(
        kf_pose=np.stack([np.asarray(k.get("pose", IDENT), np.float64) for k in kfs]),
        kf_cam=np.zeros(len(kfs), np.int32),
        kf_feat_begin=np.asarray(fb, np.int32),
        feat_uv=np.asarray(uv, np.float32).reshape(nf, 2),
        feat_octave=np.asarray(oc, np.uint8),
        feat_angle=np.asarray(an, np.float32),
        feat_desc=np.asarray(de, np.uint8).reshape(nf, 32),
        feat_mp=np.asarray(fm, np.int32),
        mp_pos=np.asarray([m["pos"] for m in mps], np.float32).reshape(-1, 3),
        mp_normal=np.asarray([m.get("normal", (0, 0, -1)) for m in mps], np.float32).reshape(-1, 3),
        mp_max_dist=np.asarray([m.get("dmax", 2.0) for m in mps], np.float32),
        mp_desc=np.asarray([m["desc"] for m in mps], np.uint8).reshape(-1, 32),
        mp_angle=np.asarray([m.get("angle", 0.0) for m in mps], np.float32),
        mp_ref_kf=np.asarray([m.get("ref_kf", 0) for m in mps], np.int32),
        mp_flags=np.asarray([m.get("flags", 0) for m in mps], np.uint8),
    )


def random_rotation(rng):
    q, r = np.linalg.qr(rng.standard_normal((3, 3)))
    q = q * np.sign(np.diag(r))
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    return q


def random_sim3(rng, scale=True):
    S = np.empty(13)
    S[:9] = random_rotation(rng).reshape(-1)
    S[9:12] = rng.standard_normal(3) * 2.0
    S[12] = float(np.exp(rng.uniform(-1, 1))) if scale else 1.0
    return S


def to_mat4(S):
    """Homogeneous 4x4 [[s R, t], [0, 1]] of a 13-vector Sim3."""
    M = np.eye(4)
    M[:3, :3] = S[12] * S[:9].reshape(3, 3)
    M[:3, 3] = S[9:12]
    return M
