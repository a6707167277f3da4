"""Seeded synthetic scenes and cameras shaped like the paper's indoor workloads.

Recipe (SURVEY.md §8(d) "Synthetic inputs"):

* room scenes: a 5 x 5 x 3 m box; 85 % of the Gaussians lie on walls, floor, ceiling
  and six floor boxes (area-weighted, normal jitter N(0, 5 mm)); 15 % are uniform in
  the volume outside the 1.3 m ball that contains every camera centre;
* tangential scale 0.7 x mean surface spacing, normal axis 0.1 x, log-normal spread
  0.3; the thin axis is aligned with the surface normal plus a random twist;
* raw (un-normalised) quaternions with norm in [0.5, 2];
* opacity logit ~ U(-2, 4); SH DC ~ U(-1.5, 1.5); higher SH bands ~ N(0, 0.05);
* the map covers the part of the room seen by the keyframes: Gaussians within +-55 deg of
  azimuth around +x; cameras inside a 1 m ball around the room centre, yaw +-20 deg around
  +x, pitch +-20 deg (visible fraction per view ~ 30-40 %).

Everything here is input construction: no projection, compositing, loss or optimiser
arithmetic of the method lives in this module.  Workload shapes follow the paper's
datasets: Replica 1200x680 (§4.2), TUM RGB-D (Table 2),
EuRoC stereo; intrinsics are synthetic choices (the paper states none).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

# name -> workload description.  'views' is the global keyframe batch.
CONFIGS = {
    # BASELINE.json configs[0]
    "tiny": dict(n=1_000, sh_degree=0, width=64, height=48, fx=60.0, fy=60.0, cx=31.5, cy=23.5,
                 views=1, kind="cube", seed=1, stereo_baseline=0.0, levels=0),
    # configs[1]: TUM-RGBD-like monocular keyframe, 3-level Gaussian pyramid (n=2)
    "tum": dict(n=200_000, sh_degree=3, width=640, height=480, fx=525.0, fy=525.0, cx=319.5, cy=239.5,
                views=1, kind="room", seed=2, stereo_baseline=0.0, levels=2),
    # configs[2]: Replica-like RGB-D keyframe (1200x680)
    "replica": dict(n=500_000, sh_degree=3, width=1200, height=680, fx=600.0, fy=600.0, cx=599.5,
                    cy=339.5, views=1, kind="room", seed=3, stereo_baseline=0.0, levels=2),
    # configs[3]: EuRoC-like stereo pairs, 8 pairs = 16 views
    "euroc": dict(n=300_000, sh_degree=3, width=752, height=480, fx=458.0, fy=458.0, cx=367.0, cy=248.0,
                  views=16, kind="room", seed=4, stereo_baseline=0.11, levels=2),
    # configs[4]: large-scene stress, 64 keyframes at 1200x680
    "stress": dict(n=3_000_000, sh_degree=3, width=1200, height=680, fx=600.0, fy=600.0, cx=599.5,
                   cy=339.5, views=64, kind="room", seed=5, stereo_baseline=0.0, levels=2),
}

ROOM_LO = np.array([-2.5, -2.5, 0.0])
ROOM_HI = np.array([2.5, 2.5, 3.0])
ROOM_CENTRE = np.array([0.0, 0.0, 1.5])
CAMERA_BALL = 1.0
KEEP_OUT = 1.3  # volume Gaussians stay >= 0.3 m from any camera centre
SECTOR = math.radians(55.0)     # mapped azimuth sector (half-width) around +x
YAW_SPREAD = math.radians(20.0)  # camera yaw within +-25 deg of +x


def config(name_or_cfg, **overrides) -> dict:
    cfg = dict(CONFIGS[name_or_cfg]) if isinstance(name_or_cfg, str) else dict(name_or_cfg)
    cfg.update(overrides)
    return cfg


@dataclass
class Camera:
    """World->camera pose p_c = R p + t (row-major R), pinhole intrinsics in pixels with
    pixel (x, y) centred at integer (x, y), near plane and the tan clamp used
    for the EWA Jacobian."""
    R: np.ndarray            # (3, 3) float32
    t: np.ndarray            # (3,) float32
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    znear: float = 0.2
    lim_x: float = float("inf")
    lim_y: float = float("inf")

    def centre(self) -> np.ndarray:
        return -(self.R.astype(np.float64).T @ self.t.astype(np.float64))


@dataclass
class Scene:
    """Gaussian parameters, per-class arrays (§3.1: P, r, s, sigma, SH)."""
    means: np.ndarray           # (n, 3) float32   position P
    quats: np.ndarray           # (n, 4) float32   raw quaternion (w, x, y, z)
    log_scales: np.ndarray      # (n, 3) float32   log of the scaling s
    opacity_logits: np.ndarray  # (n,)   float32   logit of density sigma
    sh: np.ndarray              # (n, (D+1)^2, 3) float32 SH coefficients
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.means.shape[0])

    @property
    def sh_degree(self) -> int:
        return int(round(math.sqrt(self.sh.shape[1]))) - 1

    def copy(self) -> "Scene":
        return Scene(self.means.copy(), self.quats.copy(), self.log_scales.copy(),
                     self.opacity_logits.copy(), self.sh.copy(), dict(self.meta))

    def subset(self, idx) -> "Scene":
        return Scene(self.means[idx].copy(), self.quats[idx].copy(), self.log_scales[idx].copy(),
                     self.opacity_logits[idx].copy(), self.sh[idx].copy(), dict(self.meta))


def _quat_mul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    aw, ax, ay, az = a[..., 0], a[..., 1], a[..., 2], a[..., 3]
    bw, bx, by, bz = b[..., 0], b[..., 1], b[..., 2], b[..., 3]
    return np.stack([aw * bw - ax * bx - ay * by - az * bz,
                     aw * bx + ax * bw + ay * bz - az * by,
                     aw * by - ax * bz + ay * bw + az * bx,
                     aw * bz + ax * by - ay * bx + az * bw], axis=-1)


def _quat_z_to(normals: np.ndarray) -> np.ndarray:
    """Unit quaternion of the shortest rotation taking +z onto each unit normal."""
    ez = np.array([0.0, 0.0, 1.0])
    d = normals @ ez
    axis = np.cross(np.broadcast_to(ez, normals.shape), normals)
    q = np.concatenate([(1.0 + d)[:, None], axis], axis=1)
    flip = d < -0.999999  # antiparallel: rotate pi about x
    q[flip] = np.array([0.0, 1.0, 0.0, 0.0])
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def _random_unit_quats(rng, n):
    q = rng.normal(size=(n, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def _room_surfaces(rng):
    """Rectangles (origin, u, v, normal) of walls, floor, ceiling and six floor boxes."""
    lo, hi = ROOM_LO, ROOM_HI
    rects = []

    def add(o, u, v, n):
        rects.append((np.asarray(o, float), np.asarray(u, float), np.asarray(v, float),
                      np.asarray(n, float)))

    sx, sy, sz = hi - lo
    add([lo[0], lo[1], lo[2]], [sx, 0, 0], [0, sy, 0], [0, 0, 1])        # floor
    add([lo[0], lo[1], hi[2]], [sx, 0, 0], [0, sy, 0], [0, 0, -1])       # ceiling
    add([lo[0], lo[1], lo[2]], [sx, 0, 0], [0, 0, sz], [0, 1, 0])        # wall y=lo
    add([lo[0], hi[1], lo[2]], [sx, 0, 0], [0, 0, sz], [0, -1, 0])       # wall y=hi
    add([lo[0], lo[1], lo[2]], [0, sy, 0], [0, 0, sz], [1, 0, 0])        # wall x=lo
    add([hi[0], lo[1], lo[2]], [0, sy, 0], [0, 0, sz], [-1, 0, 0])       # wall x=hi
    boxes = 0
    while boxes < 6:
        size = rng.uniform(0.3, 1.0, size=3)
        c = rng.uniform(lo[:2] + size[:2] / 2 + 0.05, hi[:2] - size[:2] / 2 - 0.05)
        # keep boxes clear of the camera ball (horizontal distance of the nearest point)
        near = np.clip(ROOM_CENTRE[:2], c - size[:2] / 2, c + size[:2] / 2)
        if np.linalg.norm(near - ROOM_CENTRE[:2]) < 1.4:
            continue
        bx0, by0 = c - size[:2] / 2
        bx1, by1 = c + size[:2] / 2
        h = size[2]
        add([bx0, by0, h], [bx1 - bx0, 0, 0], [0, by1 - by0, 0], [0, 0, 1])      # top
        add([bx0, by0, 0], [bx1 - bx0, 0, 0], [0, 0, h], [0, -1, 0])
        add([bx0, by1, 0], [bx1 - bx0, 0, 0], [0, 0, h], [0, 1, 0])
        add([bx0, by0, 0], [0, by1 - by0, 0], [0, 0, h], [-1, 0, 0])
        add([bx1, by0, 0], [0, by1 - by0, 0], [0, 0, h], [1, 0, 0])
        boxes += 1
    return rects


def _sh_coeffs(rng, n, D):
    sh = np.zeros((n, (D + 1) ** 2, 3), np.float64)
    sh[:, 0, :] = rng.uniform(-1.5, 1.5, size=(n, 3))
    if D > 0:
        sh[:, 1:, :] = rng.normal(0.0, 0.05, size=(n, (D + 1) ** 2 - 1, 3))
    return sh


def make_scene(cfg, seed: int | None = None, n: int | None = None) -> Scene:
    cfg = config(cfg)
    seed = cfg["seed"] if seed is None else seed
    n = cfg["n"] if n is None else n
    D = cfg["sh_degree"]
    rng = np.random.default_rng(np.random.PCG64(seed))
    if cfg["kind"] == "cube":
        means = rng.uniform(-0.5, 0.5, size=(n, 3)) + np.array([0.0, 0.0, 2.0])
        log_scales = math.log(0.04) + rng.normal(0.0, 0.3, size=(n, 3))
        quats = _random_unit_quats(rng, n)
    else:
        rects = _room_surfaces(rng)
        areas = np.array([np.linalg.norm(np.cross(u, v)) for (_, u, v, _) in rects])
        n_surf = int(round(0.85 * n))
        n_vol = n - n_surf
        O_all = np.stack([r[0] for r in rects]); U_all = np.stack([r[1] for r in rects])
        V_all = np.stack([r[2] for r in rects]); N_all = np.stack([r[3] for r in rects])
        # the mapped part of the room: azimuth within +-SECTOR of +x seen from the centre
        # (a keyframe map built while looking at one side of the room)
        parts, kept_area = [], 0.0
        got = 0
        while got < n_surf:
            m = 2 * (n_surf - got) + 64
            which = rng.choice(len(rects), size=m, p=areas / areas.sum())
            a = rng.uniform(size=(m, 1))
            b = rng.uniform(size=(m, 1))
            pos = O_all[which] + a * U_all[which] + b * V_all[which]
            keep = np.abs(np.arctan2(pos[:, 1] - ROOM_CENTRE[1], pos[:, 0] - ROOM_CENTRE[0])) <= SECTOR
            parts.append((pos[keep], N_all[which][keep]))
            got += int(keep.sum())
        pos_s = np.concatenate([p for p, _ in parts])[:n_surf]
        Nrm = np.concatenate([q for _, q in parts])[:n_surf]
        frac = keep.mean()
        spacing = math.sqrt(frac * areas.sum() / max(n_surf, 1))
        sig_t = 0.7 * spacing
        pos_s = pos_s + Nrm * rng.normal(0.0, 0.005, size=(n_surf, 1))
        ls_s = np.empty((n_surf, 3))
        ls_s[:, :2] = math.log(sig_t) + rng.normal(0.0, 0.3, size=(n_surf, 2))
        ls_s[:, 2] = math.log(0.1 * sig_t) + rng.normal(0.0, 0.3, size=n_surf)
        twist = rng.uniform(0, 2 * math.pi, size=n_surf)
        q_tw = np.stack([np.cos(twist / 2), np.zeros(n_surf), np.zeros(n_surf), np.sin(twist / 2)], 1)
        q_s = _quat_mul(_quat_z_to(Nrm), q_tw)
        pos_v = np.empty((0, 3))
        while pos_v.shape[0] < n_vol:
            cand = rng.uniform(ROOM_LO, ROOM_HI, size=(2 * (n_vol - pos_v.shape[0]) + 16, 3))
            keep = (np.linalg.norm(cand - ROOM_CENTRE, axis=1) >= KEEP_OUT) & (
                np.abs(np.arctan2(cand[:, 1] - ROOM_CENTRE[1], cand[:, 0] - ROOM_CENTRE[0])) <= SECTOR)
            pos_v = np.concatenate([pos_v, cand[keep]])[:n_vol]
        ls_v = math.log(sig_t) + rng.normal(0.0, 0.3, size=(n_vol, 3))
        q_v = _random_unit_quats(rng, n_vol)
        perm = rng.permutation(n)  # interleave surface and volume Gaussians in memory
        means = np.concatenate([pos_s, pos_v])[perm]
        log_scales = np.concatenate([ls_s, ls_v])[perm]
        quats = np.concatenate([q_s, q_v])[perm]
    quats = quats * rng.uniform(0.5, 2.0, size=(n, 1))
    opac = rng.uniform(-2.0, 4.0, size=n)
    sh = _sh_coeffs(rng, n, D)
    return Scene(means.astype(np.float32), quats.astype(np.float32), log_scales.astype(np.float32),
                 opac.astype(np.float32), sh.astype(np.float32),
                 meta=dict(config=cfg, seed=seed))


def _look_camera(centre, yaw, pitch):
    f = np.array([math.cos(pitch) * math.cos(yaw), math.cos(pitch) * math.sin(yaw), math.sin(pitch)])
    up = np.array([0.0, 0.0, 1.0])
    right = np.cross(f, up)
    right /= np.linalg.norm(right)
    down = np.cross(f, right)
    R = np.stack([right, down, f])  # rows: camera x (right), y (down), z (forward)
    return R


def make_cameras(cfg, n_views: int | None = None, seed: int | None = None) -> list[Camera]:
    cfg = config(cfg)
    n_views = cfg["views"] if n_views is None else n_views
    seed = cfg["seed"] if seed is None else seed
    rng = np.random.default_rng(np.random.PCG64(1000 * seed + 7))
    W, H = cfg["width"], cfg["height"]
    cams = []
    lim_x = 1.3 * (0.5 * W) / cfg["fx"]
    lim_y = 1.3 * (0.5 * H) / cfg["fy"]
    base = dict(fx=cfg["fx"], fy=cfg["fy"], cx=cfg["cx"], cy=cfg["cy"], width=W, height=H,
                znear=0.2, lim_x=np.float32(lim_x).item(), lim_y=np.float32(lim_y).item())
    if cfg["kind"] == "cube":
        for v in range(n_views):
            ang = rng.normal(0.0, 0.05, size=3) if v > 0 else np.zeros(3)
            R = _small_rotation(ang)
            t = -(R @ (rng.normal(0.0, 0.05, size=3) if v > 0 else np.zeros(3)))
            cams.append(Camera(R.astype(np.float32), t.astype(np.float32), **base))
        return cams
    stereo = cfg.get("stereo_baseline", 0.0) > 0
    n_poses = (n_views + 1) // 2 if stereo else n_views
    for _ in range(n_poses):
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        centre = ROOM_CENTRE + d * CAMERA_BALL * rng.uniform() ** (1.0 / 3.0)
        yaw = rng.uniform(-YAW_SPREAD, YAW_SPREAD)
        pitch = math.radians(rng.uniform(-20.0, 20.0))
        R = _look_camera(centre, yaw, pitch)
        centres = [centre] + ([centre + cfg["stereo_baseline"] * R[0]] if stereo else [])
        for c in centres:
            cams.append(Camera(R.astype(np.float32), (-(R @ c)).astype(np.float32), **base))
    return cams[:n_views]


def _small_rotation(a):
    ax, ay, az = a
    Rx = np.array([[1, 0, 0], [0, math.cos(ax), -math.sin(ax)], [0, math.sin(ax), math.cos(ax)]])
    Ry = np.array([[math.cos(ay), 0, math.sin(ay)], [0, 1, 0], [-math.sin(ay), 0, math.cos(ay)]])
    Rz = np.array([[math.cos(az), -math.sin(az), 0], [math.sin(az), math.cos(az), 0], [0, 0, 1]])
    return Rz @ Ry @ Rx


def level_shape(height: int, width: int, level: int) -> tuple[int, int]:
    """Image size at pyramid level l: ceil halving per level (SPEC.md:402 'width/height halve (ceil)')."""
    for _ in range(level):
        height, width = (height + 1) // 2, (width + 1) // 2
    return height, width


def noise_image(height: int, width: int, seed: int, channels: int = 3) -> np.ndarray:
    """A smooth, seeded RGB image in [0.05, 0.95] (sum of random plane waves + fine noise)."""
    rng = np.random.default_rng(np.random.PCG64(seed))
    y, x = np.mgrid[0:height, 0:width].astype(np.float64)
    img = np.zeros((channels, height, width))
    for c in range(channels):
        for _ in range(6):
            k = rng.normal(0.0, 0.15, size=2)
            img[c] += rng.uniform(0.2, 1.0) * np.sin(k[0] * x + k[1] * y + rng.uniform(0, 2 * math.pi))
        img[c] += rng.normal(0.0, 0.1, size=(height, width))
    lo, hi = img.min(axis=(1, 2), keepdims=True), img.max(axis=(1, 2), keepdims=True)
    img = 0.05 + 0.9 * (img - lo) / np.maximum(hi - lo, 1e-9)
    return img.astype(np.float32)


def perturb(scene: Scene, seed: int) -> Scene:
    """Perturb trained parameters away from the scene that produced the targets
    (SURVEY §8(d) 'Ground truth'): position N(0,5mm), log-scale N(0,0.1), SH DC N(0,0.2),
    opacity logit N(0,0.5)."""
    rng = np.random.default_rng(np.random.PCG64(seed))
    s = scene.copy()
    n = s.n
    s.means += rng.normal(0.0, 0.005, size=(n, 3)).astype(np.float32)
    s.log_scales += rng.normal(0.0, 0.1, size=(n, 3)).astype(np.float32)
    s.sh[:, 0, :] += rng.normal(0.0, 0.2, size=(n, 3)).astype(np.float32)
    s.opacity_logits += rng.normal(0.0, 0.5, size=n).astype(np.float32)
    return s


def edge_scene(cfg, cam: Camera, n: int | None = None, seed: int = 0, frac_beyond: float = 0.05) -> Scene:
    """The workload's scene with the method's degenerate cases made common (parity inputs):
    opacity logits U(-2, 7) (sigma up to 0.999: alpha = min(0.99, .) clamps near the centres,
    SPEC.md:348), SH DC U(-3, 1.5) (negative colour channels: the max(0, .) clamp of R6), and a
    fraction of Gaussians moved beyond the EWA tan clamp of `cam` (|x/z| or |y/z| in 1.05-1.4 x
    lim, R15) with footprints large enough to reach into the image."""
    s = make_scene(cfg, n=n)
    rng = np.random.default_rng(np.random.PCG64(10_000 + seed))
    m = s.n
    s.opacity_logits[:] = rng.uniform(-2.0, 7.0, size=m).astype(np.float32)
    s.sh[:, 0, :] = rng.uniform(-3.0, 1.5, size=(m, 3)).astype(np.float32)
    k = int(frac_beyond * m)
    idx = rng.choice(m, size=k, replace=False)
    z = rng.uniform(1.0, 3.0, size=k)
    lim_x = cam.lim_x if math.isfinite(cam.lim_x) else 1.3 * (0.5 * cam.width) / cam.fx
    lim_y = cam.lim_y if math.isfinite(cam.lim_y) else 1.3 * (0.5 * cam.height) / cam.fy
    side = rng.integers(0, 3, size=k)  # 0: beyond in x, 1: in y, 2: both
    tx = np.where(side != 1, rng.choice([-1.0, 1.0], size=k) * lim_x * rng.uniform(1.05, 1.4, size=k),
                  rng.uniform(-0.5, 0.5, size=k) * lim_x)
    ty = np.where(side != 0, rng.choice([-1.0, 1.0], size=k) * lim_y * rng.uniform(1.05, 1.4, size=k),
                  rng.uniform(-0.5, 0.5, size=k) * lim_y)
    pc = np.stack([tx * z, ty * z, z], 1)
    R, t = cam.R.astype(np.float64), cam.t.astype(np.float64)
    s.means[idx] = ((pc - t) @ R).astype(np.float32)   # P = R^T (p_c - t)
    # 3-sigma footprint of ~0.3 lim z: reaches well inside the image from beyond the clamp
    s.log_scales[idx] = np.log(0.12 * lim_x * z[:, None] * rng.uniform(0.8, 1.25, size=(k, 3))).astype(np.float32)
    s.meta = dict(s.meta, edge=True, beyond=idx)
    return s


def densify_samples(n: int, seed: int) -> np.ndarray:
    """Standard-normal samples [n][2][3] float32: the randomness densify draws (one offset per
    clone, two per split), generated here and passed to both sides as an input."""
    rng = np.random.default_rng(np.random.PCG64(seed))
    return rng.normal(size=(n, 2, 3)).astype(np.float32)


def make_keypoints(cam: Camera, n: int, seed: int, active_frac: float = 0.3):
    """Synthetic keyframe features for geometry-based densification: n keypoint
    pixels (uniform, rounded pixel inside the image), an `active` flag (fraction active_frac,
    PAPER.md:231 "less than 30% ... are active"), a smooth depth map in [0.8, 4] m with 5 % invalid
    (0) pixels, the active keypoints' depths read from it, and a smooth keyframe image."""
    rng = np.random.default_rng(np.random.PCG64(seed))
    W, H = cam.width, cam.height
    uv = rng.uniform([0.0, 0.0], [W - 1.0, H - 1.0], size=(n, 2)).astype(np.float32)
    active = (rng.uniform(size=n) < active_frac).astype(np.int32)
    y, x = np.mgrid[0:H, 0:W].astype(np.float64)
    depth = 2.4 + 0.8 * np.sin(x / W * 3.0 + rng.uniform(0, 6)) * np.cos(y / H * 2.0 + rng.uniform(0, 6))
    depth += 0.4 * (x / W) - 0.2 * (y / H)
    depth = np.clip(depth, 0.8, 4.0).astype(np.float32)
    depth[rng.uniform(size=(H, W)) < 0.05] = 0.0
    px = np.rint(uv[:, 0]).astype(int)
    py = np.rint(uv[:, 1]).astype(int)
    kp_depth = np.where(active == 1, np.maximum(depth[py, px], 0.8), 0.0).astype(np.float32)
    image = noise_image(H, W, seed + 17)
    return uv, active, kp_depth, depth, image
