"""Generate the golden fixtures under tests/golden/ from the UNMODIFIED reference.

Run here (where /root/reference exists): ``python tests/golden/make_golden.py``.
Everything is produced through oracle/_ref (the reference headers compiled by
oracle/Makefile): the bundled desk scene is parsed with the reference's own
loaders (io.hpp), images/stats come from render_scene, hit sets from
particle_ray_footprint, knots from quantize_particle, merged pieces from
accumulate<Int128>.  The GPU box has no /root/reference; the tests read these
files instead.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from tests import helpers as H  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def cam_fields(cam: ref.Camera):
    return dict(mode=np.array(cam.mode), position=np.array(cam.position),
                look_at=np.array(cam.look_at), up=np.array(cam.up), width=np.array(cam.width),
                height=np.array(cam.height), fov_deg=np.array(cam.fov_deg),
                ortho_height=np.array(cam.ortho_height), near=np.array(cam.near),
                far=np.array(cam.far))


def digest(*arrays):
    import hashlib
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return np.array(h.hexdigest())


def scene_golden(name, ps, cam, tf, lut_path, bg, full=True):
    rl = ref.Lut(lut_path)
    ds = ref.dataset_stats(ps, rl)
    qc = ref.choose_quanta(rl, ds)
    rgb, st, _, bits = ref.render_robust(ps, cam, tf, rl, qc, ds, 0.0, bg)
    ray, pid, lam, tchi = ref.footprint(ps, cam, rl.q)
    out = dict(particles=ps, tf=tf, background=np.array(bg, np.float64), lut=os.path.basename(lut_path),
               rgb=rgb, accum_bits=np.array(bits), tau=np.array(qc.tau), sigma=np.array(qc.sigma),
               h_r=np.array(ds.h_r), a_max=np.array(ds.a_max), phi_repr=np.array(ds.phi_repr),
               hit_ray=ray, hit_pidx=pid, hit_lam=lam, hit_tchi=tchi,
               **{"cam_" + k: v for k, v in cam_fields(cam).items()},
               **{"stat_" + k: np.array(v) for k, v in st.items()})
    # per-hit knots (quantize_particle<int64_t>)
    kt, kb, kn = [], [], []
    for r, p, l, t in zip(ray, pid, lam, tchi):
        tt, bb = ref.quantize(ps[p], int(r), float(t), float(l), rl, qc, int(p))
        kn.append(len(tt))
        kt.append(tt)
        kb.append(bb)
    knot_count = np.array(kn, np.int32)
    knot_t = np.concatenate(kt) if kt else np.zeros(0, np.int64)
    knot_b = np.concatenate(kb) if kb else np.zeros((0, 7), np.int64)
    pl = ref.pipeline(ps, cam, rl, qc)
    if full:
        out.update(knot_count=knot_count, knot_t=knot_t, knot_b=knot_b)
        for k in ("rays", "piece_off", "piece_t", "piece_a", "piece_fits", "ray_ops"):
            out["pl_" + k] = pl[k]
    else:
        # large scenes: size-independent checks (counts + SHA-256 of the exact arrays)
        out.update(n_knots=np.array(len(knot_t)), n_pieces=np.array(len(pl["piece_t"])),
                   digest_knots=digest(knot_count, knot_t, knot_b),
                   digest_pieces=digest(pl["rays"], pl["piece_off"], pl["piece_t"], pl["piece_a"]),
                   pl_rays=pl["rays"], pl_piece_off=pl["piece_off"])
        for k in ("hit_ray", "hit_pidx", "hit_lam", "hit_tchi"):
            out[k] = out[k][:0]
        out["digest_hits"] = digest(ray, pid, lam, tchi)
        out["n_hits"] = np.array(len(ray))
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
    print(name, {k: (v.shape if hasattr(v, "shape") else v) for k, v in out.items() if k in (
        "rgb", "hit_ray", "knot_t", "pl_piece_t")}, st)


def config1_golden():
    """BASELINE.json config 1 (1e5-particle blob, 256^2, K=4 D=3 N=1024, w64), the
    one configuration the reference renders whole: the full frame from
    render_scene<int64_t>, its RenderStats, a digest of the full hit set and the
    per-ray records of rp_render_region over the whole frame (knots, pieces,
    hits, residual/termination flags and the checksum of every ray's
    accumulate<Int128> FieldPieces, sphray_piece_mix)."""
    ps = ref.generate_scene(1)
    lut_path = H.lut_path(4, 3, 1024)
    rl = ref.Lut(lut_path)
    ds = ref.dataset_stats(ps, rl)
    qc = ref.choose_quanta(rl, ds)
    cam = ref.Camera(**H.synth_camera_kwargs(256, 256))
    rgb, st, _, bits = ref.render_robust(ps, cam, H.SYNTH_TF, rl, qc, ds)
    _, rec, rst, _, _ = ref.render_region(ps, cam, H.SYNTH_TF, rl, qc, st["step"], 0, 0, 256, 256)
    for k in ("knots", "rays_touched", "int_ops", "residual_failures"):
        assert rst[k] == st[k], k
    ray, pid, lam, tchi = ref.footprint(ps, cam, rl.q)
    o = np.lexsort((pid, ray))  # ray-major, as the GPU dump returns them
    out = dict(particles_digest=digest(ps), n_particles=np.array(len(ps)), lut=os.path.basename(lut_path),
               rgb=rgb, accum_bits=np.array(bits), tau=np.array(qc.tau), sigma=np.array(qc.sigma),
               h_r=np.array(ds.h_r), a_max=np.array(ds.a_max),
               n_hits=np.array(len(ray)), digest_hits=digest(ray[o], pid[o], lam[o], tchi[o]),
               rec_checksum=rec["piece_checksum"], rec_knots=rec["knots"], rec_pieces=rec["pieces"],
               rec_hits=rec["hits"], rec_flags=rec["flags"],
               **{"cam_" + k: v for k, v in cam_fields(cam).items()},
               **{"stat_" + k: np.array(v) for k, v in st.items()})
    np.savez_compressed(os.path.join(OUT, "config1.npz"), **out)
    print("config1", st, "hits", len(ray), "bits", bits)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "config1":
        config1_golden()
        return
    # the bundled example scene, parsed by the reference's io.hpp loaders
    ps = ref.load_particles(f"{H.REF_DATA}/desk_scene.csv")
    tf = ref.load_tf(f"{H.REF_DATA}/tf.csv")
    cam = ref.load_camera(f"{H.REF_DATA}/camera.json")
    scene_golden("desk", ps, cam, tf, H.lut_path(4, 3, 1024), (0.0, 0.0, 0.0), full=False)

    # raycast_tests.cpp:390-443 scene
    ps = H.random_cloud(H.MT19937_64(31337), 120, 1.6, -1.2, 1.2)
    scene_golden("render_test", ps, ref.Camera(**H.render_test_camera_kwargs()), H.TEST_TF,
                 H.lut_path(4, 3, 16), (0.01, 0.02, 0.03))

    # raycast_tests.cpp:152-199 footprint scenes
    ps = H.random_cloud(H.MT19937_64(5150), 40, 2.5, -1.0, 2.0)
    ortho, pin = H.footprint_test_cameras()
    scene_golden("footprint_ortho", ps, ref.Camera(**ortho), H.TEST_TF, H.lut_path(4, 3, 16), (0, 0, 0))
    scene_golden("footprint_pinhole", ps, ref.Camera(**pin), H.TEST_TF, H.lut_path(4, 3, 16), (0, 0, 0))
    ps = H.random_cloud(H.MT19937_64(77), 60, 2.0, -4.0, 4.2)
    cam = ref.Camera(mode="pinhole", width=24, height=18, position=(0, 0, 4), look_at=(0, 0, 0),
                     near=2.0, far=6.5)
    scene_golden("clip_planes", ps, cam, H.TEST_TF, H.lut_path(4, 3, 16), (0, 0, 0))

    # odd K and other (K, D) through the mirror closure (lut_tests.cpp:134-169 pairs)
    for K, D, N in ((3, 2, 64), (5, 4, 64), (2, 3, 64), (6, 6, 32), (7, 5, 32)):
        ps = H.random_cloud(H.MT19937_64(1000 + K * 10 + D), 50, 1.6, -1.2, 1.2)
        scene_golden(f"kd_K{K}_D{D}", ps, ref.Camera(**H.render_test_camera_kwargs()), H.TEST_TF,
                     H.lut_path(K, D, N), (0.0, 0.0, 0.0))

    # a small blob of the synthetic generator family (config-1 shape at 48^2)
    import paper_2401_02896_b200 as S
    ps = S.generate_scene(1, n=3000)
    scene_golden("blob3000", ps, ref.Camera(**H.synth_camera_kwargs(48, 48)), H.SYNTH_TF,
                 H.lut_path(4, 3, 1024), (0.0, 0.0, 0.0), full=False)


if __name__ == "__main__":
    main()
