"""Generate tests/golden/*.npz from the UNMODIFIED reference library
(oracle/_ref/libpegrad_ref.so, compiled from /root/reference/proj by
oracle/Makefile). Run here, where the reference sources exist:

    python tests/golden/gen_golden.py

Every fixture is produced by the reference's own public API: models::build,
io::synth_for_model, GradEngine<T>::compute (per-example grads + global
norms), gaussian<T>, dpsgd_step. The noise-free clipped sum is assembled in
fp64 from the reference's fp64 per-example stacks and norms
(sum_i min(1, C/||g_i||) g_i, dpsgd.cpp:54-99,277-307).
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402

CONFIGS = [
    # name, builder, batch, strategy, clip, keep every k-th clipped-sum element
    ("logreg", lambda: O.build_desc(O.LOGREG), 64, O.OUTER, 1.0, 1),
    ("fcnn", lambda: O.build_desc(O.FCNN), 32, O.VMAP, 1.0, 1),
    ("fcnn_104_50_2", lambda: O.custom_desc(O.FCNN, [(0, 104, 50, 0, 1, 0), (6, 0, 0, 0, 1, 0),
                                                    (0, 50, 2, 0, 1, 0)], (104,), 2),
     32, O.VMAP, 1.0, 1),
    ("mnist_cnn", lambda: O.build_desc(O.MNIST_CNN), 256, O.GROUPCONV, 1.0, 1),
    ("cifar_cnn", lambda: O.build_desc(O.CIFAR_CNN), 2, O.GROUPCONV, 0.5, 13),
    ("embed_small", lambda: O.build_desc(O.EMBED, seq_len=16, vocab=50, hidden=8), 8, O.JACMM,
     0.05, 1),
]


# Full-size fixtures (BASELINE configs 4 and 5 at their stated batch): norms,
# clip count and a strided sample of the fp64 clipped sum, from the
# reference's fp64 GradEngine::compute. About a minute; generated on request:
#     python tests/golden/gen_golden.py full
# clip: near the median norm, so about half the examples clip.
FULL = [
    ("cifar_cnn_b256", lambda: O.build_desc(O.CIFAR_CNN), 256, O.GROUPCONV, None, 11),
    ("embed_b512", lambda: O.build_desc(O.EMBED, hidden=100), 512, O.JACMM, None, 17),
]


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def full():
    assert O.ref_available(), "build the reference first: make -C oracle ref"
    for name, mk, B, strat, C, every in FULL:
        d = mk()
        p64 = O.ref_init_params(d, 0)
        x64, y64 = O.ref_synth(d, B, 0)
        x32, y32 = O.ref_synth(d, B, 0, np.float32)
        R = O.RefModel(d, strat, B, p64)
        stacks, norms = R.per_example(x64, y64)
        del R
        if C is None:
            # near the median, in the widest gap between consecutive norms of
            # the middle fifth: no example sits within fp32 noise of C
            srt = np.sort(norms)
            lo, hi = int(0.4 * B), int(0.6 * B)
            k = lo + int(np.argmax(np.diff(srt[lo:hi + 1])))
            C = float(0.5 * (srt[k] + srt[k + 1]))
        s = np.where(norms > C, C / norms, 1.0)
        parts, off = [], 0
        for n in d.blocks:
            blk = stacks[off: off + B * n].reshape(B, n)
            parts.append(s @ blk)  # sum_i s_i g_i, fp64
            off += B * n
        del stacks
        clipped_sum = np.concatenate(parts)
        nclip = int((norms > C).sum())
        # the reference's own fp32 build on the same inputs: its fp32 stacks
        # and norms, clip factors and the views path's fp32 ascending sum
        # (dpsgd.cpp:277-307); its per-block normwise error against the fp64
        # sum (on the sample) is the accuracy an fp32 implementation reaches
        p32 = O.ref_init_params(d, 0, np.float32)
        R32 = O.RefModel(d, strat, B, p32, np.float32)
        st32, n32 = R32.per_example(x32, y32)
        del R32
        s32 = np.where(n32 > np.float32(C), np.float32(C) / n32, np.float32(1)).astype(np.float32)
        f32_err, f32_norm_err, off = [], float(np.max(np.abs(n32 - norms) / norms)), 0
        for n in d.blocks:
            blk = st32[off: off + B * n].reshape(B, n)
            acc = np.zeros(n, np.float32)
            for i in range(B):
                acc = acc + blk[i] * s32[i]
            f32_err.append(acc)
            off += B * n
        del st32
        f32_sum = np.concatenate(f32_err).astype(np.float64)[::every]
        want = clipped_sum[::every]
        rel, off = [], 0
        for n in d.blocks:
            lo, hi = -(-off // every), -(-(off + n) // every)
            den = np.linalg.norm(want[lo:hi])
            rel.append(np.linalg.norm(f32_sum[lo:hi] - want[lo:hi]) / den if den > 0 else 0.0)
            off += n
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), norms=norms, clip_scales=s,
                            ref_f32_block_rel=np.array(rel), ref_f32_norm_rel=f32_norm_err,
                            clipped_count=np.int64(nclip), clipped_sum=clipped_sum[::every],
                            every=np.int64(every), blocks=np.array(d.blocks, np.int64),
                            B=np.int64(B), clip=np.float64(C), x_sha=np.array(digest(x32)),
                            y_sha=np.array(digest(y32)))
        print(name, "B", B, "P", d.param_count, "C", C, "clipped", nclip, "norm0", norms[0])


def main():
    assert O.ref_available(), "build the reference first: make -C oracle ref"
    for name, mk, B, strat, C, every in CONFIGS:
        d = mk()
        p64 = O.ref_init_params(d, 0)
        p32 = O.ref_init_params(d, 0, np.float32)
        x64, y64 = O.ref_synth(d, B, 0)
        x32, y32 = O.ref_synth(d, B, 0, np.float32)
        R = O.RefModel(d, strat, B, p64)
        stacks, norms = R.per_example(x64, y64)
        blocks = O.split_stacks(d, stacks, B)
        s = np.where(norms > C, C / norms, 1.0)
        clipped_sum = np.concatenate([(blk * s[:, None]).sum(axis=0) for blk in blocks])
        nclip = int((norms > C).sum())
        out = dict(norms=norms, clip_scales=s, clipped_count=np.int64(nclip),
                   clipped_sum=clipped_sum[::every], every=np.int64(every),
                   blocks=np.array(d.blocks, np.int64), B=np.int64(B), clip=np.float64(C),
                   init_sha=np.array(digest(p32)), x_sha=np.array(digest(x32)),
                   y_sha=np.array(digest(y32)), init64_head=p64[:64])
        if name == "mnist_cnn":
            # one reference fp32 step at C=1, sigma=1.1, lr=0.1, seed 0, step 0
            R32 = O.RefModel(d, strat, B, p32, np.float32)
            n32, c32 = R32.step(x32, y32, 1.0, 1.1, 0.1, 1, 0, 0)
            out.update(step_params_f32=R32.params(), step_norms_f32=n32,
                       step_clipped=np.int64(c32),
                       noise_f32=np.concatenate([O.ref_gaussian(0, O.noise_stream(0, p), n,
                                                                np.float32)
                                                 for p, n in enumerate(d.blocks)]))
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(name, "B", B, "P", d.param_count, "clipped", nclip, "norm0", norms[0])
    # reference KAT anchors: splitmix values and the first normals of stream 2^32
    np.savez_compressed(os.path.join(HERE, "rng.npz"),
                        rng_value_at_0=np.array([0x618640d511ea0c16, 0x8858072c497acfb9],
                                                np.uint64),
                        gauss_f64=O.ref_gaussian(0, 1 << 32, 1001),
                        gauss_f32=O.ref_gaussian(0, 1 << 32, 1001, np.float32),
                        gauss_f32_odd=O.ref_gaussian(99, 7, 7, np.float32))


if __name__ == "__main__":
    full() if sys.argv[1:] == ["full"] else main()
