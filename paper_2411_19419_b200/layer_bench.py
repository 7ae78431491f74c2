"""DenseNet121 layer-table bench on the GPU -- the paper's Table 1 protocol
(reference harness inc/bench.hpp:174-349).

Per layer of ``densenet121_layers()`` (123 single-channel shapes, pooling
layers run as random-kernel convolutions as the paper does), the transform is
built once on the device (build time reported separately, as
``build_time_us``) and the apply is timed over ``trials`` trials:

* ``device``: one SpMV on a device-resident image, timed as a CUDA graph of
  ``graph_reps`` back-to-back launches replayed per trial (launch overhead
  amortised the way a GPU-resident network would see it); the same for the
  layer as a CSC transform (the reference's CSC-SpMV column: the CSC storage
  itself is read), its output checked equal to the CSR one;
* ``host``: the reference's call shape -- an fp32 image in pinned host memory,
  H2D + SpMV + D2H through the C ABI (``spconv_convolve_host``) per trial.

Each layer's device output is cross-checked before timing against a float64
direct convolution (the reference's ``direct_conv``, inc/reference.hpp:41-61,
restated in numpy) within the north-star tolerance
|y - ref| <= 1e-5 * sum|w x|, as the reference harness cross-checks its
methods (inc/bench.hpp:218-233).  Totals are sums of per-layer means and the
root-sum-square of per-layer SEMs (inc/bench.hpp:284-349).  A whole-network
graph (all 123 layers back to back) gives the end-to-end pass time, and the
grouped apply (``spmv_group``: the 123 layers in ONE launch; on host arrays
``convolve_group``: one packed copy each way) the same pass without the
per-layer launches.
"""
from __future__ import annotations

import math
import statistics
import time
from typing import Dict, List

import numpy as np

from .layers import LayerConfig, densenet121_layers

TOL = 1e-5


def direct_conv_f64(a: np.ndarray, w: np.ndarray, s: int, p: int):
    """Padded, strided correlation in float64 plus sum|w x| per output."""
    m, n = a.shape
    k = w.shape[0]
    ap = np.zeros((m + 2 * p, n + 2 * p))
    ap[p:p + m, p:p + n] = a
    mo, no = (m + 2 * p - k) // s + 1, (n + 2 * p - k) // s + 1
    out = np.zeros((mo, no))
    mag = np.zeros((mo, no))
    for j in range(k):
        for i in range(k):
            win = ap[j:j + s * (mo - 1) + 1:s, i:i + s * (no - 1) + 1:s]
            out += w[j, i] * win
            mag += abs(w[j, i]) * np.abs(win)
    return out, mag


def _stats(us: List[float]):
    mean = statistics.fmean(us)
    sem = statistics.stdev(us) / math.sqrt(len(us)) if len(us) > 1 else 0.0
    return mean, sem


def run_table_bench(layers: List[LayerConfig] = None, trials: int = 100, warmup: int = 10,
                    graph_reps: int = 20, seed: int = 42, device: int = 0) -> Dict:
    import torch

    from . import ConvSpec, Kernel, build_transform, convolve_group, spmm_f64, spmv, spmv_group
    from . import lib, _check

    layers = layers or densenet121_layers()
    dev = torch.device("cuda", device)
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(dev)
    rows = []
    graphs_all = []
    keep = []
    with torch.cuda.stream(stream):
        for li, L in enumerate(layers):
            rng = np.random.default_rng([seed, li])
            a = rng.standard_normal((L.m, L.n)).astype(np.float32)
            w = rng.standard_normal((L.k, L.k)).astype(np.float32)
            spec = ConvSpec(L.m, L.n, L.k, L.s, L.p)
            # one-time build, device-timed (a GPU sleep covers the host enqueue)
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(1_000_000)
            e0.record(stream)
            t = build_transform(Kernel(L.k, w.reshape(-1)), spec, device=device, stream=stream)
            e1.record(stream)
            x = torch.from_numpy(a.reshape(-1)).to(dev)
            y = torch.empty(t.rows, dtype=torch.float32, device=dev)
            spmv(t, x, y, stream=stream)
            torch.cuda.synchronize(dev)
            build_us = e0.elapsed_time(e1) * 1e3
            # cross-check (inc/bench.hpp:218-233)
            ref, mag = direct_conv_f64(a.astype(np.float64), w.astype(np.float64), L.s, L.p)
            got = y.cpu().numpy().astype(np.float64).reshape(ref.shape)
            dev_max = float(np.max(np.abs(got - ref) - TOL * mag - 1e-30))
            if dev_max > 0:
                raise RuntimeError(f"cross-check failed for layer '{L.name}'")
            kernel_name = t.last_kernel
            # device-resident: graph of graph_reps launches, replayed per trial
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for _ in range(graph_reps):
                    spmv(t, x, y, stream=stream)
            for _ in range(warmup):
                g.replay()
            torch.cuda.synchronize(dev)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(trials)]
            for i in range(trials):
                ev[i][0].record(stream)
                g.replay()
                ev[i][1].record(stream)
            torch.cuda.synchronize(dev)
            dev_us = [a_.elapsed_time(b_) * 1e3 / graph_reps for a_, b_ in ev]
            # the same layer as a CSC transform (the reference's CSC-SpMV column):
            # the CSC storage itself is read (csc_gather), cross-checked bit for bit
            tc = build_transform(Kernel(L.k, w.reshape(-1)), spec, layout=1, device=device, stream=stream)
            yc = torch.empty(t.rows, dtype=torch.float32, device=dev)
            spmv(tc, x, yc, stream=stream)
            torch.cuda.synchronize(dev)
            if not torch.equal(yc, y):
                raise RuntimeError(f"CSC / CSR outputs differ for layer '{L.name}'")
            gc = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gc, stream=stream):
                for _ in range(graph_reps):
                    spmv(tc, x, yc, stream=stream)
            for _ in range(warmup):
                gc.replay()
            torch.cuda.synchronize(dev)
            evc = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(trials)]
            for i in range(trials):
                evc[i][0].record(stream)
                gc.replay()
                evc[i][1].record(stream)
            torch.cuda.synchronize(dev)
            csc_us = [a_.elapsed_time(b_) * 1e3 / graph_reps for a_, b_ in evc]
            csc_kernel = tc.last_kernel
            del gc
            tc.close()
            # host call shape: pinned fp32 image in, fp32 out (H2D + SpMV + D2H)
            xh = torch.from_numpy(a.reshape(1, -1)).pin_memory()
            yh = torch.empty(1, t.rows, dtype=torch.float32).pin_memory()
            for _ in range(warmup):
                _check(lib.spconv_convolve_host(t._h, xh.data_ptr(), yh.data_ptr(), 1))
            host_us = []
            for _ in range(trials):
                h0 = time.perf_counter()
                _check(lib.spconv_convolve_host(t._h, xh.data_ptr(), yh.data_ptr(), 1))
                host_us.append((time.perf_counter() - h0) * 1e6)
            dm, ds = _stats(dev_us)
            hm, hs = _stats(host_us)
            cm, cs_ = _stats(csc_us)
            rows.append(dict(layer=L.name, m=L.m, n=L.n, k=L.k, s=L.s, p=L.p, nnz=t.nnz,
                             kernel=kernel_name, device_mean_us=dm, device_sem_us=ds,
                             host_mean_us=hm, host_sem_us=hs, build_time_us=build_us,
                             csc_kernel=csc_kernel, csc_device_mean_us=cm, csc_device_sem_us=cs_))
            keep.append((t, x, y, g))
            graphs_all.append((t, x, y))
        # whole network: every layer's SpMV back to back in one graph
        gnet = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gnet, stream=stream):
            for t, x, y in graphs_all:
                spmv(t, x, y, stream=stream)
        for _ in range(warmup):
            gnet.replay()
        torch.cuda.synchronize(dev)
        net_us = []
        for _ in range(trials):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            gnet.replay()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            net_us.append(e0.elapsed_time(e1) * 1e3)
        # whole network as ONE grouped launch (spconv_spmv_group): every
        # layer's output checked equal to its own SpMV's, then a graph of
        # graph_reps grouped launches replayed per trial
        ts = [t for t, _, _ in graphs_all]
        xs = [x for _, x, _ in graphs_all]
        yg = [torch.empty_like(y) for _, _, y in graphs_all]
        spmv_group(ts, xs, yg, stream=stream)
        torch.cuda.synchronize(dev)
        for (t, x, y), z in zip(graphs_all, yg):
            if not torch.equal(y, z):
                raise RuntimeError("grouped and per-layer outputs differ")
        ggr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(ggr, stream=stream):
            for _ in range(graph_reps):
                spmv_group(ts, xs, yg, stream=stream)
        for _ in range(warmup):
            ggr.replay()
        torch.cuda.synchronize(dev)
        grp_us = []
        for _ in range(trials):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ggr.replay()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            grp_us.append(e0.elapsed_time(e1) * 1e3 / graph_reps)
        del ggr
    # the whole table end to end through the host-buffer grouped call: the
    # images as numpy arrays in, numpy arrays out (convolve_group)
    imgs = [x.cpu().numpy() for x in xs]
    want = [y.cpu().numpy() for _, _, y in graphs_all]
    got = convolve_group(ts, imgs)
    if not all(np.array_equal(a_.view(np.uint32), b_.view(np.uint32)) for a_, b_ in zip(got, want)):
        raise RuntimeError("host grouped outputs differ from the per-layer SpMVs")
    for _ in range(warmup):
        convolve_group(ts, imgs)
    e2e_py = []
    for _ in range(trials):
        h0 = time.perf_counter()
        convolve_group(ts, imgs)
        e2e_py.append((time.perf_counter() - h0) * 1e6)
    # the C-ABI call itself, its pointer arrays set up once (what a C / C++
    # caller holds): pageable host images in, pageable outputs out
    outs = [np.empty(t.rows, np.float32) for t in ts]
    nl = len(ts)
    H = np.fromiter((t._h.value for t in ts), np.uintp, nl)
    X = np.fromiter((x.__array_interface__["data"][0] for x in imgs), np.uintp, nl)
    Y = np.fromiter((y.__array_interface__["data"][0] for y in outs), np.uintp, nl)
    call = lambda: _check(lib.spconv_convolve_host_group(H.ctypes.data, nl, X.ctypes.data, Y.ctypes.data))  # noqa: E731
    call()
    if not all(np.array_equal(a_.view(np.uint32), b_.view(np.uint32)) for a_, b_ in zip(outs, want)):
        raise RuntimeError("host grouped outputs differ from the per-layer SpMVs")
    for _ in range(warmup):
        call()
    e2e_grp = []
    for _ in range(trials):
        h0 = time.perf_counter()
        call()
        e2e_grp.append((time.perf_counter() - h0) * 1e6)
    # the same in the reference's fp64 arithmetic (spconv_convolve_host_group_f64):
    # outputs checked bit for bit against each layer's own spmm_f64
    imgs64 = [x.astype(np.float64) for x in imgs]
    outs64 = [np.empty(t.rows, np.float64) for t in ts]
    X64 = np.fromiter((x.__array_interface__["data"][0] for x in imgs64), np.uintp, nl)
    Y64 = np.fromiter((y.__array_interface__["data"][0] for y in outs64), np.uintp, nl)
    call64 = lambda: _check(lib.spconv_convolve_host_group_f64(H.ctypes.data, nl, X64.ctypes.data, Y64.ctypes.data))  # noqa: E731
    call64()
    for t, x, y in zip(ts, imgs64, outs64):
        w = spmm_f64(t, torch.from_numpy(x).to(dev)[None])[0].cpu().numpy()
        if not np.array_equal(w.view(np.uint64), y.view(np.uint64)):
            raise RuntimeError("fp64 grouped outputs differ from the per-layer fp64 SpMVs")
    for _ in range(warmup):
        call64()
    e2e_64 = []
    for _ in range(trials):
        h0 = time.perf_counter()
        call64()
        e2e_64.append((time.perf_counter() - h0) * 1e6)
    for t, *_ in keep:
        t.close()
    tot = lambda key: sum(r[key] for r in rows)  # noqa: E731
    rss = lambda key: math.sqrt(sum(r[key] ** 2 for r in rows))  # noqa: E731
    nm, ns = _stats(net_us)
    gm, gs = _stats(grp_us)
    em, es = _stats(e2e_grp)
    pm, ps = _stats(e2e_py)
    fm, fs = _stats(e2e_64)
    return {
        "layers": rows,
        "total_device_us": tot("device_mean_us"), "total_device_sem_us": rss("device_sem_us"),
        "total_csc_device_us": tot("csc_device_mean_us"),
        "total_host_us": tot("host_mean_us"), "total_host_sem_us": rss("host_sem_us"),
        "total_build_us": tot("build_time_us"),
        "network_graph_us": nm, "network_graph_sem_us": ns,
        "network_group_us": gm, "network_group_sem_us": gs,
        "e2e_group_us": em, "e2e_group_sem_us": es,
        "e2e_group_python_us": pm, "e2e_group_python_sem_us": ps,
        "e2e_group_f64_us": fm, "e2e_group_f64_sem_us": fs,
        "trials": trials, "warmup": warmup, "graph_reps": graph_reps,
    }


def markdown(res: Dict, ref: Dict = None) -> str:
    """Per-layer table in the reference report's shape (inc/bench.hpp:318-349)."""
    out = ["| layer | m | n | k | s | p | nnz | device CSR us | sem | device CSC us | host mean us | sem | build us |"
           + (" reference CSR-SpMV us | reference CSC-SpMV us |" if ref else ""),
           "|---|---|---|---|---|---|---|---|---|---|---|---|---|" + ("---|---|" if ref else "")]
    for i, r in enumerate(res["layers"]):
        line = (f"| {r['layer']} | {r['m']} | {r['n']} | {r['k']} | {r['s']} | {r['p']} | {r['nnz']} | "
                f"{r['device_mean_us']:.3f} | {r['device_sem_us']:.3f} | {r['csc_device_mean_us']:.3f} | "
                f"{r['host_mean_us']:.3f} | {r['host_sem_us']:.3f} | {r['build_time_us']:.1f} |")
        if ref:
            line += f" {ref['layers'][i]['CSR-SpMV'][0]:.3f} | {ref['layers'][i]['CSC-SpMV'][0]:.3f} |"
        out.append(line)
    line = (f"| TOTAL | | | | | | | {res['total_device_us']:.3f} | {res['total_device_sem_us']:.3f} | "
            f"{res['total_csc_device_us']:.3f} | {res['total_host_us']:.3f} | {res['total_host_sem_us']:.3f} | "
            f"{res['total_build_us']:.1f} |")
    if ref:
        line += f" {ref['total_csr_us']:.3f} | {ref['total_csc_us']:.3f} |"
    out.append(line)
    return "\n".join(out) + "\n"
