"""Tensor-core and CUDA-core peaks the fp32-accurate kernels are judged
against ("TF32 and FP32 peaks are not in MEASURED_PEAKS.json --
measure them on the box"). cuBLAS through torch.matmul, 8192^3, CUDA events,
best of 10 after warm-up:

  tf32  : fp32 operands, allow_tf32 = True (tcgen05 kind::tf32 GEMM)
  fp32  : allow_tf32 = False (CUDA-core SGEMM: the FFMA roofline)
  bf16  : the MEASURED_PEAKS.json denominator, re-measured beside them

Writes one JSON object (stdout, and profiles/<tag>_peaks.json when a tag is
given). The 3xTF32 effective ceiling of an fp32-accurate tensor-core kernel
is tf32 / 3."""
import json
import os
import sys

import torch


def best_tflops(dtype, tf32, n=8192, reps=10):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    torch.backends.cudnn.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    return 2 * n ** 3 / best / 1e12


def main():
    props = torch.cuda.get_device_properties(0)
    out = {
        "gpu": props.name, "sms": props.multi_processor_count,
        "tf32_tflops": best_tflops(torch.float32, True),
        "fp32_sgemm_tflops": best_tflops(torch.float32, False),
        "bf16_tflops": best_tflops(torch.bfloat16, False),
        "how": "torch.matmul 8192^3 (2 N^3 flop), best of 10 after 3 warm-ups, CUDA events; "
               "tf32 = fp32 with allow_tf32, fp32 = allow_tf32 off",
    }
    try:
        import pynvml as N
        N.nvmlInit()
        h = N.nvmlDeviceGetHandleByIndex(0)
        mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        out["sm_max_mhz"] = mhz
        out["fp32_ffma_nominal_tflops"] = props.multi_processor_count * 128 * 2 * mhz * 1e6 / 1e12
    except Exception:
        pass
    out["tf32x3_effective_tflops"] = out["tf32_tflops"] / 3
    line = json.dumps(out)
    print(line)
    if len(sys.argv) > 1:
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        with open(os.path.join(root, "profiles", f"{sys.argv[1]}_peaks.json"), "w") as f:
            f.write(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
