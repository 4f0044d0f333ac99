"""Measure the FP64-pipe instruction count of CUDA's own libdevice routines on
their main (fast) path: compile one-call kernels for sm_100a, count FP64 SASS
(DFMA/DMUL/DADD/DSETP/DMNMX and *.F64 conversions/rounding) up to the first
EXIT.  These counts define the algorithmic FP64 cost table of bench.py /
DESIGN.md §5 (what a plain, standard implementation of the method issues)."""
import os
import re
import subprocess
import sys
import tempfile

SRC = r'''
extern "C" __global__ void k_log(const double* x, double* y) { int i = threadIdx.x; y[i] = log(x[i]); }
extern "C" __global__ void k_exp(const double* x, double* y) { int i = threadIdx.x; y[i] = exp(x[i]); }
extern "C" __global__ void k_sqrt(const double* x, double* y) { int i = threadIdx.x; y[i] = sqrt(x[i]); }
extern "C" __global__ void k_div(const double* x, double* y) { int i = threadIdx.x; y[i] = x[i] / x[i + 64]; }
extern "C" __global__ void k_tanh(const double* x, double* y) { int i = threadIdx.x; y[i] = tanh(x[i]); }
extern "C" __global__ void k_sincospi(const double* x, double* y) { int i = threadIdx.x; double s, c; sincospi(x[i], &s, &c); y[i] = s; y[i + 64] = c; }
extern "C" __global__ void k_cospi(const double* x, double* y) { int i = threadIdx.x; y[i] = cospi(x[i]); }
extern "C" __global__ void k_u2d(const unsigned long long* x, double* y) { int i = threadIdx.x; y[i] = (double)x[i]; }
'''
FP64 = ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX", "DSET")


def main():
    d = tempfile.mkdtemp()
    cu = os.path.join(d, "ld.cu")
    open(cu, "w").write(SRC)
    cubin = os.path.join(d, "ld.cubin")
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-O3", "-cubin", cu, "-o", cubin])
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", cubin], capture_output=True,
                          text=True).stdout
    out = {}
    for f in re.split(r"\n\s+Function : ", sass)[1:]:
        name = f.split("\n")[0].strip()[2:]
        n = 0
        for ins in re.findall(r"/\*[0-9a-f]{4}\*/\s+(.*?);", f):
            op = ins.split()[1] if ins.startswith("@") else ins.split()[0]
            base = op.split(".")[0]
            if op.startswith("EXIT"):
                break
            if base in FP64 or (base in ("FRND", "F2F", "I2F", "F2I") and "F64" in op):
                n += 1
        out[name] = n
    for k, v in sorted(out.items()):
        print(f"{k:10s} {v}")
    return out


if __name__ == "__main__":
    main()
