// Host-call latency anatomy from C++ (no Python in the loop): one 56^2 k3 s1 p1
// layer (DenseNet-sized), one image, page-locked buffers.  Prints per-call
// microseconds for the pieces of spconv_convolve_host and for alternatives.
// Build: nvcc -O2 -std=c++17 -Iinclude scripts/probe_host_lat.cu -o gpurun_out/probe_host_lat \
//          -Lpaper_2411_19419_b200 -lspconv_b200 -lcuda -Xlinker -rpath=$PWD/paper_2411_19419_b200
#include <cuda.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <functional>
#include <vector>

#include "spconv_b200.h"

static double per_call(const std::function<void()>& f, int n = 4000) {
    for (int i = 0; i < 200; ++i) f();
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i) f();
    auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double, std::micro>(t1 - t0).count() / n;
}

__global__ void empty_kernel() {}

int main(int argc, char** argv) {
    int m = 56, n = 56, k = 3;
    if (argc > 1) m = n = atoi(argv[1]);
    if (argc > 2) k = atoi(argv[2]);
    cudaSetDevice(0);
    cudaFree(0);
    std::vector<float> taps(k * k);
    for (int i = 0; i < k * k; ++i) taps[i] = 0.25f * (i + 1);
    spconv_csr* h = nullptr;
    if (spconv_build_csr(m, n, k, 1, k / 2, taps.data(), 0, nullptr, &h)) return printf("build: %s\n", spconv_last_error()), 1;
    cudaDeviceSynchronize();
    const size_t cols = (size_t)m * n, rows = cols;
    float *xh, *yh, *xd, *yd, *yhd;
    cudaHostAlloc(&xh, cols * 4, cudaHostAllocMapped);
    cudaHostAlloc(&yh, rows * 4, cudaHostAllocMapped);
    cudaHostGetDevicePointer(&yhd, yh, 0);
    float* xhd;
    cudaHostGetDevicePointer(&xhd, xh, 0);
    cudaMalloc(&xd, cols * 4);
    cudaMalloc(&yd, rows * 4);
    for (size_t i = 0; i < cols; ++i) xh[i] = (float)(i % 7);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    volatile int* flag;
    cudaHostAlloc((void**)&flag, 64, cudaHostAllocMapped);
    CUdeviceptr flag_d;
    cuMemHostGetDevicePointer(&flag_d, (void*)flag, 0);
    int seq = 0;

    printf("%d^2 k%d\n", m, k);
    printf("  sync idle stream          %7.2f us\n", per_call([&] { cudaStreamSynchronize(st); }));
    printf("  empty kernel + sync       %7.2f us\n", per_call([&] { empty_kernel<<<1, 32, 0, st>>>(); cudaStreamSynchronize(st); }));
    printf("  H2D + sync                %7.2f us\n",
           per_call([&] { cudaMemcpyAsync(xd, xh, cols * 4, cudaMemcpyHostToDevice, st); cudaStreamSynchronize(st); }));
    printf("  spmv dev + sync           %7.2f us\n", per_call([&] { spconv_spmv(h, xd, yd, st); cudaStreamSynchronize(st); }));
    printf("  spmv dev->host y + sync   %7.2f us\n", per_call([&] { spconv_spmv(h, xd, yhd, st); cudaStreamSynchronize(st); }));
    printf("  spmv host x,y + sync      %7.2f us\n", per_call([&] { spconv_spmv(h, xhd, yhd, st); cudaStreamSynchronize(st); }));
    printf("  H2D + spmv(y host) + sync %7.2f us\n", per_call([&] {
               cudaMemcpyAsync(xd, xh, cols * 4, cudaMemcpyHostToDevice, st);
               spconv_spmv(h, xd, yhd, st);
               cudaStreamSynchronize(st);
           }));
    printf("  H2D + spmv + D2H + sync   %7.2f us\n", per_call([&] {
               cudaMemcpyAsync(xd, xh, cols * 4, cudaMemcpyHostToDevice, st);
               spconv_spmv(h, xd, yd, st);
               cudaMemcpyAsync(yh, yd, rows * 4, cudaMemcpyDeviceToHost, st);
               cudaStreamSynchronize(st);
           }));
    printf("  H2D+spmv+writeflag+spin   %7.2f us\n", per_call([&] {
               cudaMemcpyAsync(xd, xh, cols * 4, cudaMemcpyHostToDevice, st);
               spconv_spmv(h, xd, yhd, st);
               ++seq;
               cuStreamWriteValue32(st, flag_d, (cuuint32_t)seq, 0);
               while (*flag != seq) {
               }
           }));
    cudaStreamSynchronize(st);
    // the same three steps captured once as a graph
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    cudaMemcpyAsync(xd, xh, cols * 4, cudaMemcpyHostToDevice, st);
    spconv_spmv(h, xd, yhd, st);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    printf("  graph(H2D+spmv) + sync    %7.2f us\n", per_call([&] { cudaGraphLaunch(ge, st); cudaStreamSynchronize(st); }));
    printf("  convolve_host (pinned)    %7.2f us\n", per_call([&] { spconv_convolve_host(h, xh, yh, 1); }));
    std::vector<float> xq(cols), yq(rows);
    printf("  convolve_host (pageable)  %7.2f us\n", per_call([&] { spconv_convolve_host(h, xq.data(), yq.data(), 1); }));
    spconv_set_option("stage", "window");
    printf("  [window] spmv dev + sync  %7.2f us\n", per_call([&] { spconv_spmv(h, xd, yd, st); cudaStreamSynchronize(st); }));
    printf("  [window] host x,y + sync  %7.2f us\n", per_call([&] { spconv_spmv(h, xhd, yhd, st); cudaStreamSynchronize(st); }));
    printf("  [window] H2D+spmv(yh)+sync%7.2f us\n", per_call([&] {
               cudaMemcpyAsync(xd, xh, cols * 4, cudaMemcpyHostToDevice, st);
               spconv_spmv(h, xd, yhd, st);
               cudaStreamSynchronize(st);
           }));
    spconv_set_option("stage", "auto");
    printf("  spmv dev + sync (again)   %7.2f us\n", per_call([&] { spconv_spmv(h, xd, yd, st); cudaStreamSynchronize(st); }));
    {
        float ms = 0;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int v = 0; v < 3; ++v) {
            const float* X = v == 2 ? xhd : xd;
            float* Y = v == 0 ? yd : yhd;
            if (v == 2) spconv_set_option("stage", "window");
            for (int i = 0; i < 50; ++i) spconv_spmv(h, X, Y, st);
            cudaEventRecord(e0, st);
            for (int i = 0; i < 200; ++i) spconv_spmv(h, X, Y, st);
            cudaEventRecord(e1, st);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            printf("  device time per spmv (%s) %7.2f us\n", v == 0 ? "dev" : v == 1 ? "y host" : "win x,y host", ms * 1e3 / 200);
        }
        spconv_set_option("stage", "auto");
    }
    cudaPointerAttributes a{};
    printf("  cudaPointerGetAttributes  %7.2f us\n", per_call([&] { cudaPointerGetAttributes(&a, yh); }));
    int dev;
    printf("  cudaGetDevice+Set         %7.2f us\n", per_call([&] { cudaGetDevice(&dev); cudaSetDevice(dev); }));
    printf("  launch only (spmv)        %7.2f us\n", per_call([&] { spconv_spmv(h, xd, yd, st); }, 2000));
    cudaStreamSynchronize(st);
    printf("  launch only (empty)       %7.2f us\n", per_call([&] { empty_kernel<<<1, 32, 0, st>>>(); }, 2000));
    cudaStreamSynchronize(st);
    printf("  memcpyAsync only (H2D)    %7.2f us\n", per_call([&] { cudaMemcpyAsync(xd, xh, cols * 4, cudaMemcpyHostToDevice, st); }, 2000));
    cudaStreamSynchronize(st);
    spconv_csr_free(h);
    return 0;
}
