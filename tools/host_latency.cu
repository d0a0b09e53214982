// Floor of the end-to-end host call from C (no Python): metro_route_host_v1 in
// zero-copy and copy mode vs an empty kernel launch + stream sync.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/host_latency tools/host_latency.cu \
//        -Lpaper_2512_09277_b200/_lib -lmetro_b200 -Xlinker -rpath=$PWD/paper_2512_09277_b200/_lib
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "../include/metro_route.h"
#include "../include/metro_serve.h"

__global__ void empty_kernel() {}

static double median(std::vector<double> v) { std::sort(v.begin(), v.end()); return v[v.size() / 2]; }

int main() {
    const int N = 256, G = 8, B = 1024, k = 8, P = B * k;
    // simple placement: expert e on rank e % 8 and, for e < 128, also on (e + 3) % 8
    std::vector<int8_t> A(N * G, 0);
    for (int e = 0; e < N; ++e) { A[e * G + e % G] = 1; if (e < 128) A[e * G + (e + 3) % G] = 1; }
    std::vector<uint32_t> mask(N);
    metro_pack_placement(A.data(), N, G, mask.data());
    uint32_t *dmask; cudaMalloc(&dmask, N * 4); cudaMemcpy(dmask, mask.data(), N * 4, cudaMemcpyHostToDevice);
    int32_t *ids, *out, *pr;
    cudaMallocHost(&ids, P * 4); cudaMallocHost(&out, (8 + G + N) * 4); cudaMallocHost(&pr, P * 4);
    srand(1);
    for (int i = 0; i < P; ++i) ids[i] = (rand() % 64) * ((rand() % 4) + 1) % N;
    void *ws; cudaMalloc(&ws, metro_host_workspace_bytes(P, N, G));
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    auto bench = [&](const char *name, auto fn) {
        for (int i = 0; i < 50; ++i) fn();
        std::vector<double> t;
        for (int i = 0; i < 2000; ++i) {
            auto t0 = std::chrono::high_resolution_clock::now();
            fn();
            auto t1 = std::chrono::high_resolution_clock::now();
            t.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
        }
        printf("%-28s median %.2f us\n", name, median(t));
    };
    bench("empty launch+sync", [&] { empty_kernel<<<1, 32, 0, s>>>(); cudaStreamSynchronize(s); });
    bench("host_v1 zero-copy", [&] {
        int rc = metro_route_host_v1(ids, P, dmask, N, G, ws, out, pr, 0, METRO_HOST_ZEROCOPY, s);
        if (rc) { printf("rc %d\n", rc); exit(1); }
    });
    bench("host_v1 copy", [&] {
        int rc = metro_route_host_v1(ids, P, dmask, N, G, ws, out, pr, 0, 0, s);
        if (rc) { printf("rc %d\n", rc); exit(1); }
    });
    int32_t *dids; cudaMalloc(&dids, P * 4);
    cudaMemcpy(dids, ids, P * 4, cudaMemcpyHostToDevice);
    int32_t *dout; cudaMalloc(&dout, (8 + G + N + P) * 4);
    for (int R : {1, 2, 4, 8}) {
        char name[64]; snprintf(name, sizeof name, "device route R=%d +sync", R);
        bench(name, [&] {
            metro_route_v1(dids, P, dmask, N, G, nullptr, dout + 8 + G, dout + 8, dout + 4, dout + 8 + G + N, dout, R, s);
            cudaStreamSynchronize(s);
        });
    }
    // persistent server (metro_serve.h): both fence variants
    struct Var { const char *name, *warps, *stagger; };
    const Var vars[] = {
        {"served 4 pollers st500", "4", "500"}, {"served 4 pollers st1000", "4", "1000"},
        {"served 2 pollers st700", "2", "700"}, {"served 2 pollers st1000", "2", "1000"},
        {"served 2 pollers st1500", "2", "1500"}, {"served 1 poller", "1", "0"},
    };
    for (const Var &v : vars) {
        setenv("METRO_SERVE_STAGGER_NS", v.stagger, 1);
        setenv("METRO_SERVE_DOORBELL_WARPS", v.warps, 1);
        for (int np : {P, 0}) {
            metro_server *srv = nullptr;
            int rc = metro_server_create_v1(dmask, N, G, P, 500000, &srv);
            if (rc) { printf("create rc %d\n", rc); exit(1); }
            char name[96]; snprintf(name, sizeof name, "%s%s", v.name, np ? "" : " (empty batch)");
            double acc[8] = {0};
            int nacc = 0;
            bench(name, [&] {
                int rc2 = metro_server_route_v1(srv, ids, np, out, pr);
                if (rc2) { printf("route rc %d\n", rc2); exit(1); }
                int64_t st[8];
                metro_server_debug_stamps(srv, st);
                for (int i = 1; i < 8; ++i) acc[i] += st[i];
                ++nacc;
            });
            printf("  phases (mean ns): staged %.0f routed %.0f stored %.0f fence %.0f | total %.0f ns, %.0f MHz | "
                   "doorbell RTT %.0f ns | status %d lam %d launches %lld\n",
                   acc[1] / nacc, acc[2] / nacc, acc[3] / nacc, acc[4] / nacc, acc[6] / nacc,
                   acc[5] / acc[6] * 1e3, acc[7] / nacc, out[0], out[4], (long long)metro_server_launches(srv));
            metro_server_destroy_v1(srv);
        }
    }
    printf("status %d lam %d\n", out[0], out[4]);
    return 0;
}
