// Dependent-chain latency probe for the greedy's candidate instructions (one
// warp, clock64).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o
// latency_probe latency_probe.cu ; run on the B200 box.  Informs DESIGN.md §4.
#include <cstdio>
#include <cstdint>

#define ITERS 4096

__global__ void probe(int64_t *out, uint32_t seed) {
    __shared__ uint32_t sm[64];
    if (threadIdx.x < 64) sm[threadIdx.x] = (threadIdx.x + 1) & 63;
    __syncthreads();
    uint32_t x = seed, y = seed * 3 + 1, z = 0x1111 * (seed & 7);
    int64_t t0, t1;
    int k = 0;
#define RUN(NAME, BODY)                                        \
    t0 = clock64();                                            \
    for (int i = 0; i < ITERS; ++i) { BODY; }                  \
    t1 = clock64();                                            \
    if (threadIdx.x == 0) out[k] = (t1 - t0);                  \
    k++;
    // 0: PRMT chain
    RUN("prmt", asm volatile("prmt.b32 %0, %0, %1, %2;" : "+r"(x) : "r"(y), "r"(z)));
    // 1: IADD chain
    RUN("iadd", asm volatile("add.u32 %0, %0, %1;" : "+r"(x) : "r"(y)));
    // 2: setp + predicated add (x feeds setp)
    RUN("setp_padd", asm volatile("{.reg .pred p; setp.le.u32 p, %0, %1; @p add.u32 %0, %0, %2;}" : "+r"(x) : "r"(y), "r"(z)));
    // 3: setp + selp
    RUN("setp_selp", asm volatile("{.reg .pred p; setp.le.u32 p, %0, %1; selp.u32 %0, %1, %2, p;}" : "+r"(x) : "r"(y), "r"(z)));
    // 4: min chain
    RUN("min", asm volatile("min.u32 %0, %0, %1;" : "+r"(x) : "r"(y)));
    // 5: lop3 chain
    RUN("lop3", asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x) : "r"(y), "r"(z)));
    // 6: shift chain
    RUN("shf", asm volatile("shf.l.wrap.b32 %0, %0, %0, %1;" : "+r"(x) : "r"(y)));
    // 7: redux.sync.min
    RUN("redux", { uint32_t v; asm volatile("redux.sync.min.u32 %0, %1, 0xffffffff;" : "=r"(v) : "r"(x)); x = v + 1; });
    // 8: shfl
    RUN("shfl", x = __shfl_xor_sync(0xffffffffu, x, 1) + 1);
    // 9: lds pointer chase
    RUN("lds", x = sm[x & 63]);
    // 10: r=2 step: prmt x2, setp, 2 predicated adds per half (lo/hi)
    {
        uint32_t lo = x, hi = y, ia = 1, ib = 0x100;
        t0 = clock64();
        for (int i = 0; i < ITERS; ++i) {
            uint32_t va, vb;
            asm volatile("prmt.b32 %0, %1, %2, 0x1111;" : "=r"(va) : "r"(lo), "r"(hi));
            asm volatile("prmt.b32 %0, %1, %2, 0x5555;" : "=r"(vb) : "r"(lo), "r"(hi));
            asm volatile("{.reg .pred p; setp.le.u32 p, %2, %3; @p add.u32 %0, %0, %4; @!p add.u32 %0, %0, %5;"
                         " @p add.u32 %1, %1, %5; @!p add.u32 %1, %1, %4;}"
                         : "+r"(lo), "+r"(hi) : "r"(va), "r"(vb), "r"(ia), "r"(ib));
        }
        t1 = clock64();
        if (threadIdx.x == 0) out[k] = t1 - t0;
        k++;
        x = lo ^ hi;
    }
    // 11: r=2 step, select-then-add form
    {
        uint32_t lo = x, hi = y, ia = 1, ib = 0x100;
        t0 = clock64();
        for (int i = 0; i < ITERS; ++i) {
            uint32_t va, vb, sl, sh;
            asm volatile("prmt.b32 %0, %1, %2, 0x1111;" : "=r"(va) : "r"(lo), "r"(hi));
            asm volatile("prmt.b32 %0, %1, %2, 0x5555;" : "=r"(vb) : "r"(lo), "r"(hi));
            asm volatile("{.reg .pred p; setp.le.u32 p, %2, %3; selp.u32 %0, %4, %5, p; selp.u32 %1, %5, %4, p;}"
                         : "=r"(sl), "=r"(sh) : "r"(va), "r"(vb), "r"(ia), "r"(ib));
            asm volatile("add.u32 %0, %0, %1;" : "+r"(lo) : "r"(sl));
            asm volatile("add.u32 %0, %0, %1;" : "+r"(hi) : "r"(sh));
        }
        t1 = clock64();
        if (threadIdx.x == 0) out[k] = t1 - t0;
        k++;
        x ^= lo ^ hi;
    }
    // 12: vimnmx u16x2 chain (packed 16-bit min)
    RUN("min16x2", asm volatile("min.u16x2 %0, %0, %1;" : "+r"(x) : "r"(y)));
    // 13: 64-bit add chain
    {
        uint64_t a = x, b = y;
        t0 = clock64();
        for (int i = 0; i < ITERS; ++i) asm volatile("add.u64 %0, %0, %1;" : "+l"(a) : "l"(b));
        t1 = clock64();
        if (threadIdx.x == 0) out[k] = t1 - t0;
        k++;
        x ^= (uint32_t)a;
    }
    // 14: imad chain
    RUN("imad", asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(y), "r"(z)));
    // 15: new r2 step: prmt x2, sub, prmt sign, lop3 pick x2, add x2
    {
        uint32_t lo = x & 0x3f3f3f3f, hi = y & 0x3f3f3f3f, ia = 1, xa = 0x101;
        t0 = clock64();
        for (int i = 0; i < ITERS; ++i) {
            uint32_t va, vb, m, pl, ph;
            asm volatile("prmt.b32 %0, %1, %2, 0x8881;" : "=r"(va) : "r"(lo), "r"(hi));
            asm volatile("prmt.b32 %0, %1, %2, 0xDDD5;" : "=r"(vb) : "r"(lo), "r"(hi));
            asm volatile("sub.u32 %0, %1, %2;" : "=r"(m) : "r"(vb), "r"(va));
            asm volatile("prmt.b32 %0, %0, 0, 0xBBBB;" : "+r"(m));
            asm volatile("lop3.b32 %0, %1, %2, %3, 0x78;" : "=r"(pl) : "r"(ia), "r"(xa), "r"(m));
            asm volatile("lop3.b32 %0, %1, %2, %3, 0x78;" : "=r"(ph) : "r"(ia), "r"(xa), "r"(m));
            asm volatile("add.u32 %0, %0, %1;" : "+r"(lo) : "r"(pl));
            asm volatile("add.u32 %0, %0, %1;" : "+r"(hi) : "r"(ph));
            lo &= 0x3f3f3f3f;
        }
        t1 = clock64();
        if (threadIdx.x == 0) out[k] = t1 - t0;
        k++;
        x ^= lo ^ hi;
    }
    // 16: imad-pick r2 step: L' = mad(dinc, m, L + incA)
    {
        uint32_t lo = x & 0x3f3f3f3f, hi = y & 0x3f3f3f3f, ia = 1, da = 0xff;
        t0 = clock64();
        for (int i = 0; i < ITERS; ++i) {
            uint32_t va, vb, m, la, ha;
            asm volatile("prmt.b32 %0, %1, %2, 0x8881;" : "=r"(va) : "r"(lo), "r"(hi));
            asm volatile("prmt.b32 %0, %1, %2, 0xDDD5;" : "=r"(vb) : "r"(lo), "r"(hi));
            asm volatile("add.u32 %0, %1, %2;" : "=r"(la) : "r"(lo), "r"(ia));
            asm volatile("add.u32 %0, %1, %2;" : "=r"(ha) : "r"(hi), "r"(ia));
            asm volatile("sub.u32 %0, %1, %2;" : "=r"(m) : "r"(vb), "r"(va));
            asm volatile("prmt.b32 %0, %0, 0, 0xBBBB;" : "+r"(m));
            asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(lo) : "r"(da), "r"(m), "r"(la));
            asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(hi) : "r"(da), "r"(m), "r"(ha));
        }
        t1 = clock64();
        if (threadIdx.x == 0) out[k] = t1 - t0;
        k++;
        x ^= lo ^ hi;
    }
    // 17: prmt -> add (lo only)
    {
        uint32_t lo = x, hi = y;
        t0 = clock64();
        for (int i = 0; i < ITERS; ++i) {
            uint32_t va;
            asm volatile("prmt.b32 %0, %1, %2, 0x8881;" : "=r"(va) : "r"(lo), "r"(hi));
            asm volatile("add.u32 %0, %0, %1;" : "+r"(lo) : "r"(va));
        }
        t1 = clock64();
        if (threadIdx.x == 0) out[k] = t1 - t0;
        k++;
        x ^= lo;
    }
    // 18: sub -> prmt sign chain
    RUN("sub_sgn", { asm volatile("sub.u32 %0, %0, %1;" : "+r"(x) : "r"(y)); asm volatile("prmt.b32 %0, %0, 0, 0xBBBB;" : "+r"(x)); });
    // 19: prmt -> add.cc (carry form, hoping for IADD3 on the ALU pipe)
    {
        uint32_t lo = x, hi = y;
        t0 = clock64();
        for (int i = 0; i < ITERS; ++i) {
            uint32_t va;
            asm volatile("prmt.b32 %0, %1, %2, 0x8881;" : "=r"(va) : "r"(lo), "r"(hi));
            asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(lo) : "r"(va));
        }
        t1 = clock64();
        if (threadIdx.x == 0) out[k] = t1 - t0;
        k++;
        x ^= lo;
    }
    // 20: r2 step with add.cc / sub.cc on the chain
    {
        uint32_t lo = x & 0x3f3f3f3f, hi = y & 0x3f3f3f3f, ia = 1, xa = 0x101;
        t0 = clock64();
        for (int i = 0; i < ITERS; ++i) {
            uint32_t va, vb, m, pl, ph;
            asm volatile("prmt.b32 %0, %1, %2, 0x8881;" : "=r"(va) : "r"(lo), "r"(hi));
            asm volatile("prmt.b32 %0, %1, %2, 0xDDD5;" : "=r"(vb) : "r"(lo), "r"(hi));
            asm volatile("sub.cc.u32 %0, %1, %2;" : "=r"(m) : "r"(vb), "r"(va));
            asm volatile("prmt.b32 %0, %0, 0, 0xBBBB;" : "+r"(m));
            asm volatile("lop3.b32 %0, %1, %2, %3, 0x78;" : "=r"(pl) : "r"(ia), "r"(xa), "r"(m));
            asm volatile("lop3.b32 %0, %1, %2, %3, 0x78;" : "=r"(ph) : "r"(ia), "r"(xa), "r"(m));
            asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(lo) : "r"(pl));
            asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(hi) : "r"(ph));
        }
        t1 = clock64();
        if (threadIdx.x == 0) out[k] = t1 - t0;
        k++;
        x ^= lo ^ hi;
    }
    // 21: same step, plain add/sub (for comparison without the mask lop3)
    {
        uint32_t lo = x & 0x3f3f3f3f, hi = y & 0x3f3f3f3f, ia = 1, xa = 0x101;
        t0 = clock64();
        for (int i = 0; i < ITERS; ++i) {
            uint32_t va, vb, m, pl, ph;
            asm volatile("prmt.b32 %0, %1, %2, 0x8881;" : "=r"(va) : "r"(lo), "r"(hi));
            asm volatile("prmt.b32 %0, %1, %2, 0xDDD5;" : "=r"(vb) : "r"(lo), "r"(hi));
            asm volatile("sub.u32 %0, %1, %2;" : "=r"(m) : "r"(vb), "r"(va));
            asm volatile("prmt.b32 %0, %0, 0, 0xBBBB;" : "+r"(m));
            asm volatile("lop3.b32 %0, %1, %2, %3, 0x78;" : "=r"(pl) : "r"(ia), "r"(xa), "r"(m));
            asm volatile("lop3.b32 %0, %1, %2, %3, 0x78;" : "=r"(ph) : "r"(ia), "r"(xa), "r"(m));
            asm volatile("add.u32 %0, %0, %1;" : "+r"(lo) : "r"(pl));
            asm volatile("add.u32 %0, %0, %1;" : "+r"(hi) : "r"(ph));
        }
        t1 = clock64();
        if (threadIdx.x == 0) out[k] = t1 - t0;
        k++;
        x ^= lo ^ hi;
    }
    // 22: r2 step using vadd-free 3-input iadd: lo = lo + pl + 0 via add.cc/addc
    if (threadIdx.x == 0) out[63] = x;
}

int main() {
    int64_t *d;
    cudaMalloc(&d, 64 * sizeof(int64_t));
    probe<<<1, 32>>>(d, 5);
    probe<<<1, 32>>>(d, 7);
    cudaDeviceSynchronize();
    int64_t h[64];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const char *names[] = {"prmt", "iadd", "setp+pred_add", "setp+selp", "min.u32", "lop3", "shf", "redux.min",
                           "shfl.xor", "lds chase", "r2 step (pred add)", "r2 step (selp+add)", "min.u16x2",
                           "add.u64", "imad", "r2 new (lop3 pick)", "r2 imad pick", "prmt->add", "sub->prmt sign", "prmt->add.cc", "r2 step add.cc", "r2 step plain"};
    for (int i = 0; i < 22; ++i) printf("%-22s %6.2f cycles/iter\n", names[i], (double)h[i] / ITERS);
    return 0;
}
