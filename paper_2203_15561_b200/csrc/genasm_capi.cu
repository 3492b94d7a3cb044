// genasm_capi.cu -- host side of the C ABI in include/genasm.h.
//
// Replaces the reference's driver/batch layer (pkg/src/bitalign/window.py:
// 85-163) for the hot path: config validation (window.py:58-70), batch
// fan-out (align_batch, :152-163 -- here a persistent kernel instead of a
// process pool), longest-first ordering, device buffer management and the
// host<->device copies.  One context per device; contexts are independent,
// so a multi-GPU caller runs one host thread per context.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/genasm.h"
#include "genasm_kernel.cuh"

struct DevBuf {
    void* ptr = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap && ptr) return cudaSuccess;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
        size_t want = bytes < 256 ? 256 : bytes;
        cudaError_t e = cudaMalloc(&ptr, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
    }
};

struct ga_ctx {
    int device = 0;
    int num_sms = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    int64_t launches = 0;
    unsigned long long* queue = nullptr;
    uint32_t* overflow = nullptr;
    size_t overflow_cap = 0;
    DevBuf codes, pat_off, pat_len, txt_off, txt_len, order, results, ops_off, ops, win_off, dists;
    std::vector<int32_t> host_order;
    genasm::LaunchShape last_shape{};
};

static int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v && *v ? atoi(v) : dflt;
}

extern "C" {

const char* ga_version(void) { return "genasm-b200 0.1.0 (sm_100a)"; }

int64_t ga_num_windows(int64_t len, int32_t W, int32_t O) {
    if (len <= 0) return 0;
    if (len <= W) return 1;
    const int64_t step = W - O;
    return 1 + (len - W + step - 1) / step;
}

int ga_check_config(const ga_config* cfg, char* msg, int msg_len) {
    char buf[160];
    buf[0] = 0;
    int rc = 0;
    const int W = cfg->window, O = cfg->overlap, k = cfg->k;
    if (W < 1) {
        snprintf(buf, sizeof buf, "window must be >= 1, got %d", W);
        rc = 1;
    } else if (!(0 <= O && O < W)) {
        snprintf(buf, sizeof buf, "overlap must be in [0, window), got %d for window %d", O, W);
        rc = 1;
    } else if (!(1 <= k && k <= W)) {
        snprintf(buf, sizeof buf, "k must be in [1, %d], got %d", W, k);
        rc = 1;
    } else {
        char s[5] = {cfg->priority[0], cfg->priority[1], cfg->priority[2], cfg->priority[3], 0};
        char t[5];
        memcpy(t, s, 5);
        std::sort(t, t + 4);
        if (strcmp(t, "DIMS") != 0) {
            snprintf(buf, sizeof buf, "priority must be a permutation of 'MSID', got '%s'", s);
            rc = 1;
        } else if (W > GA_MAX_WINDOW) {
            snprintf(buf, sizeof buf, "window %d exceeds the kernel maximum of %d", W,
                     GA_MAX_WINDOW);
            rc = 1;
        }
    }
    if (msg && msg_len > 0) {
        strncpy(msg, buf, (size_t)msg_len - 1);
        msg[msg_len - 1] = 0;
    }
    return rc;
}

void ga_encode_ascii(const char* seq, int64_t n, uint8_t* out) {
    static uint8_t lut[256];
    static bool init = false;
    if (!init) {
        memset(lut, 4, sizeof lut);
        lut[(unsigned char)'A'] = 0;
        lut[(unsigned char)'C'] = 1;
        lut[(unsigned char)'G'] = 2;
        lut[(unsigned char)'T'] = 3;
        init = true;
    }
    for (int64_t i = 0; i < n; ++i) out[i] = lut[(unsigned char)seq[i]];
}

void ga_lpt_order(int64_t n, const int32_t* pat_len, int32_t* order) {
    std::iota(order, order + n, 0);
    std::stable_sort(order, order + n,
                     [&](int32_t a, int32_t b) { return pat_len[a] > pat_len[b]; });
}

void* ga_host_alloc(int64_t bytes) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, (size_t)(bytes > 0 ? bytes : 1), cudaHostAllocDefault) != cudaSuccess)
        return nullptr;
    return p;
}

void ga_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

int ga_create(int device, ga_ctx** out) {
    *out = nullptr;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return (int)e;
    ga_ctx* c = new ga_ctx();
    c->device = device;
    e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&c->queue, sizeof(unsigned long long));
    if (e != cudaSuccess) {
        delete c;
        return (int)e;
    }
    *out = c;
    return 0;
}

void ga_destroy(ga_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    for (DevBuf* b : {&c->codes, &c->pat_off, &c->pat_len, &c->txt_off, &c->txt_len, &c->order,
                      &c->results, &c->ops_off, &c->ops, &c->win_off, &c->dists})
        b->release();
    if (c->overflow) cudaFree(c->overflow);
    if (c->queue) cudaFree(c->queue);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

const char* ga_last_error(const ga_ctx* c) { return c ? c->err.c_str() : "null context"; }

int64_t ga_last_launch_count(const ga_ctx* c) { return c ? c->launches : 0; }

static int fail(ga_ctx* c, cudaError_t e, const char* what) {
    c->err = std::string(what) + ": " + cudaGetErrorString(e);
    return (int)e;
}

static uint32_t pack_priority(const char* pr) {
    uint32_t v = 0;
    for (int u = 0; u < 4; ++u) {
        uint32_t id = pr[u] == 'M' ? 0 : pr[u] == 'S' ? 1 : pr[u] == 'I' ? 2 : 3;
        v |= id << (2 * u);
    }
    return v;
}

int ga_align_batch_device(ga_ctx* c, const ga_batch_in* in, const ga_config* cfg,
                          ga_batch_out* out, void* stream_ptr) {
    if (!c) return -1;
    char msg[160];
    if (ga_check_config(cfg, msg, sizeof msg)) {
        c->err = msg;
        return -2;
    }
    c->launches = 0;
    if (in->n_pairs <= 0) return 0;
    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) return fail(c, e, "cudaSetDevice");
    cudaStream_t st = stream_ptr ? (cudaStream_t)stream_ptr : c->stream;
    genasm::KernelParams P{};
    P.codes = in->codes;
    P.pat_off = in->pat_off;
    P.pat_len = in->pat_len;
    P.txt_off = in->txt_off;
    P.txt_len = in->txt_len;
    P.order = in->order;
    P.n_pairs = in->n_pairs;
    P.W = cfg->window;
    P.O = cfg->overlap;
    P.k = cfg->k;
    P.prio = pack_priority(cfg->priority);
    // first active edge in priority order (backtrace.py:134-160); 5 = none (stuck)
    P.prio_lut = 0;
    for (uint64_t mask = 0; mask < 16; ++mask) {
        uint64_t op = 5;
        for (int u = 3; u >= 0; --u) {
            const uint64_t id = (P.prio >> (2 * u)) & 3u;
            if (mask & (1ull << id)) op = id;
        }
        P.prio_lut |= op << (4 * mask);
    }
    P.results = out->results;
    P.ops_off = out->ops_off;
    P.ops = out->ops;
    P.win_off = out->win_off;
    P.dists = out->window_distances;
    P.queue = c->queue;
    e = cudaMemsetAsync(c->queue, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return fail(c, e, "queue reset");
    // tuning knobs (defaults measured on config 3): lanes per pair group, threads per block
    const int group = env_int("GA_GROUP", 8);
    const int block = env_int("GA_BLOCK", 0);
    e = genasm::launch_genasm_lockstep(P, group, block, c->num_sms, st, &c->overflow,
                                       &c->overflow_cap, &c->last_shape);
    if (e != cudaSuccess) return fail(c, e, "genasm kernel launch");
    c->launches = 1;
    return 0;
}

int ga_align_batch(ga_ctx* c, const ga_batch_in* in, const ga_config* cfg, ga_batch_out* out) {
    if (!c) return -1;
    char msg[160];
    if (ga_check_config(cfg, msg, sizeof msg)) {
        c->err = msg;
        return -2;
    }
    const int64_t n = in->n_pairs;
    c->launches = 0;
    if (n <= 0) return 0;
    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) return fail(c, e, "cudaSetDevice");
    cudaStream_t st = c->stream;
    const int32_t* order = in->order;
    if (!order) {
        c->host_order.resize((size_t)n);
        ga_lpt_order(n, in->pat_len, c->host_order.data());
        order = c->host_order.data();
    }
    struct Cp {
        DevBuf* buf;
        const void* src;
        size_t bytes;
    } h2d[] = {
        {&c->codes, in->codes, (size_t)in->codes_len},
        {&c->pat_off, in->pat_off, (size_t)n * 8},
        {&c->pat_len, in->pat_len, (size_t)n * 4},
        {&c->txt_off, in->txt_off, (size_t)n * 8},
        {&c->txt_len, in->txt_len, (size_t)n * 4},
        {&c->order, order, (size_t)n * 4},
        {&c->ops_off, out->ops_off, (size_t)n * 8},
        {&c->win_off, out->win_off, (size_t)n * 8},
    };
    for (auto& x : h2d) {
        if ((e = x.buf->ensure(x.bytes)) != cudaSuccess) return fail(c, e, "cudaMalloc");
        if (x.bytes && (e = cudaMemcpyAsync(x.buf->ptr, x.src, x.bytes, cudaMemcpyHostToDevice,
                                            st)) != cudaSuccess)
            return fail(c, e, "H2D copy");
    }
    if ((e = c->results.ensure((size_t)n * sizeof(ga_pair_result))) != cudaSuccess ||
        (e = c->ops.ensure((size_t)out->ops_capacity)) != cudaSuccess ||
        (e = c->dists.ensure((size_t)out->win_capacity)) != cudaSuccess)
        return fail(c, e, "cudaMalloc");
    ga_batch_in din = *in;
    din.codes = (const uint8_t*)c->codes.ptr;
    din.pat_off = (const int64_t*)c->pat_off.ptr;
    din.pat_len = (const int32_t*)c->pat_len.ptr;
    din.txt_off = (const int64_t*)c->txt_off.ptr;
    din.txt_len = (const int32_t*)c->txt_len.ptr;
    din.order = (const int32_t*)c->order.ptr;
    ga_batch_out dout = *out;
    dout.results = (ga_pair_result*)c->results.ptr;
    dout.ops_off = (const int64_t*)c->ops_off.ptr;
    dout.ops = (uint8_t*)c->ops.ptr;
    dout.win_off = (const int64_t*)c->win_off.ptr;
    dout.window_distances = (uint8_t*)c->dists.ptr;
    int rc = ga_align_batch_device(c, &din, cfg, &dout, st);
    if (rc) return rc;
    if ((e = cudaMemcpyAsync(out->results, dout.results, (size_t)n * sizeof(ga_pair_result),
                             cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(out->ops, dout.ops, (size_t)out->ops_capacity,
                             cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(out->window_distances, dout.window_distances,
                             (size_t)out->win_capacity, cudaMemcpyDeviceToHost, st)) !=
            cudaSuccess)
        return fail(c, e, "D2H copy");
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return fail(c, e, "kernel execution");
    return 0;
}

}  // extern "C"
