// genasm_capi.cu -- host side of the C ABI in include/genasm.h.
//
// Replaces the reference's driver/batch layer (pkg/src/bitalign/window.py:
// 85-163) for the hot path: config validation (window.py:58-70), batch
// fan-out (align_batch, :152-163 -- here a persistent kernel instead of a
// process pool), longest-first ordering, device buffer management and the
// host<->device copies.  One context per device; contexts are independent,
// so a multi-GPU caller runs one host thread per context.
//
// The host-buffer call (ga_align_batch) splits the batch into chunks of
// consecutive pairs and pipelines them over three streams: the H2D of chunk
// k+1 and the D2H of chunk k-1 overlap the kernel of chunk k.  Sequences can
// travel 2 bits per symbol and ops 2 bits per op.
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

namespace genasm {
cudaError_t launch_unpack2(const uint8_t* packed, int64_t nsym, uint8_t* out, cudaStream_t st);
cudaError_t launch_patch(const int64_t* pos, int64_t n, int64_t base, uint8_t* out, cudaStream_t st);
cudaError_t launch_pack_ops(const uint8_t* ascii, int64_t nops, uint8_t* out, cudaStream_t st);
}  // namespace genasm

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

// device buffers and chunk-local host arrays of one pipeline slot
struct Slot {
    DevBuf codes, packed, exc, pat_off, pat_len, txt_off, txt_len, order, results, ops_off, ops,
        ops2, win_off, dists;
    std::vector<int64_t> h_pat_off, h_txt_off, h_ops_off, h_win_off, h_exc;
    std::vector<int32_t> h_order;
    cudaEvent_t in_done = nullptr, out_done = nullptr, kern_done = nullptr;
    void release() {
        for (DevBuf* b : {&codes, &packed, &exc, &pat_off, &pat_len, &txt_off, &txt_len, &order,
                          &results, &ops_off, &ops, &ops2, &win_off, &dists})
            b->release();
        for (cudaEvent_t ev : {in_done, out_done, kern_done})
            if (ev) cudaEventDestroy(ev);
    }
};

struct ga_ctx {
    int device = 0;
    int num_sms = 0;
    cudaStream_t stream = nullptr, stream_in = nullptr, stream_out = nullptr;
    std::string err;
    int64_t launches = 0;
    unsigned long long* queue = nullptr;
    uint32_t* overflow = nullptr;
    size_t overflow_cap = 0;
    Slot slot[2];
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
    for (cudaStream_t* s : {&c->stream, &c->stream_in, &c->stream_out})
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
    for (Slot& sl : c->slot)
        for (cudaEvent_t* ev : {&sl.in_done, &sl.out_done, &sl.kern_done})
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
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
    cudaDeviceSynchronize();
    for (Slot& sl : c->slot) sl.release();
    if (c->overflow) cudaFree(c->overflow);
    if (c->queue) cudaFree(c->queue);
    for (cudaStream_t s : {c->stream, c->stream_in, c->stream_out})
        if (s) cudaStreamDestroy(s);
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
    if (out->ops2) {
        for (int64_t q = 0; q < n; ++q)
            if (out->ops_off[q] & 3) {
                c->err = "ops2 output needs every ops_off to be a multiple of 4";
                return -3;
            }
    }
    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) return fail(c, e, "cudaSetDevice");

    // ---- chunk plan: consecutive pairs; 2 chunks overlap copies with the kernel
    // when the batch is large enough that each chunk still fills the GPU ----
    int chunks = env_int("GA_CHUNKS", n >= 65536 ? 2 : 1);
    if (chunks < 1) chunks = 1;
    if (chunks > n) chunks = (int)n;
    // chunking needs output offsets that grow with the input index (the
    // prefix-sum layout every caller in this package uses)
    for (int64_t q = 1; q < n && chunks > 1; ++q)
        if (out->ops_off[q] < out->ops_off[q - 1] || out->win_off[q] < out->win_off[q - 1])
            chunks = 1;
    int64_t launches = 0;
    for (int k = 0; k < chunks; ++k) {
        const int64_t q0 = n * k / chunks, q1 = n * (k + 1) / chunks;
        const int64_t m = q1 - q0;
        Slot& S = c->slot[k & 1];
        // the symbol, op and window ranges the chunk touches
        int64_t lo = INT64_MAX, hi = 0;
        for (int64_t q = q0; q < q1; ++q) {
            lo = std::min(lo, std::min(in->pat_off[q], in->txt_off[q]));
            hi = std::max(hi, std::max(in->pat_off[q] + in->pat_len[q], in->txt_off[q] + in->txt_len[q]));
        }
        if (lo > hi) lo = hi;
        int64_t olo = INT64_MAX, ohi = 0, wlo = INT64_MAX, whi = 0;
        for (int64_t q = q0; q < q1; ++q) {
            olo = std::min(olo, out->ops_off[q]);
            wlo = std::min(wlo, out->win_off[q]);
        }
        // a pair's capacity ends where the next larger offset (or the buffer) begins
        ohi = out->ops_capacity;
        whi = out->win_capacity;
        for (int64_t q = 0; q < n; ++q) {
            if (q >= q0 && q < q1) continue;
            if (out->ops_off[q] >= olo) ohi = std::min(ohi, out->ops_off[q]);
            if (out->win_off[q] >= wlo) whi = std::min(whi, out->win_off[q]);
        }
        const int64_t base = in->packed2 ? (lo & ~int64_t(3)) : lo;
        const int64_t nsym = hi - base;
        // chunk-local host arrays (rebased offsets, LPT order)
        S.h_pat_off.resize((size_t)m);
        S.h_txt_off.resize((size_t)m);
        S.h_ops_off.resize((size_t)m);
        S.h_win_off.resize((size_t)m);
        S.h_order.resize((size_t)m);
        for (int64_t q = 0; q < m; ++q) {
            S.h_pat_off[(size_t)q] = in->pat_off[q0 + q] - base;
            S.h_txt_off[(size_t)q] = in->txt_off[q0 + q] - base;
            S.h_ops_off[(size_t)q] = out->ops_off[q0 + q] - olo;
            S.h_win_off[(size_t)q] = out->win_off[q0 + q] - wlo;
        }
        if (in->order && chunks == 1) {
            std::copy(in->order, in->order + n, S.h_order.begin());
        } else {
            ga_lpt_order(m, in->pat_len + q0, S.h_order.data());
        }
        int64_t nexc = 0, exc0 = 0;
        if (in->packed2 && in->n_exceptions > 0) {
            exc0 = std::lower_bound(in->exceptions, in->exceptions + in->n_exceptions, base) -
                   in->exceptions;
            const int64_t exc1 = std::lower_bound(in->exceptions, in->exceptions + in->n_exceptions,
                                                  hi) - in->exceptions;
            nexc = exc1 - exc0;
        }
        const int64_t nops = ohi - olo;
        const int64_t nwin = whi - wlo;
        if ((e = S.codes.ensure((size_t)nsym + 16)) || (e = S.pat_off.ensure((size_t)m * 8)) ||
            (e = S.txt_off.ensure((size_t)m * 8)) || (e = S.pat_len.ensure((size_t)m * 4)) ||
            (e = S.txt_len.ensure((size_t)m * 4)) || (e = S.order.ensure((size_t)m * 4)) ||
            (e = S.ops_off.ensure((size_t)m * 8)) || (e = S.win_off.ensure((size_t)m * 8)) ||
            (e = S.results.ensure((size_t)m * sizeof(ga_pair_result))) ||
            (e = S.ops.ensure((size_t)nops + 16)) || (e = S.dists.ensure((size_t)nwin + 16)))
            return fail(c, e, "cudaMalloc");
        if (in->packed2 && ((e = S.packed.ensure((size_t)(nsym + 3) / 4 + 16)) ||
                            (e = S.exc.ensure((size_t)(nexc > 0 ? nexc : 1) * 8))))
            return fail(c, e, "cudaMalloc");
        if (out->ops2 && (e = S.ops2.ensure((size_t)(nops + 3) / 4 + 16)))
            return fail(c, e, "cudaMalloc");

        // ---- H2D (input stream), after this slot's previous chunk left the device ----
        cudaStream_t si = c->stream_in, sk = c->stream, so = c->stream_out;
        if (k >= 2 && (e = cudaStreamWaitEvent(si, S.out_done, 0))) return fail(c, e, "wait");
        auto h2d = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
            return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, si) : cudaSuccess;
        };
        if (in->packed2) {
            e = h2d(S.packed.ptr, in->codes + base / 4, (size_t)(nsym + 3) / 4);
            if (!e && nexc) e = h2d(S.exc.ptr, in->exceptions + exc0, (size_t)nexc * 8);
        } else {
            e = h2d(S.codes.ptr, in->codes + base, (size_t)nsym);
        }
        if (!e) e = h2d(S.pat_off.ptr, S.h_pat_off.data(), (size_t)m * 8);
        if (!e) e = h2d(S.txt_off.ptr, S.h_txt_off.data(), (size_t)m * 8);
        if (!e) e = h2d(S.pat_len.ptr, in->pat_len + q0, (size_t)m * 4);
        if (!e) e = h2d(S.txt_len.ptr, in->txt_len + q0, (size_t)m * 4);
        if (!e) e = h2d(S.order.ptr, S.h_order.data(), (size_t)m * 4);
        if (!e) e = h2d(S.ops_off.ptr, S.h_ops_off.data(), (size_t)m * 8);
        if (!e) e = h2d(S.win_off.ptr, S.h_win_off.data(), (size_t)m * 8);
        if (!e) e = cudaEventRecord(S.in_done, si);
        if (e) return fail(c, e, "H2D copy");

        // ---- compute stream: expand 2-bit sequences, align, pack ops ----
        if ((e = cudaStreamWaitEvent(sk, S.in_done, 0))) return fail(c, e, "wait");
        if (in->packed2) {
            if ((e = genasm::launch_unpack2((const uint8_t*)S.packed.ptr, nsym, (uint8_t*)S.codes.ptr,
                                            sk)) ||
                (e = genasm::launch_patch((const int64_t*)S.exc.ptr, nexc, base, (uint8_t*)S.codes.ptr,
                                          sk)))
                return fail(c, e, "unpack kernel");
            launches += 1 + (nexc > 0);
        }
        ga_batch_in din{};
        din.n_pairs = m;
        din.codes = (const uint8_t*)S.codes.ptr;
        din.codes_len = nsym;
        din.pat_off = (const int64_t*)S.pat_off.ptr;
        din.pat_len = (const int32_t*)S.pat_len.ptr;
        din.txt_off = (const int64_t*)S.txt_off.ptr;
        din.txt_len = (const int32_t*)S.txt_len.ptr;
        din.order = (const int32_t*)S.order.ptr;
        ga_batch_out dout{};
        dout.results = (ga_pair_result*)S.results.ptr;
        dout.ops_off = (const int64_t*)S.ops_off.ptr;
        dout.ops = (uint8_t*)S.ops.ptr;
        dout.ops_capacity = nops;
        dout.win_off = (const int64_t*)S.win_off.ptr;
        dout.window_distances = (uint8_t*)S.dists.ptr;
        dout.win_capacity = nwin;
        int rc = ga_align_batch_device(c, &din, cfg, &dout, sk);
        if (rc) return rc;
        launches += c->launches;
        if (out->ops2) {
            if ((e = genasm::launch_pack_ops((const uint8_t*)S.ops.ptr, nops, (uint8_t*)S.ops2.ptr, sk)))
                return fail(c, e, "pack kernel");
            launches += 1;
        }
        if ((e = cudaEventRecord(S.kern_done, sk))) return fail(c, e, "record");

        // ---- D2H (output stream) ----
        if ((e = cudaStreamWaitEvent(so, S.kern_done, 0))) return fail(c, e, "wait");
        auto d2h = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
            return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, so) : cudaSuccess;
        };
        e = d2h(out->results + q0, S.results.ptr, (size_t)m * sizeof(ga_pair_result));
        if (!e) {
            if (out->ops2) e = d2h(out->ops + olo / 4, S.ops2.ptr, (size_t)(nops + 3) / 4);
            else e = d2h(out->ops + olo, S.ops.ptr, (size_t)nops);
        }
        if (!e) e = d2h(out->window_distances + wlo, S.dists.ptr, (size_t)nwin);
        if (!e) e = cudaEventRecord(S.out_done, so);
        if (e) return fail(c, e, "D2H copy");
    }
    if ((e = cudaStreamSynchronize(c->stream_out)) != cudaSuccess)
        return fail(c, e, "kernel execution");
    c->launches = launches;
    return 0;
}

}  // extern "C"
