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

struct HostBuf {  // pinned host staging
    void* ptr = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap && ptr) return cudaSuccess;
        if (ptr) cudaFreeHost(ptr);
        ptr = nullptr;
        cap = 0;
        cudaError_t e = cudaHostAlloc(&ptr, bytes, cudaHostAllocDefault);
        if (e == cudaSuccess) cap = bytes;
        return e;
    }
    void release() {
        if (ptr) cudaFreeHost(ptr);
        ptr = nullptr;
        cap = 0;
    }
};

// Scratch one kernel launch owns: the work queue head and the overflow slabs
// + band tables.  Chunks in flight on different slots use different scratch,
// so their kernels can overlap (the next chunk fills SMs as one drains).
struct Scratch {
    unsigned long long* queue = nullptr;
    uint32_t* overflow = nullptr;  // lane-group kernel
    size_t overflow_cap = 0;
    uint32_t* thr = nullptr;       // lane-per-pair kernel
    size_t thr_cap = 0;
    uint64_t* dense = nullptr;     // unimproved engine: dense edge tables
    size_t dense_cap = 0;
    void release() {
        if (overflow) cudaFree(overflow);
        if (thr) cudaFree(thr);
        if (queue) cudaFree(queue);
        if (dense) cudaFree(dense);
        overflow = thr = nullptr;
        queue = nullptr;
        dense = nullptr;
        overflow_cap = thr_cap = dense_cap = 0;
    }
};

// One pipeline slot of the host-buffer path: device buffers, a pinned staging
// area for the chunk's per-pair metadata, its kernel stream and events.
// Metadata layout (host staging and device `meta` alike), per chunk of m pairs:
//   int64 pat_off[m] | txt_off[m] | ops_off[m] | win_off[m] | int32 pat_len[m] | txt_len[m] | order[m]
struct Slot {
    DevBuf codes, packed, exc, meta, results, ops, ops2, dists;
    HostBuf h_pack, h_exc;  // packed2 == GA_PACK_HOST: this chunk's 2-bit symbols
    void* h_meta = nullptr;
    size_t h_meta_cap = 0;
    Scratch scratch;
    cudaStream_t stream = nullptr;
    cudaEvent_t in_done = nullptr, out_done = nullptr, kern_done = nullptr;
    bool used = false;  // in_done/out_done have been recorded
    void release() {
        for (DevBuf* b : {&codes, &packed, &exc, &meta, &results, &ops, &ops2, &dists}) b->release();
        h_pack.release();
        h_exc.release();
        if (h_meta) cudaFreeHost(h_meta);
        h_meta = nullptr;
        scratch.release();
        for (cudaEvent_t ev : {in_done, out_done, kern_done})
            if (ev) cudaEventDestroy(ev);
        if (stream) cudaStreamDestroy(stream);
    }
};

constexpr int kSlots = 8;

struct ga_ctx {
    int device = 0;
    int num_sms = 0;
    cudaStream_t stream = nullptr, stream_in = nullptr, stream_out = nullptr;
    std::string err;
    int64_t launches = 0;
    Scratch scratch;  // ga_align_batch_device
    Slot slot[kSlots];
    DevBuf dp_in, dp_meta, dp_out;  // ga_edit_distance
    uint64_t* dp_slab = nullptr;
    size_t dp_cap = 0;
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
        } else if (cfg->mode != GA_MODE_IMPROVED && cfg->mode != GA_MODE_BASELINE) {
            snprintf(buf, sizeof buf, "mode must be one of ('improved', 'baseline'), got %d",
                     cfg->mode);
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
    for (Slot& sl : c->slot) {
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&sl.stream, cudaStreamNonBlocking);
        for (cudaEvent_t* ev : {&sl.in_done, &sl.out_done, &sl.kern_done})
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
        ga_destroy(c);
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
    c->scratch.release();
    for (DevBuf* b : {&c->dp_in, &c->dp_meta, &c->dp_out}) b->release();
    if (c->dp_slab) cudaFree(c->dp_slab);
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

// one fused DC+TB launch over device buffers with the given scratch
static int launch_batch(ga_ctx* c, const ga_batch_in* in, const ga_config* cfg,
                        const ga_batch_out* out, cudaStream_t st, Scratch* sc,
                        bool overlapped = false) {
    cudaError_t e;
    // [0] the fresh-pair queue, [1] finished pairs (lane-per-pair kernel)
    if (!sc->queue && (e = cudaMalloc(&sc->queue, 2 * sizeof(unsigned long long))))
        return fail(c, e, "cudaMalloc");
    genasm::KernelParams P{};
    P.codes = in->codes;
    P.codes_len = in->codes_len;
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
    P.ops_capacity = out->ops_capacity;
    P.win_off = out->win_off;
    P.dists = out->window_distances;
    P.queue = sc->queue;
    P.overlapped = overlapped ? 1 : 0;
    e = cudaMemsetAsync(sc->queue, 0, 2 * sizeof(unsigned long long), st);
    if (e != cudaSuccess) return fail(c, e, "queue reset");
    // tuning knobs (defaults measured on config 3): lanes per pair group, threads per block
    // W <= 64: the lane-per-pair kernel; GA_KERNEL=lockstep forces the
    // lane-group kernel, which also serves W > 64
    if (cfg->mode == GA_MODE_BASELINE) {
        e = genasm::launch_genasm_baseline(P, c->num_sms, st, &sc->dense, &sc->dense_cap,
                                           &c->last_shape);
        if (e != cudaSuccess) return fail(c, e, "genasm baseline kernel launch");
        return 0;
    }
    const char* kern = getenv("GA_KERNEL");
    const bool lockstep = P.W > 64 || (kern && strcmp(kern, "lockstep") == 0);
    if (lockstep) {
        // 16 lanes per pair while the pairs fill at most about half the GPU's
        // threads at 16 each (config 5 at W = 128, 8,192 pairs: 53.7 -> 45.3 ms
        // against 8), else 8
        const int group = env_int("GA_GROUP", P.n_pairs * 16 <= (int64_t)c->num_sms * 1024 ? 16 : 8);
        const int block = env_int("GA_BLOCK", 0);
        e = genasm::launch_genasm_lockstep(P, group, block, c->num_sms, st, &sc->overflow,
                                           &sc->overflow_cap, &c->last_shape);
    } else {
        e = genasm::launch_genasm_thread(P, c->num_sms, st, &sc->thr, &sc->thr_cap,
                                         &c->last_shape);
    }
    if (e != cudaSuccess) return fail(c, e, "genasm kernel launch");
    return 0;
}

int ga_edit_distance(ga_ctx* c, const ga_batch_in* in, int32_t semiglobal, int64_t* dist) {
    if (!c) return -1;
    const int64_t n = in->n_pairs;
    c->launches = 0;
    if (n <= 0) return 0;
    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) return fail(c, e, "cudaSetDevice");
    int max_words = 1;
    for (int64_t q = 0; q < n; ++q) max_words = std::max(max_words, (in->pat_len[q] + 63) / 64);
    const size_t syms = (size_t)std::max<int64_t>(in->codes_len, 1);
    const size_t meta = (size_t)n * (8 + 4 + 8 + 4 + 4);
    if ((e = c->dp_in.ensure(syms)) || (e = c->dp_meta.ensure(meta)) ||
        (e = c->dp_out.ensure((size_t)n * 8)))
        return fail(c, e, "cudaMalloc (edit distance)");
    if (!c->scratch.queue && (e = cudaMalloc(&c->scratch.queue, 2 * sizeof(unsigned long long))))
        return fail(c, e, "cudaMalloc");
    char* m = (char*)c->dp_meta.ptr;
    int64_t* pat_off = (int64_t*)m;
    int64_t* txt_off = pat_off + n;
    int32_t* pat_len = (int32_t*)(txt_off + n);
    int32_t* txt_len = pat_len + n;
    int32_t* order = txt_len + n;
    std::vector<int32_t> ord((size_t)n);
    if (in->order) std::copy(in->order, in->order + n, ord.begin());
    else ga_lpt_order(n, in->pat_len, ord.data());  // longest first: no straggler at the end
    cudaStream_t st = c->stream;
    const struct { void* d; const void* h; size_t b; } cp[] = {
        {c->dp_in.ptr, in->codes, (size_t)std::max<int64_t>(in->codes_len, 0)},
        {pat_off, in->pat_off, (size_t)n * 8}, {txt_off, in->txt_off, (size_t)n * 8},
        {pat_len, in->pat_len, (size_t)n * 4}, {txt_len, in->txt_len, (size_t)n * 4},
        {order, ord.data(), (size_t)n * 4}};
    for (const auto& x : cp)
        if (x.b && (e = cudaMemcpyAsync(x.d, x.h, x.b, cudaMemcpyHostToDevice, st)))
            return fail(c, e, "H2D (edit distance)");
    e = genasm::launch_edit_distance((const uint8_t*)c->dp_in.ptr, pat_off, pat_len, txt_off, txt_len,
                                     order, n, max_words, semiglobal, (int64_t*)c->dp_out.ptr,
                                     c->num_sms, st, &c->dp_slab, &c->dp_cap, c->scratch.queue);
    if (e != cudaSuccess) return fail(c, e, "edit distance kernel");
    if ((e = cudaMemcpyAsync(dist, c->dp_out.ptr, (size_t)n * 8, cudaMemcpyDeviceToHost, st)) ||
        (e = cudaStreamSynchronize(st)))
        return fail(c, e, "edit distance");
    c->launches = 1;
    return 0;
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
    if (in->packed2 || out->ops2) {  // the transfer formats belong to the host-buffer call
        c->err = "ga_align_batch_device takes 1-byte codes and writes ASCII ops (packed2/ops2 are "
                 "ga_align_batch formats)";
        return -3;
    }
    if (in->n_pairs <= 0) return 0;
    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) return fail(c, e, "cudaSetDevice");
    cudaStream_t st = stream_ptr ? (cudaStream_t)stream_ptr : c->stream;
    const int rc = launch_batch(c, in, cfg, out, st, &c->scratch);
    if (rc == 0) c->launches = c->last_shape.launches;
    return rc;
}

static int align_chunks(ga_ctx* c, const ga_batch_in* in, const ga_config* cfg, ga_batch_out* out);

int ga_align_batch(ga_ctx* c, const ga_batch_in* in, const ga_config* cfg, ga_batch_out* out) {
    if (!c) return -1;
    char msg[160];
    if (ga_check_config(cfg, msg, sizeof msg)) {
        c->err = msg;
        return -2;
    }
    const int64_t n = in->n_pairs;
    c->launches = 0;
    if (in->packed2 < 0 || in->packed2 > GA_PACK_HOST) {
        c->err = "packed2 must be 0 (bytes), 1 (2-bit input) or 2 (bytes packed per chunk by the call)";
        return -3;
    }
    if (n <= 0) return 0;
    if (out->ops2) {
        for (int64_t q = 0; q < n; ++q)
            if (out->ops_off[q] & 3) {
                c->err = "ops2 output needs every ops_off to be a multiple of 4";
                return -3;
            }
    }
    // every sequence inside codes_len, every pair's outputs inside the capacities
    for (int64_t q = 0; q < n; ++q) {
        const int64_t lp = in->pat_len[q], lt = in->txt_len[q];
        if (lp < 0 || lt < 0 || in->pat_off[q] < 0 || in->txt_off[q] < 0 ||
            in->pat_off[q] + lp > in->codes_len || in->txt_off[q] + lt > in->codes_len ||
            out->ops_off[q] < 0 || out->ops_off[q] + lp + lt > out->ops_capacity ||
            out->win_off[q] < 0 ||
            out->win_off[q] + ga_num_windows(lp, cfg->window, cfg->overlap) > out->win_capacity) {
            c->err = "pair " + std::to_string(q) + ": a sequence or output range is out of bounds";
            return -3;
        }
    }
    if (in->order) {  // a caller's order must be a permutation of 0..n-1
        std::vector<uint8_t> seen((size_t)n, 0);
        for (int64_t q = 0; q < n; ++q) {
            const int32_t v = in->order[q];
            if (v < 0 || v >= n || seen[(size_t)v]) {
                c->err = "order is not a permutation of 0.." + std::to_string(n - 1) +
                         " (entry " + std::to_string(q) + ")";
                return -3;
            }
            seen[(size_t)v] = 1;
        }
    }
    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) return fail(c, e, "cudaSetDevice");
    const int rc = align_chunks(c, in, cfg, out);
    if (rc != 0) {
        // chunks already enqueued may still be copying into the caller's
        // buffers: drain every stream before the error reaches the caller
        cudaStreamSynchronize(c->stream_in);
        for (Slot& sl : c->slot)
            if (sl.stream) cudaStreamSynchronize(sl.stream);
        cudaStreamSynchronize(c->stream_out);
    }
    return rc;
}

// the chunked pipeline of ga_align_batch (inputs validated by the caller)
static int align_chunks(ga_ctx* c, const ga_batch_in* in, const ga_config* cfg, ga_batch_out* out) {
    const int64_t n = in->n_pairs;
    // 2-bit transfer: the caller's packed array (1) or per-chunk packing into
    // pinned staging here, overlapping the previous chunk's copy (2)
    const bool xfer2 = in->packed2 != 0, host_pack = in->packed2 == GA_PACK_HOST;
    cudaError_t e;
    // ---- chunk plan: consecutive pairs, pipelined over kSlots slots.  Chunking
    // needs output offsets that grow with the input index (the prefix-sum
    // layout every caller in this package uses); otherwise one chunk. ----
    // One chunk per ~512 MB of sequence, at most 4: below that a batch's copy
    // is short against its kernel and pipelining gains nothing; above, the
    // copy of chunk k+1 hides under chunk k's kernel.
    int64_t seq_bytes = 0;
    for (int64_t q = 0; q < n; ++q) seq_bytes += (int64_t)in->pat_len[q] + in->txt_len[q];
    int chunks = env_int("GA_CHUNKS", (int)std::min<int64_t>(4, std::max<int64_t>(1, (seq_bytes + (256 << 20)) >> 29)));
    if (chunks < 1) chunks = 1;
    if (chunks > n) chunks = (int)n;
    for (int64_t q = 1; q < n && chunks > 1; ++q)
        if (out->ops_off[q] < out->ops_off[q - 1] || out->win_off[q] < out->win_off[q - 1])
            chunks = 1;
    // chunk boundaries: equal by default; GA_CHUNK_PLAN="w0,w1,..." weights (a
    // small first chunk starts the kernels early, a small last one shortens
    // the drain)
    std::vector<int64_t> cut;
    {
        std::vector<double> wts;
        const char* plan = getenv("GA_CHUNK_PLAN");
        for (const char* s = plan; s && *s;) {
            char* end = nullptr;
            const double v = strtod(s, &end);
            if (end == s) break;
            if (v > 0) wts.push_back(v);
            s = *end == ',' ? end + 1 : end;
        }
        if (!plan && chunks >= 3) {
            // twice the chunks, the first and last half-size: the kernels start
            // on a small first copy and the drain after the last copy is short
            // (tools/e2e_sweep.py on config 3: equal 4 chunks 71.5 ms, this 66.4)
            wts.assign((size_t)(2 * chunks), 2.0);
            wts.front() = wts.back() = 1.0;
        }
        if (wts.size() < 2 || (int64_t)wts.size() > n) wts.assign((size_t)chunks, 1.0);
        if (chunks == 1) wts.assign(1, 1.0);
        chunks = (int)wts.size();
        double tot = 0, acc = 0;
        for (double v : wts) tot += v;
        cut.push_back(0);
        for (double v : wts) {
            acc += v;
            cut.push_back(std::min<int64_t>(n, (int64_t)(n * (acc / tot) + 0.5)));
        }
        cut.back() = n;
    }
    int64_t launches = 0;
    for (int k = 0; k < chunks; ++k) {
        const int64_t q0 = cut[k], q1 = cut[k + 1];
        if (q1 <= q0) continue;
        const int64_t m = q1 - q0;
        Slot& S = c->slot[k % kSlots];
        // the symbol range the chunk reads
        int64_t lo = INT64_MAX, hi = 0;
        for (int64_t q = q0; q < q1; ++q) {
            lo = std::min(lo, std::min(in->pat_off[q], in->txt_off[q]));
            hi = std::max(hi, std::max(in->pat_off[q] + in->pat_len[q], in->txt_off[q] + in->txt_len[q]));
        }
        if (lo > hi) lo = hi;
        // the op and window ranges it writes: up to the next chunk's first pair
        int64_t olo, ohi, wlo, whi;
        if (chunks == 1) {
            olo = *std::min_element(out->ops_off, out->ops_off + n);
            wlo = *std::min_element(out->win_off, out->win_off + n);
            ohi = out->ops_capacity;
            whi = out->win_capacity;
        } else {
            olo = out->ops_off[q0];
            wlo = out->win_off[q0];
            ohi = q1 < n ? out->ops_off[q1] : out->ops_capacity;
            whi = q1 < n ? out->win_off[q1] : out->win_capacity;
        }
        const int64_t base = xfer2 ? (lo & ~int64_t(3)) : lo;
        const int64_t nsym = hi - base;
        const int64_t nops = ohi - olo;
        const int64_t nwin = whi - wlo;
        int64_t nexc = 0, exc0 = 0;
        if (in->packed2 == 1 && in->n_exceptions > 0) {
            const int64_t* x0 = std::lower_bound(in->exceptions, in->exceptions + in->n_exceptions, base);
            const int64_t* x1 = std::lower_bound(x0, in->exceptions + in->n_exceptions, hi);
            exc0 = x0 - in->exceptions;
            nexc = x1 - x0;
        }

        // ---- the slot is free once its previous chunk's copies are done ----
        if (S.used && (e = cudaEventSynchronize(S.in_done))) return fail(c, e, "slot wait");
        const size_t meta_bytes = (size_t)m * 44;
        if (meta_bytes > S.h_meta_cap) {
            if (S.h_meta) cudaFreeHost(S.h_meta);
            S.h_meta = nullptr;
            S.h_meta_cap = 0;
            if ((e = cudaHostAlloc(&S.h_meta, meta_bytes, cudaHostAllocDefault)))
                return fail(c, e, "cudaHostAlloc");
            S.h_meta_cap = meta_bytes;
        }
        int64_t* h64 = (int64_t*)S.h_meta;
        int32_t* h32 = (int32_t*)(h64 + 4 * m);
        for (int64_t q = 0; q < m; ++q) {
            h64[q] = in->pat_off[q0 + q] - base;
            h64[m + q] = in->txt_off[q0 + q] - base;
            h64[2 * m + q] = out->ops_off[q0 + q] - olo;
            h64[3 * m + q] = out->win_off[q0 + q] - wlo;
        }
        memcpy(h32, in->pat_len + q0, (size_t)m * 4);
        memcpy(h32 + m, in->txt_len + q0, (size_t)m * 4);
        if (in->order && chunks == 1) memcpy(h32 + 2 * m, in->order, (size_t)m * 4);
        else ga_lpt_order(m, in->pat_len + q0, h32 + 2 * m);

        if ((e = S.codes.ensure((size_t)nsym + 16)) || (e = S.meta.ensure(meta_bytes)) ||
            (e = S.results.ensure((size_t)m * sizeof(ga_pair_result))) ||
            (e = S.ops.ensure((size_t)nops + 16)) || (e = S.dists.ensure((size_t)nwin + 16)))
            return fail(c, e, "cudaMalloc");
        if (host_pack) {  // pack [base, hi) into the slot's pinned staging (free: in_done passed)
            const size_t pk = (size_t)(nsym + 3) / 4 + 16;
            if ((e = S.h_pack.ensure(pk)) || (e = S.h_exc.ensure(S.h_exc.cap ? S.h_exc.cap : 8192)))
                return fail(c, e, "cudaHostAlloc");
            nexc = ga_pack2(in->codes + base, nsym, (uint8_t*)S.h_pack.ptr, (int64_t*)S.h_exc.ptr,
                            (int64_t)(S.h_exc.cap / 8));
            if ((size_t)nexc * 8 > S.h_exc.cap) {  // rare: more code-4 symbols than staged room
                if ((e = S.h_exc.ensure((size_t)nexc * 8))) return fail(c, e, "cudaHostAlloc");
                ga_pack2(in->codes + base, nsym, (uint8_t*)S.h_pack.ptr, (int64_t*)S.h_exc.ptr, nexc);
            }
        }
        if (xfer2 && ((e = S.packed.ensure((size_t)(nsym + 3) / 4 + 16)) ||
                      (e = S.exc.ensure((size_t)(nexc > 0 ? nexc : 1) * 8))))
            return fail(c, e, "cudaMalloc");
        if (out->ops2 && (e = S.ops2.ensure((size_t)(nops + 3) / 4 + 16)))
            return fail(c, e, "cudaMalloc");

        // ---- H2D on the input stream, after the slot's previous chunk left the device ----
        cudaStream_t si = c->stream_in, sk = S.stream, so = c->stream_out;
        if (S.used && (e = cudaStreamWaitEvent(si, S.out_done, 0))) return fail(c, e, "wait");
        auto h2d = [&](void* dst, const void* src, size_t bytes) -> cudaError_t {
            return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, si) : cudaSuccess;
        };
        e = h2d(S.meta.ptr, S.h_meta, meta_bytes);
        if (!e) {
            if (host_pack) {
                e = h2d(S.packed.ptr, S.h_pack.ptr, (size_t)(nsym + 3) / 4);
                if (!e && nexc) e = h2d(S.exc.ptr, S.h_exc.ptr, (size_t)nexc * 8);
            } else if (xfer2) {
                e = h2d(S.packed.ptr, in->codes + base / 4, (size_t)(nsym + 3) / 4);
                if (!e && nexc) e = h2d(S.exc.ptr, in->exceptions + exc0, (size_t)nexc * 8);
            } else {
                e = h2d(S.codes.ptr, in->codes + base, (size_t)nsym);
            }
        }
        if (!e) e = cudaEventRecord(S.in_done, si);
        if (e) return fail(c, e, "H2D copy");
        S.used = true;

        // ---- the slot's kernel stream: expand 2-bit sequences, align, pack ops ----
        if ((e = cudaStreamWaitEvent(sk, S.in_done, 0))) return fail(c, e, "wait");
        if (xfer2) {  // host-packed exceptions are chunk-relative already
            if ((e = genasm::launch_unpack2((const uint8_t*)S.packed.ptr, nsym, (uint8_t*)S.codes.ptr,
                                            sk)) ||
                (e = genasm::launch_patch((const int64_t*)S.exc.ptr, nexc, host_pack ? 0 : base,
                                          (uint8_t*)S.codes.ptr, sk)))
                return fail(c, e, "unpack kernel");
            launches += 1 + (nexc > 0);
        }
        const int64_t* d64 = (const int64_t*)S.meta.ptr;
        const int32_t* d32 = (const int32_t*)(d64 + 4 * m);
        ga_batch_in din{};
        din.n_pairs = m;
        din.codes = (const uint8_t*)S.codes.ptr;
        din.codes_len = nsym;
        din.pat_off = d64;
        din.txt_off = d64 + m;
        din.pat_len = d32;
        din.txt_len = d32 + m;
        din.order = d32 + 2 * m;
        ga_batch_out dout{};
        dout.results = (ga_pair_result*)S.results.ptr;
        dout.ops_off = d64 + 2 * m;
        dout.ops = (uint8_t*)S.ops.ptr;
        dout.ops_capacity = nops;
        dout.win_off = d64 + 3 * m;
        dout.window_distances = (uint8_t*)S.dists.ptr;
        dout.win_capacity = nwin;
        const int rc = launch_batch(c, &din, cfg, &dout, sk, &S.scratch, chunks > 1);
        if (rc) return rc;
        launches += c->last_shape.launches;
        if (out->ops2) {
            if ((e = genasm::launch_pack_ops((const uint8_t*)S.ops.ptr, nops, (uint8_t*)S.ops2.ptr, sk)))
                return fail(c, e, "pack kernel");
            launches += 1;
        }
        if ((e = cudaEventRecord(S.kern_done, sk))) return fail(c, e, "record");

        // ---- D2H on the output stream ----
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
