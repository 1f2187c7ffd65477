// C ABI (include/refusion_b200.h) over the CUDA kernels: volume / pipeline
// objects, device buffers, frame upload and the per-frame launch sequence.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/refusion_b200.h"
#include "rf_host.cuh"
#include "rf_track.cuh"
#include "rf_volume.cuh"

namespace rfb {
// Per-frame results written by the GPU straight into mapped pinned host
// memory, then a sequence number the host spins on: replaces two D2H copies
// and a stream synchronisation at the end of every ProcessFrame.
struct FrameSignal {
    TrackOut out;
    uint32_t counters[kNumCounters];
    unsigned long long t_start;  // %globaltimer before the batch's first frame (record 0 only)
    unsigned long long t_end;    // %globaltimer when the frame's work completed
    unsigned long long seq;
};
__global__ void k_stamp(FrameSignal* sig) {
    if (threadIdx.x == 0) sig->t_start = global_ns();
}
__global__ void k_signal(const TrackOut* out, const uint32_t* counters, FrameSignal* sig, unsigned long long seq) {
    pdl_enter();
    if (threadIdx.x == 0) sig->t_end = global_ns();
    const uint32_t* src = reinterpret_cast<const uint32_t*>(out);
    uint32_t* dst = reinterpret_cast<uint32_t*>(&sig->out);
    for (int i = threadIdx.x; i < int(sizeof(TrackOut) / 4); i += blockDim.x) dst[i] = __ldcg(src + i);
    if (threadIdx.x < kNumCounters) sig->counters[threadIdx.x] = __ldcg(counters + threadIdx.x);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        *reinterpret_cast<volatile unsigned long long*>(&sig->seq) = seq;
    }
}
__global__ void k_track(TrackArgs a);
__global__ void k_import(VolumeView V, const int* coords, uint32_t n, uint32_t base) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int x = coords[3 * i], y = coords[3 * i + 1], z = coords[3 * i + 2];
    const unsigned long long key = pack_key(x, y, z);
    uint32_t idx = hash_coord(x, y, z) & V.hash_mask;
    while (atomicCAS(&V.slots[idx].key, kEmptyKey, key) != kEmptyKey) idx = (idx + 1) & V.hash_mask;
    V.slots[idx].value = base + i;
    V.coords[base + i] = make_int4(x, y, z, int(idx));
}
// Start of an allocation (AllocateForFrame / AllocateBlock batch): snapshot
// the brick count (assign_new numbers new bricks from it) and clear the
// per-allocation counters. The per-frame path does this inside k_track.
__global__ void k_alloc_begin(uint32_t* c, uint32_t max_blocks) {
    if (threadIdx.x == 0) {
        c[kBlocksBefore] = min(c[kNumBlocks], max_blocks);
        c[kOverflow] = 0;
        c[kVisible] = 0;
        c[kDdaVisits] = 0;
        c[kNewBlocks] = 0;
    }
}
// FindBlock (tsdf_volume.cpp:59-62): one probe, then the brick's 512 voxels
// (one per thread) copied to / from `io`.
__global__ void k_block_rw(VolumeView V, int x, int y, int z, uint2* io, int* found, int write) {
    __shared__ uint32_t b;
    if (threadIdx.x == 0) {
        b = hash_find(V, x, y, z);
        *found = b != kInvalid;
    }
    __syncthreads();
    if (b == kInvalid) return;
    uint2* vox = reinterpret_cast<uint2*>(V.voxels + size_t(b) * kBrickVoxels) + threadIdx.x;
    if (write) *vox = io[threadIdx.x];
    else io[threadIdx.x] = *vox;
}
// Sticky halt of the model volume when the refinement temp volume overflowed
// (RenderVirtualDepth throws before anything else of the frame runs).
__global__ void k_halt_if(const uint32_t* src, uint32_t* halt) {
    if (threadIdx.x == 0 && *src) *halt = 1u;
}
// Re-inserts bricks [0, n) into an emptied table (after an overflow left
// pending keys behind): the occupied-slot set is again exactly the allocated
// keys', as in the reference, whose AllocateBlock threw before inserting.
__global__ void k_rehash(VolumeView V, uint32_t n) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n) return;
    const int4 c = V.coords[b];
    const unsigned long long key = pack_key(c.x, c.y, c.z);
    uint32_t idx = hash_coord(c.x, c.y, c.z) & V.hash_mask;
    while (atomicCAS(&V.slots[idx].key, kEmptyKey, key) != kEmptyKey) idx = (idx + 1) & V.hash_mask;
    V.slots[idx].value = b;
    V.coords[b].w = int(idx);
}
}  // namespace rfb

using namespace rfb;

namespace rfb {
thread_local std::string g_err;
}  // namespace rfb

namespace {

// Per-frame kernels launch with programmatic stream serialization (the
// kernels call pdl_enter()); RF_PDL=0 turns it off (A/B runs).
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("RF_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}
template <class... P, class... A>
void launch(void (*k)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool cooperative, A&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    int n = 0;
    if (pdl_enabled()) {
        at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[n++].val.programmaticStreamSerializationAllowed = 1;
    }
    if (cooperative) {
        at[n].id = cudaLaunchAttributeCooperative;
        at[n++].val.cooperative = 1;
    }
    cfg.attrs = at;
    cfg.numAttrs = n;
    CK(cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...));
}

// Per-object scratch: stream, frame images, pyramid, grid-sync state.
struct Workspace {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = true;  // false when borrowed from another object (refinement temp volume)
    int track_grid = 0;
    int parity = 0;  // alternates the grid-barrier counter between cooperative launches
    DevBuf depth, rgb, mask_in, pose, res_sq, res_valid, mwork, levels, gsync, partials, result, out, list;
    DevBuf ll;                // the all-reduce's flagged lines (rf_grid.cuh block_grid_allreduce)
    uint32_t ll_seq = 0;      // launch sequence number of the flags
    DevBuf trace;            // per-pass timeline when RF_TRACE_FILE is set (diagnostics)
    std::string trace_path;
    TrackOut* h_out = nullptr;
    uint32_t* h_counters = nullptr;
    static constexpr int kSigSlots = 64;  // frames in flight per batch (rf_pipeline_process_frames)
    FrameSignal* h_sig = nullptr;          // kSigSlots records, mapped pinned (k_signal)
    FrameSignal* d_sig = nullptr;
    unsigned long long sig_seq = 0;
    int W = 0, H = 0, L = 0;
    int pxc_steps = 0, dyn_bytes = 16;  // the tracking kernel's dynamic shared memory for this frame size
    size_t lvl_off_depth[kMaxLevels] = {}, lvl_off_inten[kMaxLevels] = {}, lvl_off_mask[kMaxLevels] = {};

    void init(int dev) {
        device = dev;
        CK(cudaSetDevice(dev));
        CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        int sms = 0, per = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        // The tracking passes gather voxels through L1: leave it as much of the
        // unified L1/shared array as the kernel's static shared memory allows.
        CK(cudaFuncSetAttribute((const void*)k_track, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kTrackMaxDynSmem)));
        CK(cudaFuncSetAttribute((const void*)k_track, cudaFuncAttributePreferredSharedMemoryCarveout,
                                int(cudaSharedmemCarveoutMaxL1)));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_track, kTrackThreads, kTrackMaxDynSmem));
        require(per > 0, RF_CUDA_ERROR, "tracking kernel does not fit on an SM");
        track_grid = sms * per;
        gsync.ensure(sizeof(GridSync));
        CK(cudaMemset(gsync.p, 0, sizeof(GridSync)));
        partials.ensure(2 * size_t(track_grid) * kRedStride * sizeof(double));
        ll.ensure(2 * size_t(track_grid) * 32 * sizeof(uint4));
        CK(cudaMemset(ll.p, 0, ll.n));
        result.ensure(kRedStride * sizeof(double));
        out.ensure(sizeof(TrackOut));
        pose.ensure(12 * sizeof(double));
        CK(cudaMallocHost(&h_out, sizeof(TrackOut)));
        CK(cudaMallocHost(&h_counters, kNumCounters * sizeof(uint32_t)));
        CK(cudaHostAlloc(reinterpret_cast<void**>(&h_sig), kSigSlots * sizeof(FrameSignal), cudaHostAllocMapped));
        std::memset(h_sig, 0, kSigSlots * sizeof(FrameSignal));
        CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_sig), h_sig, 0));
        if (const char* tf = std::getenv("RF_TRACE_FILE")) {
            trace_path = tf;
            trace.ensure(kTracePasses * 8 * sizeof(unsigned long long));
        }
    }
    void destroy() {
        for (DevBuf* b : {&depth, &rgb, &mask_in, &pose, &res_sq, &res_valid, &mwork, &levels, &gsync, &partials,
                          &result, &out, &list, &trace, &ll})
            b->release();
        if (h_out) cudaFreeHost(h_out);
        if (h_counters) cudaFreeHost(h_counters);
        if (h_sig) cudaFreeHost(h_sig);
        h_sig = nullptr;
        if (stream && own_stream) cudaStreamDestroy(stream);
        h_out = nullptr;
        h_counters = nullptr;
        stream = nullptr;
    }
    void ensure_frame(int w, int h, int levels_needed) {
        if (w == W && h == H && levels_needed <= L) return;
        {  // pixel cache: one entry per pixel step of the finest level (the coarser ones need fewer);
           // at least the floodfill's tile flags (ff_flag_mode); the excess of huge frames reloads
            const size_t npx = size_t(w) * h, per = (npx + track_grid - 1) / track_grid;
            const size_t steps = (per + kTrackThreads - 1) / kTrackThreads;
            const size_t nft = size_t((w + 31) / 32) * ((h + 31) / 32);
            size_t bytes = std::max(steps * kTrackThreads * 8, ((nft + 15) & ~size_t(15)) + 2 * nft);
            bytes = std::min((bytes + 15) & ~size_t(15), kTrackMaxDynSmem);
            pxc_steps = int(std::min(steps, bytes / (size_t(kTrackThreads) * 8)));
            dyn_bytes = int(bytes);
        }
        const size_t n = size_t(w) * h;
        depth.ensure(n * 4);
        rgb.ensure(n * 3);
        mask_in.ensure(n);
        res_sq.ensure(n * 4);
        res_valid.ensure(n);
        const size_t nft = size_t((w + 31) / 32) * ((h + 31) / 32);
        mwork.ensure(ff_offset(w, h) + 4 * (3 * nft + 64));  // 3 masks + grow bits + floodfill worklists
        size_t off = 0;
        for (int l = 0; l < levels_needed; ++l) {
            const size_t nl = size_t(w >> l) * (h >> l);
            lvl_off_depth[l] = off;
            off += (nl * 4 + 255) & ~size_t(255);
            lvl_off_inten[l] = off;
            off += (nl * 4 + 255) & ~size_t(255);
            lvl_off_mask[l] = off;
            off += (nl + 255) & ~size_t(255);
        }
        levels.ensure(off + 256);
        W = w;
        H = h;
        L = levels_needed;
    }
    void sync() { CK(cudaStreamSynchronize(stream)); }
    // Grid-sync state for one cooperative launch: the barrier counters of this
    // launch's parity, and a fresh flag sequence number for the all-reduce
    // lines (after 2^20 - 1 launches the lines are cleared so no stale flag
    // can ever match).
    GridCtx grid() {
        GridCtx g{};
        g.sync = gsync.as<GridSync>();
        g.partials = partials.as<double>();
        g.result = result.as<double>();
        g.parity = parity;
        parity ^= 1;
        g.ll = ll.as<uint4>();
        if (++ll_seq >= (1u << 20)) {
            CK(cudaMemsetAsync(ll.p, 0, ll.n, stream));
            ll_seq = 1;
        }
        g.seq = ll_seq;
        return g;
    }
    // Enqueues k_signal after the frame's work: the frame's results land in
    // record `slot`, tagged with a new sequence number (returned).
    unsigned long long signal(const TrackOut* d_out, const uint32_t* d_counters, int slot) {
        const unsigned long long seq = ++sig_seq;
        launch(k_signal, 1, 128, 0, stream, false, d_out, d_counters, d_sig + slot, seq);
        return seq;
    }
    // Spins until record `slot` carries `seq` (stream errors surface, never a
    // spin on a dead stream), then copies it into h_out / h_counters.
    void wait_signal(int slot, unsigned long long seq) {
        const volatile unsigned long long* flag = &h_sig[slot].seq;
        for (unsigned long long spins = 1; *flag != seq; ++spins) {
            if ((spins & 0x3FFFu) == 0) {  // now and then: surface stream errors, never spin on a dead stream
                const cudaError_t e = cudaStreamQuery(stream);
                if (e != cudaSuccess && e != cudaErrorNotReady) CK(e);
                if (e == cudaSuccess && *flag != seq) CK(cudaErrorUnknown);
            }
        }
        std::atomic_thread_fence(std::memory_order_acquire);
        read_signal(slot);
    }
    void read_signal(int slot) {
        std::memcpy(h_out, const_cast<const TrackOut*>(&h_sig[slot].out), sizeof(TrackOut));
        std::memcpy(h_counters, const_cast<const uint32_t*>(h_sig[slot].counters), sizeof(h_sig[slot].counters));
    }
    void signal_wait(const TrackOut* d_out, const uint32_t* d_counters) { wait_signal(0, signal(d_out, d_counters, 0)); }
    // 3 masks, then the floodfill growth planes (8 words per row of every 32x32 tile), then the worklists
    static size_t ff_offset(int w, int h) {
        const size_t nft = size_t((w + 31) / 32) * ((h + 31) / 32);
        return (3 * size_t(w) * h + 255) / 256 * 256 + std::max(size_t(w) * h, nft * 8 * 32 * 4);
    }
    int* ffstamp() const { return reinterpret_cast<int*>(mwork.as<uint8_t>() + ff_offset(W, H)); }
};

Intr level_intr(const rf_intrinsics& k, int l) {  // CameraIntrinsics::Scaled (geometry.hpp:27-37)
    const double s = 1.0 / double(1 << l);
    Intr r;
    r.fx = k.fx * s;
    r.fy = k.fy * s;
    r.cx = k.cx * s;
    r.cy = k.cy * s;
    r.w = k.width >> l;
    r.h = k.height >> l;
    r.ifx = 1.0 / r.fx;
    r.ify = 1.0 / r.fy;
    return r;
}

uint64_t next_pow2(uint64_t v) {
    uint64_t c = 16;
    while (c < v) c <<= 1;
    return c;
}

void validate_volume_config(const rf_volume_config& c) {  // VolumeConfig::Validate (tsdf_volume.cpp:40-52)
    require(c.voxel_size > 0, RF_INVALID_ARGUMENT, "voxel_size must be positive");
    require(c.truncation >= c.voxel_size, RF_INVALID_ARGUMENT, "truncation must be at least one voxel_size");
    require(c.block_side >= 2, RF_INVALID_ARGUMENT, "block_side must be at least 2");
    require(c.max_weight >= 1 && c.max_weight <= 255, RF_INVALID_ARGUMENT, "max_weight must be in [1, 255]");
    require(c.carve_weight >= 1 && c.carve_weight <= c.max_weight, RF_INVALID_ARGUMENT,
            "carve_weight must be in [1, max_weight]");
    require(c.min_depth > 0 && c.max_depth > c.min_depth, RF_INVALID_ARGUMENT, "need 0 < min_depth < max_depth");
    require(c.carve_clip > 0, RF_INVALID_ARGUMENT, "carve_clip must be positive");
    require(c.max_blocks > 0, RF_INVALID_ARGUMENT, "max_blocks must be positive");
    require(c.block_side == kSide, RF_UNSUPPORTED, "the CUDA path supports block_side == 8 only");
    require(c.max_blocks < (1ull << 30), RF_UNSUPPORTED, "max_blocks must be < 2^30");
}

void check_reg_config(const rf_registration_config& r) {
    require(r.pyramid_levels >= 1, RF_INVALID_ARGUMENT, "pyramid_levels must be >= 1");
    require(r.pyramid_levels <= kMaxLevels, RF_UNSUPPORTED, "pyramid_levels > 6");
    require(r.max_iterations >= 1, RF_INVALID_ARGUMENT, "max_iterations must be >= 1");
    require(r.huber_depth >= 0 && r.huber_color >= 0, RF_INVALID_ARGUMENT, "huber thresholds must be >= 0");
}

}  // namespace

struct rf_volume {
    int device = 0;
    rf_volume_config cfg{};
    uint64_t cap = 0;
    DevBuf slots, coords, voxels, links, counters;
    DevBuf ord, newlist;  // allocation order (model volumes only, VolumeView::ord)
    DevBuf mesh_scratch;  // ExtractMesh's per-cell state, kept between calls
    DevBuf win_first;  // refinement temp volume: first window entry per hash slot
    VolumeView view{};
    Workspace ws;
    cudaEvent_t* prof = nullptr;  // stage markers when a pipeline profiles (see rf_pipeline_set_profiling)

    uint64_t num_blocks() {
        uint32_t c = 0;
        CK(cudaMemcpy(&c, view.counters + kNumBlocks, 4, cudaMemcpyDeviceToHost));
        return std::min<uint64_t>(c, cfg.max_blocks);
    }
    uint32_t overflow() {
        uint32_t c = 0;
        CK(cudaMemcpy(&c, view.counters + kOverflow, 4, cudaMemcpyDeviceToHost));
        return c;
    }
    // Uploads a frame's images into the workspace unless they already live on the device.
    const float* depth_of(const rf_frame* f) {
        const size_t n = size_t(f->intrinsics.width) * f->intrinsics.height;
        if (f->memory == RF_MEMORY_DEVICE) return f->depth;
        CK(cudaMemcpyAsync(ws.depth.p, f->depth, n * 4, cudaMemcpyHostToDevice, ws.stream));
        return ws.depth.as<float>();
    }
    const uint8_t* rgb_of(const rf_frame* f) {
        if (!f->rgb) return nullptr;
        const size_t n = size_t(f->intrinsics.width) * f->intrinsics.height;
        if (f->memory == RF_MEMORY_DEVICE) return f->rgb;
        CK(cudaMemcpyAsync(ws.rgb.p, f->rgb, n * 3, cudaMemcpyHostToDevice, ws.stream));
        return ws.rgb.as<uint8_t>();
    }
    const uint8_t* mask_of(const rf_frame* f, const uint8_t* mask, uint8_t* dst = nullptr) {
        if (!mask) return nullptr;
        const size_t n = size_t(f->intrinsics.width) * f->intrinsics.height;
        if (!dst) dst = ws.mask_in.as<uint8_t>();
        if (f->memory == RF_MEMORY_DEVICE) {
            if (dst == ws.mask_in.as<uint8_t>()) return mask;
            CK(cudaMemcpyAsync(dst, mask, n, cudaMemcpyDeviceToDevice, ws.stream));
        } else {
            CK(cudaMemcpyAsync(dst, mask, n, cudaMemcpyHostToDevice, ws.stream));
        }
        return dst;
    }
    void upload_pose(const double pose[12]) {
        CK(cudaMemcpyAsync(ws.pose.p, pose, 96, cudaMemcpyHostToDevice, ws.stream));
    }
    void prepare(const rf_frame* f, int levels = 1) {
        require(f && f->depth, RF_INVALID_ARGUMENT, "frame has no depth");
        require(f->intrinsics.width > 0 && f->intrinsics.height > 0, RF_INVALID_ARGUMENT, "bad image size");
        CK(cudaSetDevice(device));
        ws.ensure_frame(f->intrinsics.width, f->intrinsics.height, levels);
    }
    void reset_counter(int which) {
        CK(cudaMemsetAsync(view.counters + which, 0, 4, ws.stream));
    }
    // Back to the freshly created state; only the bricks in use are touched
    // unless an overflow left orphaned hash keys behind (full reset).
    void clear(bool full, bool voxels_too = true) {
        if (full) {
            CK(cudaMemsetAsync(slots.p, 0xFF, cap * sizeof(HashSlot), ws.stream));
            CK(cudaMemsetAsync(links.p, 0xFF, cap * kLinkStride * sizeof(uint32_t), ws.stream));
            CK(cudaMemsetAsync(voxels.p, 0, cfg.max_blocks * kBrickVoxels * sizeof(Voxel), ws.stream));
            if (win_first.p) CK(cudaMemsetAsync(win_first.p, 0xFF, cap * sizeof(uint32_t), ws.stream));
        } else {
            k_vol_clear<<<4 * 148, 128, 0, ws.stream>>>(view, voxels_too);
            CK(cudaGetLastError());
        }
        CK(cudaMemsetAsync(view.counters, 0, kNumCounters * sizeof(uint32_t), ws.stream));
    }
    void begin_alloc() {
        k_alloc_begin<<<1, 32, 0, ws.stream>>>(view.counters, uint32_t(cfg.max_blocks));
        CK(cudaGetLastError());
    }
    // Standalone allocation epilogue: pool indices for the claimed keys (model
    // volumes), then link records.
    void assign(int* created = nullptr) {
        if (view.ord) {
            k_assign<<<148, 256, 0, ws.stream>>>(view, created);
            CK(cudaGetLastError());
        }
        link();
    }
    // After an allocation overflowed (the host is about to throw
    // ResourceLimitError): the kept bricks are the first max_blocks in
    // allocation order already; drop the pending keys by rebuilding the table
    // from the bricks, relink, clear the sticky halt. Stream must be idle.
    void recover_overflow() {
        const uint64_t nb = num_blocks();
        CK(cudaMemsetAsync(slots.p, 0xFF, cap * sizeof(HashSlot), ws.stream));
        CK(cudaMemsetAsync(links.p, 0xFF, cap * kLinkStride * sizeof(uint32_t), ws.stream));
        if (ord.p) CK(cudaMemsetAsync(ord.p, 0xFF, cap * sizeof(unsigned long long), ws.stream));
        if (nb) k_rehash<<<unsigned((nb + 255) / 256), 256, 0, ws.stream>>>(view, uint32_t(nb));
        CK(cudaGetLastError());
        CK(cudaMemsetAsync(view.counters + kNewBlocks, 0, 4 * 4, ws.stream));  // kNewBlocks, kLinked, kLinkDone, kHalt
        CK(cudaMemsetAsync(view.counters + kOverflow, 0, 4, ws.stream));
        link();
        ws.sync();
    }
    // RenderVirtualDepth's temp-volume fusion (depth_refinement.cpp:25-30) of
    // n same-size entries, front to back, kMaxWin entries per alloc / cull /
    // fuse triple (rf_volume.cuh WindowArgs).
    struct WinIn {
        const float* depth;
        const uint8_t* rgb;
        const uint8_t* mask;
        const double* pose;  // device
        rf_intrinsics k;
        const int4* blist = nullptr;      // optional recorded brick list (device) ...
        const uint32_t* bcount = nullptr;  // ... and its length (device)
    };
    void fuse_window(const WinIn* in, int n) {
        if (!win_first.p) {
            win_first.ensure(cap * sizeof(uint32_t));
            CK(cudaMemsetAsync(win_first.p, 0xFF, cap * sizeof(uint32_t), ws.stream));
            view.win_first = win_first.as<uint32_t>();
        }
        ws.list.ensure(2 * cfg.max_blocks * sizeof(uint32_t));
        for (int c0 = 0; c0 < n; c0 += kMaxWin) {
            const int m = std::min(kMaxWin, n - c0);
            WindowArgs wa{};
            wa.V = view;
            wa.n = m;
            wa.list = ws.list.as<uint32_t>();
            for (int j = 0; j < m; ++j) {
                wa.depth[j] = in[c0 + j].depth;
                wa.rgb[j] = in[c0 + j].rgb;
                wa.mask[j] = in[c0 + j].mask;
                wa.pose[j] = in[c0 + j].pose;
                wa.K[j] = level_intr(in[c0 + j].k, 0);
                wa.blist[j] = in[c0 + j].blist;
                wa.bcount[j] = in[c0 + j].bcount;
            }
            if (c0 > 0) k_win_first_reset<<<148, 256, 0, ws.stream>>>(view);
            bool lists = false;
            for (int j = 0; j < m; ++j) lists = lists || in[c0 + j].bcount;
            if (lists) k_insert_window<<<2 * 148, 256, 0, ws.stream>>>(wa);
            // entries without a list (or whose list overflowed: decided on the device) walk their pixels
            const long long total = (long long)in[c0].k.width * in[c0].k.height * m;
            k_alloc_window<<<unsigned((total + 255) / 256), 256, 0, ws.stream>>>(wa);
            reset_counter(kVisible);
            k_cull_window<<<4 * 148, 256, 0, ws.stream>>>(wa);
            k_fuse_window<<<4 * 148, kBrickVoxels, 0, ws.stream>>>(wa);
            CK(cudaGetLastError());
        }
    }
    void link() {  // link records for bricks allocated outside the per-frame cull
        k_link<<<148, 256, 0, ws.stream>>>(view);
        k_link_commit<<<1, 32, 0, ws.stream>>>(view);
        CK(cudaGetLastError());
    }
    void fuse(const float* d, const uint8_t* rgb, const uint8_t* mask, const rf_intrinsics& k, const double* pose,
              const int* lost, bool carve, bool integrate, bool carve_only_before, bool reset_visible = true,
              bool assign = false) {
        // The visible list is appended to from counters[kVisible]; the frame
        // path's tracking kernel already zeroed it.
        if (reset_visible) reset_counter(kVisible);
        CullArgs ca{};
        ca.V = view;
        ca.K = level_intr(k, 0);
        ca.pose = pose;
        ca.lost = lost;
        ca.list = ws.list.as<uint32_t>();
        ca.do_carve = carve;
        ca.do_integrate = integrate;
        ca.carve_only_before = carve_only_before;
        ca.assign = assign && view.ord != nullptr;
        launch(k_cull, 4 * 148, 256, 0, ws.stream, false, ca);
        if (prof) CK(cudaEventRecord(prof[3], ws.stream));
        FuseArgs fa{};
        fa.V = view;
        fa.depth = d;
        fa.rgb = rgb;
        fa.mask = mask;
        fa.K = ca.K;
        fa.pose = pose;
        fa.lost = lost;
        fa.list = ca.list;
        launch(k_fuse, 4 * 148, kBrickVoxels, 0, ws.stream, false, fa);
    }
    void allocate(const float* d, const uint8_t* mask, const rf_intrinsics& k, const double* pose, const int* lost) {
        AllocArgs aa{};
        aa.V = view;
        aa.depth = d;
        aa.mask = mask;
        aa.K = level_intr(k, 0);
        aa.pose = pose;
        aa.lost = lost;
        const int n = k.width * k.height;
        launch(k_alloc, (n + 255) / 256, 256, 0, ws.stream, false, aa);
    }
    TrackArgs track_args(const rf_frame* f, const float* d, const uint8_t* rgb, int levels) {
        TrackArgs a{};
        a.V = view;
        a.F.depth0 = d;
        a.F.rgb0 = rgb;
        uint8_t* base = ws.levels.as<uint8_t>();
        for (int l = 0; l < levels; ++l) {
            a.F.K[l] = level_intr(f->intrinsics, l);
            a.F.depth[l] = reinterpret_cast<float*>(base + ws.lvl_off_depth[l]);
            a.F.inten[l] = reinterpret_cast<float*>(base + ws.lvl_off_inten[l]);
            a.F.mask[l] = base + ws.lvl_off_mask[l];
        }
        a.F.res_sq = ws.res_sq.as<float>();
        a.F.res_valid = ws.res_valid.as<uint8_t>();
        const size_t n = size_t(f->intrinsics.width) * f->intrinsics.height;
        for (int i = 0; i < 3; ++i) a.F.mwork[i] = ws.mwork.as<uint8_t>() + i * n;
        a.F.grow = ws.mwork.as<uint8_t>() + (3 * n + 255) / 256 * 256;
        a.F.ffstamp = ws.ffstamp();
        a.pose_state = ws.pose.as<double>();
        a.out = ws.out.as<TrackOut>();
        a.reg.levels = levels;
        a.trace = ws.trace.as<unsigned long long>();
        a.pxc_steps = ws.pxc_steps;
        a.dyn_bytes = ws.dyn_bytes;
        return a;
    }
    void dump_trace() {  // appends one frame's per-pass timeline (binary u64) to RF_TRACE_FILE
        if (!ws.trace.p) return;
        std::vector<unsigned long long> h(kTracePasses * 8);
        CK(cudaMemcpy(h.data(), ws.trace.p, h.size() * 8, cudaMemcpyDeviceToHost));
        if (FILE* f = std::fopen(ws.trace_path.c_str(), "ab")) {
            std::fwrite(h.data(), 8, h.size(), f);
            std::fclose(f);
        }
    }
    void launch_track(TrackArgs& a) {
        if (a.trace) CK(cudaMemsetAsync(a.trace, 0, kTracePasses * 8 * sizeof(unsigned long long), ws.stream));
        a.grid = ws.grid();
        launch(k_track, ws.track_grid, kTrackThreads, size_t(a.dyn_bytes), ws.stream, true, a);
    }
    TrackOut fetch_out() {
        CK(cudaMemcpyAsync(ws.h_out, ws.out.p, sizeof(TrackOut), cudaMemcpyDeviceToHost, ws.stream));
        ws.sync();
        return *ws.h_out;
    }
};

// Indexed triangle mesh resident on the device (Mesh, mesh.hpp:14-18).
struct rf_mesh {
    int device = 0;
    uint64_t nv = 0, nf = 0;
    DevBuf xyz, rgb, faces;
};

namespace {

RegParams to_reg(const rf_registration_config& c, int levels) {
    RegParams r;
    r.color_weight = c.color_weight;
    r.levels = levels;
    r.max_iterations = c.max_iterations;
    r.lambda_init = c.lm_lambda_init;
    r.lambda_up = c.lm_lambda_up;
    r.lambda_down = c.lm_lambda_down;
    r.eps = c.convergence_eps;
    r.min_valid = c.min_valid_residuals;
    r.huber_d = c.huber_depth;
    r.huber_c = c.huber_color;
    return r;
}

MaskParams to_mask(const rf_mask_config& c) {
    MaskParams m;
    m.gamma = c.gamma;
    m.truncation = c.truncation;
    m.theta = c.theta;
    m.erode_radius = c.erode_radius;
    m.dilate_radius = c.dilate_radius;
    m.connectivity = c.connectivity;
    m.free_space = c.free_space;
    return m;
}

void check_frame_dims(const rf_frame* f) {
    require(f && f->depth, RF_INVALID_ARGUMENT, "frame has no depth");
    require(f->intrinsics.width > 0 && f->intrinsics.height > 0, RF_INVALID_ARGUMENT, "bad image size");
}

void create_volume(const rf_volume_config* cfg, int device, rf_volume** out, bool ordered = true) {
    require(cfg && out, RF_INVALID_ARGUMENT, "null argument");
    validate_volume_config(*cfg);
    CK(cudaSetDevice(device));
    auto v = std::make_unique<rf_volume>();
    v->device = device;
    v->cfg = *cfg;
    // Default capacity: the reference's load bound (spatial_hash.hpp:51) for a
    // full pool, but at least 2^18 slots: an allocation that overflows keeps
    // its pending keys in the table until the pool indices are assigned, so the
    // table must hold one frame's distinct keys even when max_blocks is tiny.
    v->cap = cfg->hash_capacity ? cfg->hash_capacity
                                : std::max<uint64_t>(next_pow2((cfg->max_blocks * 4 + 2) / 3), uint64_t(1) << 18);
    require((v->cap & (v->cap - 1)) == 0 && v->cap <= (1ull << 31), RF_INVALID_ARGUMENT,
            "hash_capacity must be a power of two <= 2^31");
    require(v->cap >= cfg->max_blocks, RF_INVALID_ARGUMENT, "hash_capacity must be >= max_blocks");
    v->slots.ensure(v->cap * sizeof(HashSlot));
    v->coords.ensure(cfg->max_blocks * sizeof(int4));
    v->voxels.ensure(cfg->max_blocks * kBrickVoxels * sizeof(Voxel));
    v->links.ensure(v->cap * kLinkStride * sizeof(uint32_t));  // one record per hash slot
    v->counters.ensure(kNumCounters * sizeof(uint32_t));
    if (ordered) {
        v->ord.ensure(v->cap * sizeof(unsigned long long));
        v->newlist.ensure(v->cap * sizeof(uint32_t));
    }
    v->ws.init(device);
    if (ordered) CK(cudaMemsetAsync(v->ord.p, 0xFF, v->cap * sizeof(unsigned long long), v->ws.stream));
    CK(cudaMemsetAsync(v->slots.p, 0xFF, v->cap * sizeof(HashSlot), v->ws.stream));
    CK(cudaMemsetAsync(v->links.p, 0xFF, v->cap * kLinkStride * sizeof(uint32_t), v->ws.stream));
    CK(cudaMemsetAsync(v->voxels.p, 0, cfg->max_blocks * kBrickVoxels * sizeof(Voxel), v->ws.stream));
    CK(cudaMemsetAsync(v->counters.p, 0, kNumCounters * sizeof(uint32_t), v->ws.stream));
    v->ws.list.ensure(cfg->max_blocks * sizeof(uint32_t));
    VolumeView& V = v->view;
    V.slots = v->slots.as<HashSlot>();
    V.hash_mask = uint32_t(v->cap - 1);
    V.max_blocks = uint32_t(cfg->max_blocks);
    V.coords = v->coords.as<int4>();
    V.voxels = v->voxels.as<Voxel>();
    V.links = v->links.as<uint32_t>();
    V.counters = v->counters.as<uint32_t>();
    V.ord = ordered ? v->ord.as<unsigned long long>() : nullptr;
    V.newlist = ordered ? v->newlist.as<uint32_t>() : nullptr;
    V.voxel_size = cfg->voxel_size;
    V.inv_voxel_size = 1.0 / cfg->voxel_size;
    V.truncation = cfg->truncation;
    V.max_weight = cfg->max_weight;
    V.carve_weight = cfg->carve_weight;
    V.min_depth = cfg->min_depth;
    V.max_depth = cfg->max_depth;
    V.carve_clip = cfg->carve_clip;
    v->ws.sync();
    *out = v.release();
}

// Shared per-device workspace for the volume-less mask entry point.
std::mutex g_ws_mu;
std::map<int, Workspace*> g_ws;
Workspace& device_ws(int device) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    auto it = g_ws.find(device);
    if (it != g_ws.end()) return *it->second;
    auto* w = new Workspace();
    w->init(device);
    g_ws[device] = w;
    return *w;
}

}  // namespace

extern "C" {

const char* rf_last_error(void) { return g_err.c_str(); }
const char* rf_version(void) { return "refusion_b200 0.1 (sm_100a)"; }

rf_status rf_volume_create(const rf_volume_config* cfg, int device, rf_volume** out) {
    return guard([&] { create_volume(cfg, device, out); });
}

void rf_volume_destroy(rf_volume* v) {
    if (!v) return;
    cudaSetDevice(v->device);
    cudaStreamSynchronize(v->ws.stream);
    v->ws.destroy();
    v->slots.release();
    v->coords.release();
    v->voxels.release();
    v->links.release();
    v->counters.release();
    v->ord.release();
    v->newlist.release();
    v->mesh_scratch.release();
    v->win_first.release();
    delete v;
}

rf_status rf_volume_num_blocks(const rf_volume* v, uint64_t* out) {
    return guard([&] {
        require(v && out, RF_INVALID_ARGUMENT, "null argument");
        CK(cudaSetDevice(v->device));
        *out = const_cast<rf_volume*>(v)->num_blocks();
    });
}

rf_status rf_volume_hash_capacity(const rf_volume* v, uint64_t* out) {
    return guard([&] {
        require(v && out, RF_INVALID_ARGUMENT, "null argument");
        *out = v->cap;
    });
}

rf_status rf_volume_get_config(const rf_volume* v, rf_volume_config* out) {
    return guard([&] {
        require(v && out, RF_INVALID_ARGUMENT, "null argument");
        *out = v->cfg;
    });
}

rf_status rf_volume_allocate_blocks(rf_volume* v, const int32_t* coords, uint64_t n, int32_t* created) {
    return guard([&] {
        require(v && (coords || n == 0), RF_INVALID_ARGUMENT, "null argument");
        require(n < (1ull << 31), RF_INVALID_ARGUMENT, "too many coordinates in one call");
        if (n == 0) return;
        CK(cudaSetDevice(v->device));
        DevBuf dc, dr;
        dc.ensure(n * 12);
        dr.ensure(n * 4);
        CK(cudaMemcpyAsync(dc.p, coords, n * 12, cudaMemcpyHostToDevice, v->ws.stream));
        CK(cudaMemsetAsync(dr.p, 0, n * 4, v->ws.stream));
        v->begin_alloc();
        k_alloc_coords<<<unsigned((n + 255) / 256), 256, 0, v->ws.stream>>>(v->view, dc.as<int>(), int(n),
                                                                             dr.as<int>());
        CK(cudaGetLastError());
        v->assign(dr.as<int>());  // AllocateBlock in coordinate order (tsdf_volume.cpp:64-77)
        if (created) CK(cudaMemcpyAsync(created, dr.p, n * 4, cudaMemcpyDeviceToHost, v->ws.stream));
        v->ws.sync();
        dc.release();
        dr.release();
        if (v->overflow()) {
            v->recover_overflow();
            throw Error{RF_RESOURCE_LIMIT, "voxel block budget exhausted (" + std::to_string(v->cfg.max_blocks) + " blocks)"};
        }
    });
}

rf_status rf_volume_allocate_for_frame(rf_volume* v, const rf_frame* f, const double pose[12],
                                       const uint8_t* mask) {
    return guard([&] {
        require(v && pose, RF_INVALID_ARGUMENT, "null argument");
        v->prepare(f);
        const float* d = v->depth_of(f);
        const uint8_t* m = v->mask_of(f, mask);
        v->upload_pose(pose);
        v->begin_alloc();
        v->allocate(d, m, f->intrinsics, v->ws.pose.as<double>(), nullptr);
        v->assign();
        v->ws.sync();
        if (v->overflow()) {
            v->recover_overflow();
            throw Error{RF_RESOURCE_LIMIT, "voxel block budget exhausted (" + std::to_string(v->cfg.max_blocks) + " blocks)"};
        }
    });
}

rf_status rf_volume_integrate(rf_volume* v, const rf_frame* f, const double pose[12], const uint8_t* mask) {
    return guard([&] {
        require(v && pose, RF_INVALID_ARGUMENT, "null argument");
        v->prepare(f);
        const float* d = v->depth_of(f);
        const uint8_t* rgb = v->rgb_of(f);
        const uint8_t* m = v->mask_of(f, mask);
        v->upload_pose(pose);
        v->fuse(d, rgb, m, f->intrinsics, v->ws.pose.as<double>(), nullptr, false, true, false);
        v->ws.sync();
    });
}

rf_status rf_volume_carve(rf_volume* v, const rf_frame* f, const double pose[12]) {
    return guard([&] {
        require(v && pose, RF_INVALID_ARGUMENT, "null argument");
        v->prepare(f);
        const float* d = v->depth_of(f);
        v->upload_pose(pose);
        v->fuse(d, nullptr, nullptr, f->intrinsics, v->ws.pose.as<double>(), nullptr, true, false, false);
        v->ws.sync();
    });
}

rf_status rf_volume_sample(const rf_volume* cv, int32_t mode, const double* points, uint64_t n, double* value,
                           double* grad, uint8_t* valid) {
    return guard([&] {
        rf_volume* v = const_cast<rf_volume*>(cv);
        require(v && points && value && valid && mode >= 0 && mode <= 4, RF_INVALID_ARGUMENT, "bad argument");
        if (n == 0) return;
        CK(cudaSetDevice(v->device));
        DevBuf dp, dv, dg, dk;
        dp.ensure(n * 24);
        dv.ensure(n * 8);
        dg.ensure(n * 24);
        dk.ensure(n);
        CK(cudaMemcpyAsync(dp.p, points, n * 24, cudaMemcpyHostToDevice, v->ws.stream));
        k_sample<<<unsigned((n + 127) / 128), 128, 0, v->ws.stream>>>(v->view, dp.as<double>(), int(n), mode,
                                                                        dv.as<double>(), dg.as<double>(),
                                                                        dk.as<uint8_t>());
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(value, dv.p, n * 8, cudaMemcpyDeviceToHost, v->ws.stream));
        if (grad) CK(cudaMemcpyAsync(grad, dg.p, n * 24, cudaMemcpyDeviceToHost, v->ws.stream));
        CK(cudaMemcpyAsync(valid, dk.p, n, cudaMemcpyDeviceToHost, v->ws.stream));
        v->ws.sync();
    });
}

static rf_status voxel_rw(const rf_volume* cv, const int32_t* vc, uint64_t n, uint8_t* io, uint8_t* found,
                          uint64_t* missing, bool write) {
    return guard([&] {
        rf_volume* v = const_cast<rf_volume*>(cv);
        require(v && vc && io, RF_INVALID_ARGUMENT, "null argument");
        if (n == 0) {
            if (missing) *missing = 0;
            return;
        }
        CK(cudaSetDevice(v->device));
        DevBuf dc, dio, df;
        dc.ensure(n * 12);
        dio.ensure(n * 8);
        df.ensure(n);
        CK(cudaMemcpyAsync(dc.p, vc, n * 12, cudaMemcpyHostToDevice, v->ws.stream));
        if (write) CK(cudaMemcpyAsync(dio.p, io, n * 8, cudaMemcpyHostToDevice, v->ws.stream));
        k_voxel_rw<<<unsigned((n + 255) / 256), 256, 0, v->ws.stream>>>(v->view, dc.as<int>(), int(n),
                                                                          dio.as<Voxel>(), df.as<uint8_t>(),
                                                                          write ? 1 : 0);
        CK(cudaGetLastError());
        std::vector<uint8_t> hf(n);
        if (!write) CK(cudaMemcpyAsync(io, dio.p, n * 8, cudaMemcpyDeviceToHost, v->ws.stream));
        CK(cudaMemcpyAsync(hf.data(), df.p, n, cudaMemcpyDeviceToHost, v->ws.stream));
        v->ws.sync();
        uint64_t miss = 0;
        for (uint64_t i = 0; i < n; ++i) {
            if (!hf[i]) {
                ++miss;
                if (!write) std::memset(io + 8 * i, 0, 8);
            }
        }
        if (found) std::memcpy(found, hf.data(), n);
        if (missing) *missing = miss;
    });
}

rf_status rf_volume_get_voxels(const rf_volume* v, const int32_t* vc, uint64_t n, uint8_t* voxels,
                               uint8_t* found) {
    return voxel_rw(v, vc, n, voxels, found, nullptr, false);
}

rf_status rf_volume_set_voxels(rf_volume* v, const int32_t* vc, uint64_t n, const uint8_t* voxels,
                               uint64_t* missing) {
    return voxel_rw(v, vc, n, const_cast<uint8_t*>(voxels), nullptr, missing, true);
}

rf_status rf_volume_export_blocks(const rf_volume* cv, int32_t* coords, uint8_t* voxels, uint64_t capacity,
                                  uint64_t* count) {
    return guard([&] {
        rf_volume* v = const_cast<rf_volume*>(cv);
        require(v && count, RF_INVALID_ARGUMENT, "null argument");
        CK(cudaSetDevice(v->device));
        const uint64_t nb = v->num_blocks();
        *count = nb;
        if (!coords || capacity < nb || nb == 0) return;
        std::vector<int4> c(nb);
        CK(cudaMemcpy(c.data(), v->coords.p, nb * sizeof(int4), cudaMemcpyDeviceToHost));
        for (uint64_t i = 0; i < nb; ++i) {
            coords[3 * i] = c[i].x;
            coords[3 * i + 1] = c[i].y;
            coords[3 * i + 2] = c[i].z;
        }
        if (voxels) CK(cudaMemcpy(voxels, v->voxels.p, nb * kBrickVoxels * sizeof(Voxel), cudaMemcpyDeviceToHost));
    });
}

rf_status rf_volume_hash_occupancy(const rf_volume* cv, uint8_t* bitmap) {
    return guard([&] {
        rf_volume* v = const_cast<rf_volume*>(cv);
        require(v && bitmap, RF_INVALID_ARGUMENT, "null argument");
        CK(cudaSetDevice(v->device));
        DevBuf b;
        b.ensure(v->cap);
        k_occupancy<<<1024, 256, 0, v->ws.stream>>>(v->view, b.as<uint8_t>());
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(bitmap, b.p, v->cap, cudaMemcpyDeviceToHost, v->ws.stream));
        v->ws.sync();
    });
}

rf_status rf_volume_reset(rf_volume* v) {
    return guard([&] {
        require(v, RF_INVALID_ARGUMENT, "null argument");
        CK(cudaSetDevice(v->device));
        const uint64_t nb = v->num_blocks();
        CK(cudaMemsetAsync(v->slots.p, 0xFF, v->cap * sizeof(HashSlot), v->ws.stream));
        CK(cudaMemsetAsync(v->voxels.p, 0, nb * kBrickVoxels * sizeof(Voxel), v->ws.stream));
        CK(cudaMemsetAsync(v->links.p, 0xFF, v->cap * kLinkStride * sizeof(uint32_t), v->ws.stream));
        if (v->ord.p) CK(cudaMemsetAsync(v->ord.p, 0xFF, v->cap * sizeof(unsigned long long), v->ws.stream));
        CK(cudaMemsetAsync(v->counters.p, 0, kNumCounters * sizeof(uint32_t), v->ws.stream));
        v->ws.sync();
    });
}

// TsdfVolume::Save / Load (tsdf_volume.cpp:375-449): "TSDFVOL\0", u32 version 1,
// config, u64 block count, then per block i32[3] + 512 voxels, little-endian.
rf_status rf_volume_save(const rf_volume* cv, const char* path) {
    return guard([&] {
        rf_volume* v = const_cast<rf_volume*>(cv);
        require(v && path, RF_INVALID_ARGUMENT, "null argument");
        CK(cudaSetDevice(v->device));
        const uint64_t nb = v->num_blocks();
        std::vector<int4> c(nb);
        std::vector<Voxel> vox(nb * kBrickVoxels);
        if (nb) {
            CK(cudaMemcpy(c.data(), v->coords.p, nb * sizeof(int4), cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(vox.data(), v->voxels.p, vox.size() * sizeof(Voxel), cudaMemcpyDeviceToHost));
        }
        std::ofstream out(path, std::ios::binary);
        require(bool(out), RF_IO_ERROR, std::string("cannot open for writing: ") + path);
        const char magic[8] = {'T', 'S', 'D', 'F', 'V', 'O', 'L', '\0'};
        out.write(magic, 8);
        auto w = [&](const auto& x) { out.write(reinterpret_cast<const char*>(&x), sizeof(x)); };
        w(uint32_t(1));
        w(v->cfg.voxel_size);
        w(v->cfg.truncation);
        w(int32_t(v->cfg.block_side));
        w(int32_t(v->cfg.max_weight));
        w(int32_t(v->cfg.carve_weight));
        w(v->cfg.min_depth);
        w(v->cfg.max_depth);
        w(v->cfg.carve_clip);
        w(uint64_t(v->cfg.max_blocks));
        w(uint64_t(nb));
        for (uint64_t i = 0; i < nb; ++i) {
            const int32_t cc[3] = {c[i].x, c[i].y, c[i].z};
            out.write(reinterpret_cast<const char*>(cc), 12);
            out.write(reinterpret_cast<const char*>(&vox[i * kBrickVoxels]), kBrickVoxels * sizeof(Voxel));
        }
        require(bool(out), RF_IO_ERROR, std::string("write failed: ") + path);
    });
}

rf_status rf_volume_load(const char* path, int device, rf_volume** out) {
    return guard([&] {
        require(path && out, RF_INVALID_ARGUMENT, "null argument");
        std::ifstream in(path, std::ios::binary);
        require(bool(in), RF_IO_ERROR, std::string("cannot open volume snapshot: ") + path);
        char magic[8];
        in.read(magic, 8);
        require(bool(in) && std::memcmp(magic, "TSDFVOL\0", 8) == 0, RF_IO_ERROR,
                std::string("not a volume snapshot: ") + path);
        auto r = [&](auto& x) { in.read(reinterpret_cast<char*>(&x), sizeof(x)); };
        uint32_t version = 0;
        r(version);
        require(version == 1, RF_IO_ERROR, std::string("unsupported volume snapshot version in ") + path);
        rf_volume_config cfg{};
        int32_t bs, mw, cw;
        uint64_t mb, nb;
        r(cfg.voxel_size);
        r(cfg.truncation);
        r(bs);
        r(mw);
        r(cw);
        r(cfg.min_depth);
        r(cfg.max_depth);
        r(cfg.carve_clip);
        r(mb);
        r(nb);
        require(bool(in), RF_IO_ERROR, std::string("truncated volume snapshot: ") + path);
        cfg.block_side = bs;
        cfg.max_weight = mw;
        cfg.carve_weight = cw;
        cfg.max_blocks = mb;
        require(nb <= mb, RF_RESOURCE_LIMIT, "snapshot holds more blocks than max_blocks");
        std::vector<int32_t> coords(nb * 3);
        std::vector<Voxel> vox(nb * kBrickVoxels);
        for (uint64_t i = 0; i < nb; ++i) {
            in.read(reinterpret_cast<char*>(&coords[3 * i]), 12);
            in.read(reinterpret_cast<char*>(&vox[i * kBrickVoxels]), kBrickVoxels * sizeof(Voxel));
            require(bool(in), RF_IO_ERROR, std::string("truncated volume snapshot: ") + path);
        }
        rf_volume* v = nullptr;
        create_volume(&cfg, device, &v);
        std::unique_ptr<rf_volume, void (*)(rf_volume*)> hold(v, rf_volume_destroy);
        if (nb) {
            DevBuf dc;
            dc.ensure(nb * 12);
            CK(cudaMemcpy(dc.p, coords.data(), nb * 12, cudaMemcpyHostToDevice));
            k_import<<<unsigned((nb + 255) / 256), 256, 0, v->ws.stream>>>(v->view, dc.as<int>(), uint32_t(nb), 0);
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(v->voxels.p, vox.data(), vox.size() * sizeof(Voxel), cudaMemcpyHostToDevice,
                               v->ws.stream));
            const uint32_t cnt = uint32_t(nb);
            CK(cudaMemcpyAsync(v->view.counters + kNumBlocks, &cnt, 4, cudaMemcpyHostToDevice, v->ws.stream));
            v->link();
            v->ws.sync();
        }
        *out = hold.release();
    });
}

static rf_status block_rw(const rf_volume* cv, const int32_t c[3], uint8_t* io, int32_t* found, bool write) {
    return guard([&] {
        rf_volume* v = const_cast<rf_volume*>(cv);
        require(v && c && found && (io || !write), RF_INVALID_ARGUMENT, "null argument");
        CK(cudaSetDevice(v->device));
        DevBuf d;
        d.ensure(kBrickVoxels * sizeof(Voxel) + 16);
        int* dfound = reinterpret_cast<int*>(d.as<uint8_t>() + kBrickVoxels * sizeof(Voxel));
        if (write) CK(cudaMemcpyAsync(d.p, io, kBrickVoxels * sizeof(Voxel), cudaMemcpyHostToDevice, v->ws.stream));
        k_block_rw<<<1, kBrickVoxels, 0, v->ws.stream>>>(v->view, c[0], c[1], c[2], d.as<uint2>(), dfound, write);
        CK(cudaGetLastError());
        int f = 0;
        CK(cudaMemcpyAsync(&f, dfound, 4, cudaMemcpyDeviceToHost, v->ws.stream));
        v->ws.sync();
        *found = f;
        if (f && !write && io) CK(cudaMemcpy(io, d.p, kBrickVoxels * sizeof(Voxel), cudaMemcpyDeviceToHost));
    });
}

rf_status rf_volume_find_block(const rf_volume* v, const int32_t c[3], uint8_t* voxels, int32_t* found) {
    return block_rw(v, c, voxels, found, false);
}

rf_status rf_volume_write_block(rf_volume* v, const int32_t c[3], const uint8_t* voxels, int32_t* found) {
    return block_rw(v, c, const_cast<uint8_t*>(voxels), found, true);
}

// ---------------------------------------------------------------- registration
namespace {
// LinearizeResult::degenerate (registration.cpp:136-138): the eigenvalues of
// the symmetric 6x6 H (cyclic Jacobi rotations to convergence, in place of
// Eigen's SelfAdjointEigenSolver) and min(ev) <= 1e-12 * max(max |ev|, 1).
bool hessian_degenerate(const double* Hin, uint64_t valid) {
    if (valid == 0) return true;
    double A[6][6];
    for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j) A[i][j] = Hin[6 * i + j];
    for (int sweep = 0; sweep < 64; ++sweep) {
        double off = 0.0, diag = 0.0;
        for (int i = 0; i < 6; ++i) {
            diag += A[i][i] * A[i][i];
            for (int j = i + 1; j < 6; ++j) off += A[i][j] * A[i][j];
        }
        if (off <= 1e-34 * diag || off == 0.0) break;
        for (int p = 0; p < 5; ++p)
            for (int q = p + 1; q < 6; ++q) {
                if (A[p][q] == 0.0) continue;
                // rotation zeroing A[p][q]: tan(2 phi) = 2 A_pq / (A_qq - A_pp), smaller root
                const double zeta = (A[q][q] - A[p][p]) / (2.0 * A[p][q]);
                const double t = std::copysign(1.0, zeta) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / std::sqrt(1.0 + t * t), sn = t * c;
                for (int k = 0; k < 6; ++k) {  // columns p, q
                    const double kp = A[k][p], kq = A[k][q];
                    A[k][p] = c * kp - sn * kq;
                    A[k][q] = sn * kp + c * kq;
                }
                for (int k = 0; k < 6; ++k) {  // rows p, q
                    const double pk = A[p][k], qk = A[q][k];
                    A[p][k] = c * pk - sn * qk;
                    A[q][k] = sn * pk + c * qk;
                }
            }
    }
    double mn = A[0][0], mx = std::fabs(A[0][0]);
    for (int i = 1; i < 6; ++i) {
        mn = std::min(mn, A[i][i]);
        mx = std::max(mx, std::fabs(A[i][i]));
    }
    return mn <= 1e-12 * std::max(mx, 1.0);
}
}  // namespace

rf_status rf_build_pyramid(const rf_frame* f, const uint8_t* mask, int32_t levels, int device, float* depth,
                           float* intensity, uint8_t* mask_out, rf_intrinsics* k_out) {
    return guard([&] {
        require(levels >= 1, RF_INVALID_ARGUMENT, "pyramid needs at least one level");
        check_frame_dims(f);
        require(levels <= kMaxLevels, RF_UNSUPPORTED, "pyramid_levels > 6");
        for (int l = 1; l < levels; ++l)
            require((f->intrinsics.width >> l) >= 1 && (f->intrinsics.height >> l) >= 1, RF_INVALID_ARGUMENT,
                    "image too small for pyramid level");
        require(!intensity || f->rgb, RF_INVALID_ARGUMENT, "intensity levels need colour");
        require(!mask_out || mask, RF_INVALID_ARGUMENT, "mask levels need a mask");
        CK(cudaSetDevice(device));
        Workspace& ws = device_ws(device);
        const int w = f->intrinsics.width, h = f->intrinsics.height;
        ws.ensure_frame(w, h, levels);
        const size_t n = size_t(w) * h;
        const cudaMemcpyKind kind = f->memory == RF_MEMORY_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        CK(cudaMemcpyAsync(ws.depth.p, f->depth, n * 4, kind, ws.stream));
        if (f->rgb) CK(cudaMemcpyAsync(ws.rgb.p, f->rgb, n * 3, kind, ws.stream));
        uint8_t* base = ws.levels.as<uint8_t>();
        TrackArgs a{};
        a.mode = kModePyramid;
        a.reg.levels = levels;
        a.F.depth0 = ws.depth.as<float>();
        a.F.rgb0 = f->rgb ? ws.rgb.as<uint8_t>() : nullptr;
        for (int l = 0; l < levels; ++l) {
            a.F.K[l] = level_intr(f->intrinsics, l);
            a.F.depth[l] = reinterpret_cast<float*>(base + ws.lvl_off_depth[l]);
            a.F.inten[l] = reinterpret_cast<float*>(base + ws.lvl_off_inten[l]);
            a.F.mask[l] = base + ws.lvl_off_mask[l];
        }
        if (mask) {
            CK(cudaMemcpyAsync(a.F.mask[0], mask, n, kind, ws.stream));
            a.use_mask = 1;
        }
        a.pxc_steps = ws.pxc_steps;
        a.dyn_bytes = ws.dyn_bytes;
        a.grid = ws.grid();
        a.out = ws.out.as<TrackOut>();
        void* args[] = {&a};
        CK(cudaLaunchCooperativeKernel((void*)k_track, dim3(ws.track_grid), dim3(kTrackThreads), args, size_t(a.dyn_bytes),
                                       ws.stream));
        size_t off = 0;
        for (int l = 0; l < levels; ++l) {
            const size_t nl = size_t(w >> l) * size_t(h >> l);
            if (k_out) k_out[l] = rf_intrinsics{a.F.K[l].fx, a.F.K[l].fy, a.F.K[l].cx, a.F.K[l].cy, a.F.K[l].w,
                                                 a.F.K[l].h, f->intrinsics.depth_scale};
            if (depth) CK(cudaMemcpyAsync(depth + off, l ? (const void*)a.F.depth[l] : ws.depth.p, nl * 4,
                                          cudaMemcpyDeviceToHost, ws.stream));
            if (intensity) CK(cudaMemcpyAsync(intensity + off, a.F.inten[l], nl * 4, cudaMemcpyDeviceToHost, ws.stream));
            if (mask_out) CK(cudaMemcpyAsync(mask_out + off, a.F.mask[l], nl, cudaMemcpyDeviceToHost, ws.stream));
            off += nl;
        }
        ws.sync();
    });
}

static void run_pass(rf_volume* v, const rf_frame* f, const double pose[12], const uint8_t* mask, int mode,
                     double cw, TrackOut& out, const rf_registration_config* cfg = nullptr) {
    v->prepare(f);
    const float* d = v->depth_of(f);
    const uint8_t* rgb = v->rgb_of(f);
    TrackArgs a = v->track_args(f, d, rgb, 1);
    if (mask) {
        v->mask_of(f, mask, a.F.mask[0]);
        a.use_mask = 1;
    }
    v->upload_pose(pose);
    a.mode = mode;
    a.reg.color_weight = cw;
    a.reg.levels = 1;
    if (cfg) {
        a.reg.huber_d = cfg->huber_depth;
        a.reg.huber_c = cfg->huber_color;
    }
    v->launch_track(a);
    out = v->fetch_out();
}

rf_status rf_linearize(const rf_volume* cv, const rf_frame* f, const double pose[12],
                       const rf_registration_config* cfg, const uint8_t* mask, rf_linearize_result* out) {
    return guard([&] {
        rf_volume* v = const_cast<rf_volume*>(cv);
        require(v && pose && cfg && out, RF_INVALID_ARGUMENT, "null argument");
        TrackOut o;
        require(cfg->huber_depth >= 0 && cfg->huber_color >= 0, RF_INVALID_ARGUMENT, "huber thresholds must be >= 0");
        run_pass(v, f, pose, mask, kModeLinearize, cfg->color_weight, o, cfg);
        for (int i = 0, k = 0; i < 6; ++i)
            for (int j = i; j < 6; ++j, ++k) out->H[6 * i + j] = out->H[6 * j + i] = o.acc[k];
        for (int i = 0; i < 6; ++i) out->b[i] = o.acc[21 + i];
        out->depth_error = o.acc[27];
        out->color_error = o.acc[28];
        out->error = o.acc[27] + cfg->color_weight * o.acc[28];
        out->valid_count = uint64_t(o.acc[29]);
        out->degenerate = hessian_degenerate(out->H, out->valid_count) ? 1 : 0;
    });
}

rf_status rf_evaluate_depth_error(const rf_volume* cv, const rf_frame* f, const double pose[12], const uint8_t* mask,
                                  double* error, float* res_sq, uint8_t* res_valid) {
    return guard([&] {
        rf_volume* v = const_cast<rf_volume*>(cv);
        require(v && pose, RF_INVALID_ARGUMENT, "null argument");
        TrackOut o;
        run_pass(v, f, pose, mask, kModeEvalDepth, 0.0, o);
        if (error) *error = o.acc[27];
        const size_t n = size_t(f->intrinsics.width) * f->intrinsics.height;
        if (res_sq) CK(cudaMemcpy(res_sq, v->ws.res_sq.p, n * 4, cudaMemcpyDeviceToHost));
        if (res_valid) CK(cudaMemcpy(res_valid, v->ws.res_valid.p, n, cudaMemcpyDeviceToHost));
    });
}

rf_status rf_evaluate_color_error(const rf_volume* cv, const rf_frame* f, const double pose[12],
                                  const uint8_t* mask, double* error) {
    return guard([&] {
        rf_volume* v = const_cast<rf_volume*>(cv);
        require(v && pose && error, RF_INVALID_ARGUMENT, "null argument");
        TrackOut o;
        run_pass(v, f, pose, mask, kModeEvalColor, 1.0, o);
        *error = o.acc[28];
    });
}

rf_status rf_register(const rf_volume* cv, const rf_frame* f, const double init[12], const uint8_t* mask,
                      const rf_registration_config* cfg, rf_registration_result* out, float* res_sq,
                      uint8_t* res_valid) {
    return guard([&] {
        rf_volume* v = const_cast<rf_volume*>(cv);
        require(v && init && cfg && out, RF_INVALID_ARGUMENT, "null argument");
        check_reg_config(*cfg);
        check_frame_dims(f);
        for (int l = 1; l < cfg->pyramid_levels; ++l)
            require((f->intrinsics.width >> l) >= 1 && (f->intrinsics.height >> l) >= 1, RF_INVALID_ARGUMENT,
                    "image too small for pyramid level");
        v->prepare(f, cfg->pyramid_levels);
        const float* d = v->depth_of(f);
        const uint8_t* rgb = v->rgb_of(f);
        TrackArgs a = v->track_args(f, d, rgb, cfg->pyramid_levels);
        if (mask) {
            v->mask_of(f, mask, a.F.mask[0]);
            a.use_mask = 1;
        }
        v->upload_pose(init);
        a.mode = kModeRegister;
        a.reg = to_reg(*cfg, cfg->pyramid_levels);
        v->launch_track(a);
        const TrackOut o = v->fetch_out();
        require(!o.lost, RF_TRACKING_LOST, "too few valid residuals");
        std::memcpy(out->pose, o.pose, sizeof(o.pose));
        out->converged = o.converged;
        out->iterations = o.iterations;
        out->valid_residuals = o.valid;
        out->final_error = o.final_error;
        const size_t n = size_t(f->intrinsics.width) * f->intrinsics.height;
        if (res_sq) CK(cudaMemcpy(res_sq, v->ws.res_sq.p, n * 4, cudaMemcpyDeviceToHost));
        if (res_valid) CK(cudaMemcpy(res_valid, v->ws.res_valid.p, n, cudaMemcpyDeviceToHost));
    });
}

rf_status rf_mask_stages(const float* res_sq, const uint8_t* res_valid, const float* depth, int32_t w, int32_t h,
                         const rf_mask_config* cfg, int32_t stages, int device, uint8_t* out, uint64_t* masked) {
    return guard([&] {
        require(res_valid && cfg && out && w > 0 && h > 0, RF_INVALID_ARGUMENT, "null argument");
        require(!(stages & 1) || res_sq, RF_INVALID_ARGUMENT, "threshold stage needs residuals");
        require(!(stages & 4) || depth, RF_INVALID_ARGUMENT, "floodfill stage needs the depth image");
        require(cfg->free_space >= 0, RF_INVALID_ARGUMENT, "free_space must be >= 0");
        require(cfg->connectivity == 4 || cfg->connectivity == 8, RF_INVALID_ARGUMENT,
                "connectivity must be 4 or 8");
        CK(cudaSetDevice(device));
        Workspace& ws = device_ws(device);
        ws.ensure_frame(w, h, 1);
        const size_t n = size_t(w) * h;
        if (res_sq) CK(cudaMemcpyAsync(ws.res_sq.p, res_sq, n * 4, cudaMemcpyHostToDevice, ws.stream));
        CK(cudaMemcpyAsync(ws.res_valid.p, res_valid, n, cudaMemcpyHostToDevice, ws.stream));
        if (depth) CK(cudaMemcpyAsync(ws.depth.p, depth, n * 4, cudaMemcpyHostToDevice, ws.stream));
        if (!(stages & 1))
            CK(cudaMemcpyAsync(ws.mwork.p, res_valid, n, cudaMemcpyHostToDevice, ws.stream));
        TrackArgs a{};
        a.mode = kModeMask;
        a.mask_stages = stages;
        a.mp = to_mask(*cfg);
        a.F.depth0 = ws.depth.as<float>();
        a.F.K[0].w = w;
        a.F.K[0].h = h;
        a.F.res_sq = ws.res_sq.as<float>();
        a.F.res_valid = ws.res_valid.as<uint8_t>();
        for (int i = 0; i < 3; ++i) a.F.mwork[i] = ws.mwork.as<uint8_t>() + i * n;
        a.F.grow = ws.mwork.as<uint8_t>() + (3 * n + 255) / 256 * 256;
        a.F.ffstamp = ws.ffstamp();
        a.F.mask[0] = ws.mask_in.as<uint8_t>();
        a.pxc_steps = ws.pxc_steps;
        a.dyn_bytes = ws.dyn_bytes;
        a.grid = ws.grid();
        a.out = ws.out.as<TrackOut>();
        void* args[] = {&a};
        CK(cudaLaunchCooperativeKernel((void*)k_track, dim3(ws.track_grid), dim3(kTrackThreads), args, size_t(a.dyn_bytes),
                                       ws.stream));
        CK(cudaMemcpyAsync(out, ws.mask_in.p, n, cudaMemcpyDeviceToHost, ws.stream));
        CK(cudaMemcpyAsync(ws.h_out, ws.out.p, sizeof(TrackOut), cudaMemcpyDeviceToHost, ws.stream));
        ws.sync();
        if (masked) *masked = ws.h_out->masked;
    });
}

rf_status rf_raycast(const rf_volume* cv, const double view_pose[12], const rf_intrinsics* k,
                     int32_t bisection_iterations, float* out_depth) {
    return guard([&] {
        rf_volume* v = const_cast<rf_volume*>(cv);
        require(v && view_pose && k && out_depth, RF_INVALID_ARGUMENT, "null argument");
        CK(cudaSetDevice(v->device));
        const size_t n = size_t(k->width) * k->height;
        DevBuf o;
        o.ensure(n * 4);
        RaycastArgs a{};
        a.V = v->view;
        for (int i = 0; i < 9; ++i) a.view.R[i] = view_pose[i];
        for (int i = 0; i < 3; ++i) a.view.t[i] = view_pose[9 + i];
        a.K = level_intr(*k, 0);
        a.bisections = bisection_iterations;
        a.out = o.as<float>();
        k_raycast<<<unsigned((n + 127) / 128), 128, 0, v->ws.stream>>>(a);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out_depth, o.p, n * 4, cudaMemcpyDeviceToHost, v->ws.stream));
        v->ws.sync();
    });
}

// RenderVirtualDepth + RefineDepth (depth_refinement.cpp:22-93) as one call.
rf_status rf_render_virtual_depth(const rf_frame* frames, const double* poses, const uint8_t* const* masks, int32_t n,
                                  const double view_pose[12], const rf_intrinsics* k, const rf_volume_config* vcfg,
                                  int32_t bisection_iterations, double far_value, int device, float* virtual_depth,
                                  float* refined_depth) {
    return guard([&] {
        require(frames && poses && view_pose && k && vcfg && virtual_depth && n >= 1, RF_INVALID_ARGUMENT,
                "bad argument");
        require(!refined_depth || (frames[0].intrinsics.width == k->width && frames[0].intrinsics.height == k->height),
                RF_INVALID_ARGUMENT, "depth size mismatch");
        for (int i = 1; i < n; ++i)
            require(frames[i].intrinsics.width == frames[0].intrinsics.width &&
                        frames[i].intrinsics.height == frames[0].intrinsics.height,
                    RF_INVALID_ARGUMENT, "window frames must share one size");
        rf_volume* t = nullptr;
        create_volume(vcfg, device, &t, false);  // the throw-away volume: brick order unobservable
        std::unique_ptr<rf_volume, void (*)(rf_volume*)> hold(t, rf_volume_destroy);
        // every entry resident at once (the window kernels read them together)
        const size_t nf = size_t(frames[0].intrinsics.width) * frames[0].intrinsics.height;
        std::vector<DevBuf> ed(n), er(n), em(n);
        DevBuf ep;
        ep.ensure(size_t(n) * 96);
        CK(cudaMemcpyAsync(ep.p, poses, size_t(n) * 96, cudaMemcpyHostToDevice, t->ws.stream));
        std::vector<rf_volume::WinIn> in(n);
        for (int i = 0; i < n; ++i) {
            const rf_frame* f = &frames[i];
            const cudaMemcpyKind kind = f->memory == RF_MEMORY_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
            ed[i].ensure(4 * nf);
            CK(cudaMemcpyAsync(ed[i].p, f->depth, 4 * nf, kind, t->ws.stream));
            if (f->rgb) {
                er[i].ensure(3 * nf);
                CK(cudaMemcpyAsync(er[i].p, f->rgb, 3 * nf, kind, t->ws.stream));
            }
            if (masks && masks[i]) {
                em[i].ensure(nf);
                CK(cudaMemcpyAsync(em[i].p, masks[i], nf, kind, t->ws.stream));
            }
            in[i] = {ed[i].as<float>(), f->rgb ? er[i].as<uint8_t>() : nullptr,
                     (masks && masks[i]) ? em[i].as<uint8_t>() : nullptr, ep.as<double>() + 12 * i, f->intrinsics};
        }
        t->reset_counter(kOverflow);
        t->fuse_window(in.data(), n);
        t->ws.sync();
        require(t->overflow() == 0, RF_RESOURCE_LIMIT,
                "voxel block budget exhausted (" + std::to_string(vcfg->max_blocks) + " blocks)");
        const size_t np = size_t(k->width) * k->height;
        DevBuf vo, ro;
        vo.ensure(np * 4);
        ro.ensure(np * 4);
        RaycastArgs a{};
        a.V = t->view;
        for (int i = 0; i < 9; ++i) a.view.R[i] = view_pose[i];
        for (int i = 0; i < 3; ++i) a.view.t[i] = view_pose[9 + i];
        a.K = level_intr(*k, 0);
        a.bisections = bisection_iterations;
        a.out = vo.as<float>();
        if (refined_depth) {
            t->prepare(&frames[0]);
            a.raw = t->depth_of(&frames[0]);
            a.refined = ro.as<float>();
            a.far_value = float(far_value);
        }
        k_raycast<<<unsigned((np + 127) / 128), 128, 0, t->ws.stream>>>(a);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(virtual_depth, vo.p, np * 4, cudaMemcpyDeviceToHost, t->ws.stream));
        if (refined_depth) CK(cudaMemcpyAsync(refined_depth, ro.p, np * 4, cudaMemcpyDeviceToHost, t->ws.stream));
        t->ws.sync();
    });
}

// ---------------------------------------------------------------- mesh
rf_status rf_volume_extract_mesh(const rf_volume* cv, int32_t min_weight, rf_mesh** out) {
    return guard([&] {
        rf_volume* v = const_cast<rf_volume*>(cv);
        require(v && out, RF_INVALID_ARGUMENT, "null argument");
        CK(cudaSetDevice(v->device));
        auto m = std::make_unique<rf_mesh>();
        m->device = v->device;
        const uint32_t n = uint32_t(v->num_blocks());
        if (n) {
            const size_t bytes = mesh_scratch_bytes(n);
            v->mesh_scratch.ensure(bytes);
            uint32_t* totals = v->ws.h_counters;  // pinned, idle between calls
            MeshArgs a{};
            CK(mesh_prepare(v->view, n, min_weight, v->ws.stream, v->mesh_scratch.p, v->mesh_scratch.n, totals, &a));
            v->ws.sync();
            m->nv = totals[0];
            m->nf = totals[1];
            m->xyz.ensure(m->nv * 12 + 16);
            m->rgb.ensure(m->nv * 3 + 16);
            m->faces.ensure(m->nf * 12 + 16);
            a.xyz = m->xyz.as<float>();
            a.rgb = m->rgb.as<uint8_t>();
            a.faces = m->faces.as<int32_t>();
            if (m->nv || m->nf) CK(mesh_emit(a, v->ws.stream));
            v->ws.sync();
        }
        *out = m.release();
    });
}

rf_status rf_mesh_counts(const rf_mesh* m, uint64_t* vertices, uint64_t* faces) {
    return guard([&] {
        require(m, RF_INVALID_ARGUMENT, "null argument");
        if (vertices) *vertices = m->nv;
        if (faces) *faces = m->nf;
    });
}

rf_status rf_mesh_copy(const rf_mesh* m, float* xyz, uint8_t* rgb, int32_t* faces) {
    return guard([&] {
        require(m, RF_INVALID_ARGUMENT, "null argument");
        CK(cudaSetDevice(m->device));
        if (xyz && m->nv) CK(cudaMemcpy(xyz, m->xyz.p, m->nv * 12, cudaMemcpyDeviceToHost));
        if (rgb && m->nv) CK(cudaMemcpy(rgb, m->rgb.p, m->nv * 3, cudaMemcpyDeviceToHost));
        if (faces && m->nf) CK(cudaMemcpy(faces, m->faces.p, m->nf * 12, cudaMemcpyDeviceToHost));
    });
}

rf_status rf_mesh_device_buffers(const rf_mesh* m, const float** xyz, const uint8_t** rgb, const int32_t** faces) {
    return guard([&] {
        require(m, RF_INVALID_ARGUMENT, "null argument");
        if (xyz) *xyz = m->xyz.as<float>();
        if (rgb) *rgb = m->rgb.as<uint8_t>();
        if (faces) *faces = m->faces.as<int32_t>();
    });
}

// WritePly (mesh.cpp:192-231): binary little-endian, float xyz + uchar rgb,
// uchar-counted int faces.
rf_status rf_mesh_write_ply(const rf_mesh* m, const char* path) {
    return guard([&] {
        require(m && path, RF_INVALID_ARGUMENT, "null argument");
        CK(cudaSetDevice(m->device));
        std::vector<float> xyz(m->nv * 3);
        std::vector<uint8_t> rgb(m->nv * 3);
        std::vector<int32_t> f(m->nf * 3);
        if (m->nv) {
            CK(cudaMemcpy(xyz.data(), m->xyz.p, m->nv * 12, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(rgb.data(), m->rgb.p, m->nv * 3, cudaMemcpyDeviceToHost));
        }
        if (m->nf) CK(cudaMemcpy(f.data(), m->faces.p, m->nf * 12, cudaMemcpyDeviceToHost));
        std::ofstream out(path, std::ios::binary);
        require(bool(out), RF_IO_ERROR, std::string("cannot open for writing: ") + path);
        out << "ply\nformat binary_little_endian 1.0\n";
        out << "element vertex " << m->nv << "\n";
        out << "property float x\nproperty float y\nproperty float z\n";
        // ExtractMesh colours every vertex, so WritePly's `colored` (mesh.cpp:197)
        // is false only for an empty mesh
        if (m->nv) out << "property uchar red\nproperty uchar green\nproperty uchar blue\n";
        out << "element face " << m->nf << "\n";
        out << "property list uchar int vertex_indices\n";
        out << "end_header\n";
        std::vector<char> buf;
        buf.reserve(m->nv * 15 + m->nf * 13);
        for (uint64_t i = 0; i < m->nv; ++i) {
            buf.insert(buf.end(), reinterpret_cast<const char*>(&xyz[3 * i]), reinterpret_cast<const char*>(&xyz[3 * i]) + 12);
            buf.insert(buf.end(), reinterpret_cast<const char*>(&rgb[3 * i]), reinterpret_cast<const char*>(&rgb[3 * i]) + 3);
        }
        for (uint64_t i = 0; i < m->nf; ++i) {
            buf.push_back(char(3));
            buf.insert(buf.end(), reinterpret_cast<const char*>(&f[3 * i]), reinterpret_cast<const char*>(&f[3 * i]) + 12);
        }
        out.write(buf.data(), std::streamsize(buf.size()));
        require(bool(out), RF_IO_ERROR, std::string("write failed: ") + path);
    });
}

void rf_mesh_destroy(rf_mesh* m) {
    if (!m) return;
    cudaSetDevice(m->device);
    m->xyz.release();
    m->rgb.release();
    m->faces.release();
    delete m;
}

// ---------------------------------------------------------------- memory helpers
void* rf_host_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes) != cudaSuccess) return nullptr;
    return p;
}
void rf_host_free(void* p) {
    if (p) cudaFreeHost(p);
}
void* rf_device_alloc(size_t bytes, int device) {
    void* p = nullptr;
    if (cudaSetDevice(device) != cudaSuccess || cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
    return p;
}
void rf_device_free(void* p) {
    if (p) cudaFree(p);
}
rf_status rf_copy_to_device(void* dst, const void* src, size_t bytes) {
    return guard([&] { CK(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice)); });
}

}  // extern "C"

// ==================================================================== pipeline
// Pipeline::ProcessFrame (pipeline.cpp:57-131) as a fixed launch sequence with
// device-side control flow: k_track (pyramid, Register, BuildMask, masked
// Register, pose update or hold), then AllocateForFrame, the frustum cull and
// the fused CarveFreeSpace+Integrate, all gated by the device `lost` flag. The
// host reads back one small struct per frame.
// One registered frame waiting in the refinement window (WindowEntry,
// depth_refinement.hpp:20-24); its images live in a device slot.
struct WinEntry {
    int slot = 0;
    double pose[12] = {};
    bool has_mask = false, has_rgb = false;
    uint64_t index = 0;
    rf_intrinsics k{};
};

struct rf_pipeline {
    rf_pipeline_config cfg{};
    rf_volume* vol = nullptr;
    // Depth-refinement window (pipeline.cpp:31-55, 111-113, 133-135).
    rf_volume* temp = nullptr;  // the throw-away TsdfVolume of RenderVirtualDepth, reused
    rf_volume* scratch = nullptr;  // records each window entry's AllocateForFrame brick list
    DevBuf win_lists, win_counts;
    static constexpr uint32_t kSlotBricks = 1u << 18;
    bool temp_full_reset = false;
    std::deque<WinEntry> window;
    DevBuf win, win_pose, virt, refined;
    size_t slot_bytes = 0, off_rgb = 0, off_mask = 0;
    int win_w = 0, win_h = 0;
    uint32_t* h_front = nullptr;  // pinned: overflow flags of the last IntegrateFront (main, temp)
    bool full_virtual = false;    // debug images: march every pixel, not only the holes
    bool has_refinement = false;
    uint64_t refined_index = 0;
    bool first = true;
    uint64_t frame_count = 0, losses = 0;
    std::vector<double> traj_t, traj_p;
    TrackOut last{};
    uint32_t last_counters[kNumCounters] = {};
    bool has_mask = false;
    bool profiling = false;
    cudaEvent_t ev[5] = {};
    double stage_ms[4] = {};
    rf_frame_counters prof_sums{};
    uint64_t prof_frames = 0, launches = 0;
    // Batched host frames (rf_pipeline_process_frames): uploads run on their
    // own stream into a ring of staging buffers, kUpSlots - 1 frames ahead of
    // the compute stream, so the H2D copies overlap the previous frames' kernels.
    static constexpr int kUpSlots = 3;
    cudaStream_t up_stream = nullptr;
    cudaEvent_t up_done[kUpSlots] = {}, use_done[kUpSlots] = {};
    bool up_used[kUpSlots] = {};
    DevBuf up_depth[kUpSlots], up_rgb[kUpSlots];
};

namespace {

void validate_pipeline_config(rf_pipeline_config c) {  // PipelineConfig::Sync (config.cpp:12-48)
    c.mask.truncation = c.volume.truncation;
    validate_volume_config(c.volume);
    require(c.mask.gamma > 0, RF_INVALID_ARGUMENT, "gamma must be positive");
    require(c.mask.theta > 0, RF_INVALID_ARGUMENT, "theta must be positive");
    require(c.mask.erode_radius >= 0 && c.mask.dilate_radius >= 0, RF_INVALID_ARGUMENT,
            "morphology radii must be non-negative");
    require(c.mask.connectivity == 4 || c.mask.connectivity == 8, RF_INVALID_ARGUMENT,
            "connectivity must be 4 or 8");
    require(c.mask.free_space >= 0, RF_INVALID_ARGUMENT, "free_space must be >= 0");
    require(c.registration.color_weight >= 0, RF_INVALID_ARGUMENT, "color_weight must be non-negative");
    check_reg_config(c.registration);
    require(c.registration.lm_lambda_init > 0 && c.registration.lm_lambda_up > 1 && c.registration.lm_lambda_down > 1,
            RF_INVALID_ARGUMENT, "invalid LM damping schedule");
    require(c.registration.convergence_eps > 0, RF_INVALID_ARGUMENT, "convergence_eps must be positive");
    require(c.registration.min_valid_residuals >= 1, RF_INVALID_ARGUMENT, "min_valid_residuals must be >= 1");
    require(c.refine_window >= 1, RF_INVALID_ARGUMENT, "refine_window must be >= 1");
    require(c.far_value > c.volume.max_depth, RF_INVALID_ARGUMENT, "far_value must exceed max_depth");
    require(c.threads >= 1, RF_INVALID_ARGUMENT, "threads must be >= 1");
    require(c.bisection_iterations >= 0, RF_INVALID_ARGUMENT, "bisection_iterations must be >= 0");
}

bool intrinsics_valid(const rf_intrinsics& k) {  // CameraIntrinsics::Valid (geometry.hpp:20-24)
    return k.fx > 0.0 && k.fy > 0.0 && k.width > 0 && k.height > 0 && k.cx > 0.0 && k.cx < double(k.width) &&
           k.cy > 0.0 && k.cy < double(k.height) && k.depth_scale > 0.0;
}

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

float* slot_depth(rf_pipeline* p, int slot) {
    return reinterpret_cast<float*>(p->win.as<uint8_t>() + size_t(slot) * p->slot_bytes);
}
uint8_t* slot_rgb(rf_pipeline* p, int slot) { return p->win.as<uint8_t>() + size_t(slot) * p->slot_bytes + p->off_rgb; }
uint8_t* slot_mask(rf_pipeline* p, int slot) { return p->win.as<uint8_t>() + size_t(slot) * p->slot_bytes + p->off_mask; }
double* slot_pose(rf_pipeline* p, int slot) { return p->win_pose.as<double>() + 12 * size_t(slot); }

void ensure_window(rf_pipeline* p, int w, int h) {
    if (p->win_w == w && p->win_h == h) return;
    require(p->window.empty(), RF_INVALID_ARGUMENT, "frame size changed while the refinement window holds frames");
    const size_t n = size_t(w) * h;
    p->off_rgb = align256(4 * n);
    p->off_mask = p->off_rgb + align256(3 * n);
    p->slot_bytes = p->off_mask + align256(n);
    // window + 1 slots: the entry IntegrateFront pops keeps its slot while the
    // current frame is staged, so it can go back to the window if the frame throws
    const size_t slots = size_t(p->cfg.refine_window) + 1;
    p->win.ensure(slots * p->slot_bytes);
    p->win_lists.ensure(slots * rf_pipeline::kSlotBricks * sizeof(int4));
    p->win_counts.ensure(slots * sizeof(uint32_t));
    p->win_pose.ensure(slots * 96);
    p->virt.ensure(4 * n);
    p->refined.ensure(4 * n);
    p->win_w = w;
    p->win_h = h;
}

// IntegrateFront (pipeline.cpp:31-55): fuse the whole window into the reused
// temp volume (RenderVirtualDepth, depth_refinement.cpp:25-30), ray-march it
// from the front pose with RefineDepth fused in (only raw-depth holes are
// marched), then CarveAndIntegrate the refined front frame into the model.
// All on the pipeline's stream; no host sync.
WinEntry integrate_front(rf_pipeline* p) {
    rf_volume* v = p->vol;
    rf_volume* t = p->temp;
    cudaStream_t s = v->ws.stream;
    t->clear(p->temp_full_reset);
    p->temp_full_reset = false;
    std::vector<rf_volume::WinIn> in;
    for (const WinEntry& e : p->window)  // front to back, like window.entries()
        in.push_back({slot_depth(p, e.slot), e.has_rgb ? slot_rgb(p, e.slot) : nullptr,
                      e.has_mask ? slot_mask(p, e.slot) : nullptr, slot_pose(p, e.slot), e.k,
                      p->win_lists.as<int4>() + size_t(e.slot) * rf_pipeline::kSlotBricks,
                      p->win_counts.as<uint32_t>() + e.slot});
    t->fuse_window(in.data(), int(in.size()));
    p->launches += 4 * ((in.size() + kMaxWin - 1) / kMaxWin);
    CK(cudaMemcpyAsync(p->h_front + 1, t->view.counters + kOverflow, 4, cudaMemcpyDeviceToHost, s));
    // A temp-volume overflow throws inside RenderVirtualDepth: nothing else of
    // this frame may run (the front's CarveAndIntegrate below is gated by the
    // temp overflow word, the frame's tracking by the halt).
    k_halt_if<<<1, 32, 0, s>>>(t->view.counters + kOverflow, v->view.counters + kHalt);
    const int* temp_overflow = reinterpret_cast<const int*>(t->view.counters + kOverflow);
    const WinEntry f = p->window.front();
    RaycastArgs a{};
    a.V = t->view;
    for (int i = 0; i < 9; ++i) a.view.R[i] = f.pose[i];
    for (int i = 0; i < 3; ++i) a.view.t[i] = f.pose[9 + i];
    a.K = level_intr(f.k, 0);
    a.bisections = p->cfg.bisection_iterations;
    a.out = p->full_virtual ? p->virt.as<float>() : nullptr;
    a.raw = slot_depth(p, f.slot);
    a.refined = p->refined.as<float>();
    a.far_value = float(p->cfg.far_value);
    const size_t n = size_t(f.k.width) * f.k.height;
    k_raycast<<<unsigned((n + 127) / 128), 128, 0, s>>>(a);
    CK(cudaGetLastError());
    // CarveAndIntegrate (pipeline.cpp:25-29) of the refined front frame.
    const float* rd = p->refined.as<float>();
    const uint8_t* m = f.has_mask ? slot_mask(p, f.slot) : nullptr;
    v->begin_alloc();
    v->allocate(rd, m, f.k, slot_pose(p, f.slot), temp_overflow);
    v->fuse(rd, f.has_rgb ? slot_rgb(p, f.slot) : nullptr, m, f.k, slot_pose(p, f.slot), temp_overflow, true, true,
            true, false, true);
    CK(cudaMemcpyAsync(p->h_front, v->view.counters + kOverflow, 4, cudaMemcpyDeviceToHost, s));
    p->launches += 7;
    p->has_refinement = true;
    p->refined_index = f.index;
    p->window.pop_front();  // WindowEntry entry = window_.PopFront() (pipeline.cpp:40)
    return f;
}

// After the stream is idle: the frame that ran IntegrateFront throws when the
// window re-fusion (temp volume) or the front's CarveAndIntegrate (model
// volume) ran out of bricks, before its own registration (pipeline.cpp:77).
// A temp overflow happens before PopFront, so the entry goes back to the front.
void check_front_overflow(rf_pipeline* p, const WinEntry& popped) {
    const std::string msg = "voxel block budget exhausted (" + std::to_string(p->cfg.volume.max_blocks) + " blocks)";
    if (p->h_front[1]) {
        p->temp_full_reset = true;
        p->window.push_front(popped);
        p->has_refinement = false;
        CK(cudaMemsetAsync(p->vol->view.counters + kHalt, 0, 4, p->vol->ws.stream));
        p->vol->ws.sync();
        throw Error{RF_RESOURCE_LIMIT, msg};
    }
    if (p->h_front[0]) {
        p->vol->recover_overflow();
        throw Error{RF_RESOURCE_LIMIT, msg};
    }
}

}  // namespace

extern "C" {

rf_status rf_pipeline_create(const rf_pipeline_config* cfg, int device, rf_pipeline** out) {
    return guard([&] {
        require(cfg && out, RF_INVALID_ARGUMENT, "null argument");
        validate_pipeline_config(*cfg);
        auto p = std::make_unique<rf_pipeline>();
        p->cfg = *cfg;
        p->cfg.mask.truncation = cfg->volume.truncation;
        create_volume(&p->cfg.volume, device, &p->vol);
        CK(cudaMallocHost(&p->h_front, 16));
        std::memset(p->h_front, 0, 16);
        if (p->cfg.refine_enabled) {
            rf_volume_config sc = p->cfg.volume;  // per-entry brick lists: bounded scratch volume
            sc.max_blocks = std::min<uint64_t>(sc.max_blocks, rf_pipeline::kSlotBricks);
            sc.hash_capacity = 0;
            create_volume(&p->cfg.volume, device, &p->temp, false);  // brick order unobservable: unordered
            create_volume(&sc, device, &p->scratch, false);
            for (rf_volume* t : {p->temp, p->scratch}) {
                cudaStreamDestroy(t->ws.stream);  // work runs on the pipeline's stream
                t->ws.stream = p->vol->ws.stream;
                t->ws.own_stream = false;
            }
        }
        *out = p.release();
    });
}

void rf_pipeline_destroy(rf_pipeline* p) {
    if (!p) return;
    cudaSetDevice(p->vol->device);
    for (cudaEvent_t& e : p->ev)
        if (e) cudaEventDestroy(e);
    for (int i = 0; i < rf_pipeline::kUpSlots; ++i) {
        if (p->up_done[i]) cudaEventDestroy(p->up_done[i]);
        if (p->use_done[i]) cudaEventDestroy(p->use_done[i]);
    }
    if (p->up_stream) cudaStreamDestroy(p->up_stream);
    if (p->temp) rf_volume_destroy(p->temp);
    if (p->scratch) rf_volume_destroy(p->scratch);
    for (DevBuf* b : {&p->win, &p->win_pose, &p->virt, &p->refined}) b->release();
    if (p->h_front) cudaFreeHost(p->h_front);
    rf_volume_destroy(p->vol);
    delete p;
}

rf_status rf_pipeline_process_frame(rf_pipeline* p, const rf_frame* f, rf_frame_stats* stats, double pose_out[12]) {
    return guard([&] {
        require(p && f, RF_INVALID_ARGUMENT, "null argument");
        require(intrinsics_valid(f->intrinsics) && f->depth && f->rgb, RF_INVALID_ARGUMENT,
                "frame images do not match the intrinsics");
        const auto t0 = std::chrono::steady_clock::now();
        rf_volume* v = p->vol;
        const int L = p->cfg.registration.pyramid_levels;
        for (int l = 1; l < L; ++l)
            require((f->intrinsics.width >> l) >= 1 && (f->intrinsics.height >> l) >= 1, RF_INVALID_ARGUMENT,
                    "image too small for pyramid level");
        v->prepare(f, L);
        Workspace& ws = v->ws;
        const float* d = v->depth_of(f);
        const uint8_t* rgb = v->rgb_of(f);
        rf_frame_stats st{};
        st.frame_index = p->frame_count;
        st.timestamp = f->timestamp;
        double* pose_state = ws.pose.as<double>();
        v->prof = p->profiling ? p->ev : nullptr;
        if (v->prof) CK(cudaEventRecord(p->ev[0], ws.stream));
        if (p->first) {  // bootstrap at the identity (pipeline.cpp:66-76)
            static const double kIdentity[12] = {1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0};
            CK(cudaMemcpyAsync(pose_state, kIdentity, 96, cudaMemcpyHostToDevice, ws.stream));
            v->begin_alloc();
            if (v->prof) CK(cudaEventRecord(p->ev[1], ws.stream));
            v->allocate(d, nullptr, f->intrinsics, pose_state, nullptr);
            if (v->prof) CK(cudaEventRecord(p->ev[2], ws.stream));
            v->fuse(d, rgb, nullptr, f->intrinsics, pose_state, nullptr, false, true, false, true, true);
            if (v->prof) CK(cudaEventRecord(p->ev[4], ws.stream));
            p->launches += 5;
            ws.signal_wait(ws.out.as<TrackOut>(), v->view.counters);
            st.converged = 1;
            std::memcpy(p->last.pose, kIdentity, 96);
            p->last.rounds = 0;
            p->last.passes = 0;
            p->last.pixel_passes = 0.0;
            p->has_mask = false;
        } else {
            const bool refine = p->cfg.refine_enabled != 0;
            bool fronted = false;
            WinEntry popped{};
            if (refine) {
                ensure_window(p, f->intrinsics.width, f->intrinsics.height);
                if (int(p->window.size()) >= p->cfg.refine_window) {  // pipeline.cpp:77
                    popped = integrate_front(p);
                    fronted = true;
                }
            }
            TrackArgs a = v->track_args(f, d, rgb, L);
            a.mode = kModeFrame;
            a.dynamics = p->cfg.dynamics_enabled;
            a.reg = to_reg(p->cfg.registration, L);
            a.mp = to_mask(p->cfg.mask);
            a.vol_counters = v->view.counters;
            v->launch_track(a);
            if (v->prof) CK(cudaEventRecord(p->ev[1], ws.stream));
            const uint8_t* mask = p->cfg.dynamics_enabled ? a.F.mask[0] : nullptr;
            const int* lost = &ws.out.as<TrackOut>()->lost;
            int slot = -1;
            if (refine) {  // window.Push (pipeline.cpp:111-113), committed below unless tracking was lost
                for (slot = 0;; ++slot) {  // a free slot: not in the window, not the entry just popped
                    bool used = fronted && popped.slot == slot;
                    for (const WinEntry& e : p->window) used = used || e.slot == slot;
                    if (!used) break;
                }
                const size_t n = size_t(f->intrinsics.width) * f->intrinsics.height;
                CK(cudaMemcpyAsync(slot_depth(p, slot), d, 4 * n, cudaMemcpyDeviceToDevice, ws.stream));
                if (rgb) CK(cudaMemcpyAsync(slot_rgb(p, slot), rgb, 3 * n, cudaMemcpyDeviceToDevice, ws.stream));
                if (mask) CK(cudaMemcpyAsync(slot_mask(p, slot), mask, n, cudaMemcpyDeviceToDevice, ws.stream));
                CK(cudaMemcpyAsync(slot_pose(p, slot), pose_state, 96, cudaMemcpyDeviceToDevice, ws.stream));
                // the entry's AllocateForFrame brick list, for every later IntegrateFront
                rf_volume* sv = p->scratch;
                sv->clear(false, false);  // hash only: its voxels are never written
                sv->allocate(slot_depth(p, slot), mask ? slot_mask(p, slot) : nullptr, f->intrinsics,
                             slot_pose(p, slot), lost);
                k_brick_list<<<148, 256, 0, ws.stream>>>(sv->view, p->win_lists.as<int4>() + size_t(slot) * rf_pipeline::kSlotBricks,
                                                         rf_pipeline::kSlotBricks, p->win_counts.as<uint32_t>() + slot);
                CK(cudaGetLastError());
                p->launches += 3;
                if (v->prof) {
                    CK(cudaEventRecord(p->ev[2], ws.stream));
                    CK(cudaEventRecord(p->ev[3], ws.stream));
                    CK(cudaEventRecord(p->ev[4], ws.stream));
                }
                p->launches += 1;
            } else {
                v->allocate(d, mask, f->intrinsics, pose_state, lost);
                if (v->prof) CK(cudaEventRecord(p->ev[2], ws.stream));
                v->fuse(d, rgb, mask, f->intrinsics, pose_state, lost, true, true, true, false, true);
                if (v->prof) CK(cudaEventRecord(p->ev[4], ws.stream));
                p->launches += 4;
            }
            p->launches += 1;
            ws.signal_wait(ws.out.as<TrackOut>(), v->view.counters);
            if (fronted) check_front_overflow(p, popped);  // throws before this frame's registration counts
            p->last = *ws.h_out;
            v->dump_trace();
            const TrackOut& o = p->last;
            st.tracking_lost = o.lost;
            st.converged = o.converged;
            st.registrations = o.registrations;
            st.iterations = o.iterations;
            st.valid_residuals = o.valid;
            st.masked_pixels = o.masked;
            st.final_error = o.final_error;
            p->has_mask = !o.lost && p->cfg.dynamics_enabled;
            if (o.lost) ++p->losses;
            if (refine && !o.lost) {
                WinEntry e;
                e.slot = slot;
                std::memcpy(e.pose, o.pose, 96);
                e.has_mask = mask != nullptr;
                e.has_rgb = rgb != nullptr;
                e.index = p->frame_count;
                e.k = f->intrinsics;
                p->window.push_back(e);
            }
        }
        std::memcpy(p->last_counters, ws.h_counters, sizeof(p->last_counters));
        const bool overflow = ws.h_counters[kOverflow] != 0;
        if (overflow && p->first) {  // AllocateForFrame threw during the bootstrap: nothing recorded (pipeline.cpp:69-74)
            v->prof = nullptr;
            v->recover_overflow();
            throw Error{RF_RESOURCE_LIMIT, "voxel block budget exhausted (" + std::to_string(p->cfg.volume.max_blocks) + " blocks)"};
        }
        p->traj_t.push_back(f->timestamp);  // pushed before CarveAndIntegrate (pipeline.cpp:101-102)
        p->traj_p.insert(p->traj_p.end(), p->last.pose, p->last.pose + 12);
        if (pose_out) std::memcpy(pose_out, p->last.pose, 96);
        p->first = false;
        if (overflow) {  // CarveAndIntegrate threw: no FrameStats, frame_count unchanged (pipeline.cpp:127-130)
            v->prof = nullptr;
            v->recover_overflow();
            throw Error{RF_RESOURCE_LIMIT, "voxel block budget exhausted (" + std::to_string(p->cfg.volume.max_blocks) + " blocks)"};
        }
        if (v->prof) {  // all events completed: the stream was synchronised above
            for (int i = 0; i < 4; ++i) {
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, p->ev[i], p->ev[i + 1]));
                p->stage_ms[i] += ms;
            }
            ++p->prof_frames;
            rf_frame_counters c{};
            rf_pipeline_last_counters(p, &c);
            rf_frame_counters& s = p->prof_sums;
            s.dda_visits += c.dda_visits;
            s.new_blocks += c.new_blocks;
            s.visible_bricks += c.visible_bricks;
            s.num_blocks = c.num_blocks;
            s.floodfill_rounds += c.floodfill_rounds;
            s.passes += c.passes;
            s.pixel_passes += c.pixel_passes;
            v->prof = nullptr;
        }
        st.runtime_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        ++p->frame_count;
        if (stats) *stats = st;
    });
}

// rf_pipeline_process_frames: the same per-frame work as ProcessFrame, with
// up to Workspace::kSigSlots frames enqueued back to back before the host
// waits -- the GPU never idles on the host between frames (RunSequence,
// pipeline.cpp:137-145). Each frame's results land in its own mapped record.
namespace {
void validate_frame(const rf_pipeline* p, const rf_frame* f) {
    require(f, RF_INVALID_ARGUMENT, "null argument");
    require(intrinsics_valid(f->intrinsics) && f->depth && f->rgb, RF_INVALID_ARGUMENT,
            "frame images do not match the intrinsics");
    for (int l = 1; l < p->cfg.registration.pyramid_levels; ++l)
        require((f->intrinsics.width >> l) >= 1 && (f->intrinsics.height >> l) >= 1, RF_INVALID_ARGUMENT,
                "image too small for pyramid level");
}

unsigned long long enqueue_frame(rf_pipeline* p, const rf_frame* f, int slot, bool first) {
    rf_volume* v = p->vol;
    Workspace& ws = v->ws;
    const int L = p->cfg.registration.pyramid_levels;
    v->prepare(f, L);
    const float* d = v->depth_of(f);
    const uint8_t* rgb = v->rgb_of(f);
    double* pose_state = ws.pose.as<double>();
    if (first) {  // bootstrap at the identity (pipeline.cpp:66-76)
        static const double kIdentity[12] = {1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0};
        CK(cudaMemcpyAsync(pose_state, kIdentity, 96, cudaMemcpyHostToDevice, ws.stream));
        v->begin_alloc();
        v->allocate(d, nullptr, f->intrinsics, pose_state, nullptr);
        v->fuse(d, rgb, nullptr, f->intrinsics, pose_state, nullptr, false, true, false, true, true);
        p->launches += 5;
    } else {
        TrackArgs a = v->track_args(f, d, rgb, L);
        a.mode = kModeFrame;
        a.dynamics = p->cfg.dynamics_enabled;
        a.reg = to_reg(p->cfg.registration, L);
        a.mp = to_mask(p->cfg.mask);
        a.vol_counters = v->view.counters;
        a.trace = nullptr;
        v->launch_track(a);
        const uint8_t* mask = p->cfg.dynamics_enabled ? a.F.mask[0] : nullptr;
        const int* lost = &ws.out.as<TrackOut>()->lost;
        v->allocate(d, mask, f->intrinsics, pose_state, lost);
        v->fuse(d, rgb, mask, f->intrinsics, pose_state, lost, true, true, true, false, true);
        p->launches += 5;
    }
    return ws.signal(ws.out.as<TrackOut>(), v->view.counters, slot);
}

// Copies a host frame into upload slot u on the upload stream (after the
// frame that last used the slot is done with it) and makes the compute stream
// wait for the copy; returns the frame pointing at the device copy.
rf_frame stage_upload(rf_pipeline* p, const rf_frame* f, int u) {
    Workspace& ws = p->vol->ws;
    if (!p->up_stream) {
        CK(cudaStreamCreateWithFlags(&p->up_stream, cudaStreamNonBlocking));
        for (int i = 0; i < rf_pipeline::kUpSlots; ++i) {
            CK(cudaEventCreateWithFlags(&p->up_done[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&p->use_done[i], cudaEventDisableTiming));
        }
    }
    const size_t n = size_t(f->intrinsics.width) * f->intrinsics.height;
    p->up_depth[u].ensure(n * 4);
    p->up_rgb[u].ensure(n * 3);
    if (p->up_used[u]) CK(cudaStreamWaitEvent(p->up_stream, p->use_done[u], 0));
    CK(cudaMemcpyAsync(p->up_depth[u].p, f->depth, n * 4, cudaMemcpyHostToDevice, p->up_stream));
    CK(cudaMemcpyAsync(p->up_rgb[u].p, f->rgb, n * 3, cudaMemcpyHostToDevice, p->up_stream));
    CK(cudaEventRecord(p->up_done[u], p->up_stream));
    CK(cudaStreamWaitEvent(ws.stream, p->up_done[u], 0));
    rf_frame d = *f;
    d.depth = p->up_depth[u].as<float>();
    d.rgb = p->up_rgb[u].as<uint8_t>();
    d.memory = RF_MEMORY_DEVICE;
    return d;
}

// Host half: FrameStats, trajectory and counters from the frame's record
// (already read into h_out / h_counters).
void finish_frame(rf_pipeline* p, const rf_frame* f, bool first, rf_frame_stats* stats, double pose_out[12]) {
    Workspace& ws = p->vol->ws;
    const std::string overflow_msg =
        "voxel block budget exhausted (" + std::to_string(p->cfg.volume.max_blocks) + " blocks)";
    const bool overflow = ws.h_counters[kOverflow] != 0;
    std::memcpy(p->last_counters, ws.h_counters, sizeof(p->last_counters));
    rf_frame_stats st{};
    st.frame_index = p->frame_count;
    st.timestamp = f->timestamp;
    if (first) {
        if (overflow) {  // the bootstrap's AllocateForFrame threw: nothing recorded; later frames were halted
            p->vol->recover_overflow();
            throw Error{RF_RESOURCE_LIMIT, overflow_msg};
        }
        static const double kIdentity[12] = {1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0};
        st.converged = 1;
        std::memcpy(p->last.pose, kIdentity, 96);
        p->last.rounds = 0;
        p->last.passes = 0;
        p->last.pixel_passes = 0.0;
        p->has_mask = false;
    } else {
        p->last = *ws.h_out;
        const TrackOut& o = p->last;
        st.tracking_lost = o.lost;
        st.converged = o.converged;
        st.registrations = o.registrations;
        st.iterations = o.iterations;
        st.valid_residuals = o.valid;
        st.masked_pixels = o.masked;
        st.final_error = o.final_error;
        p->has_mask = !o.lost && p->cfg.dynamics_enabled;
        if (o.lost) ++p->losses;
    }
    p->traj_t.push_back(f->timestamp);
    p->traj_p.insert(p->traj_p.end(), p->last.pose, p->last.pose + 12);
    if (pose_out) std::memcpy(pose_out, p->last.pose, 96);
    p->first = false;
    if (overflow) {  // CarveAndIntegrate threw: trajectory kept, no stats (pipeline.cpp:101-130); the
        p->vol->recover_overflow();  // rest of the batch was halted on the device (kHalt)
        throw Error{RF_RESOURCE_LIMIT, overflow_msg};
    }
    ++p->frame_count;
    if (stats) *stats = st;
}
}  // namespace

rf_status rf_pipeline_process_frames(rf_pipeline* p, const rf_frame* frames, uint64_t n, rf_frame_stats* stats,
                                     double* poses) {
    return guard([&] {
        require(p && (frames || n == 0), RF_INVALID_ARGUMENT, "null argument");
        if (p->cfg.refine_enabled || p->profiling || !p->vol->ws.trace_path.empty()) {
            // the refinement window's host bookkeeping is per frame: one call at a time
            for (uint64_t i = 0; i < n; ++i) {
                const rf_status r = rf_pipeline_process_frame(p, &frames[i], stats ? &stats[i] : nullptr,
                                                              poses ? poses + 12 * i : nullptr);
                if (r != RF_OK) throw Error{r, g_err};
            }
            return;
        }
        Workspace& ws = p->vol->ws;
        CK(cudaSetDevice(p->vol->device));
        for (uint64_t i = 0; i < n; ++i) validate_frame(p, &frames[i]);
        for (uint64_t c0 = 0; c0 < n; c0 += Workspace::kSigSlots) {
            const uint64_t m = std::min<uint64_t>(Workspace::kSigSlots, n - c0);
            const bool first0 = p->first;
            unsigned long long last_seq = 0;
            k_stamp<<<1, 32, 0, ws.stream>>>(ws.d_sig);
            CK(cudaGetLastError());
            for (uint64_t j = 0; j < m; ++j) {
                const rf_frame* f = &frames[c0 + j];
                if (f->memory != RF_MEMORY_DEVICE) {
                    const int u = int((c0 + j) % rf_pipeline::kUpSlots);
                    const rf_frame staged = stage_upload(p, f, u);
                    last_seq = enqueue_frame(p, &staged, int(j), first0 && j == 0);
                    CK(cudaEventRecord(p->use_done[u], ws.stream));  // the frame's kernels are done with slot u
                    p->up_used[u] = true;
                } else {
                    last_seq = enqueue_frame(p, f, int(j), first0 && j == 0);
                }
            }
            ws.wait_signal(int(m - 1), last_seq);  // stream order: every earlier record is complete too
            for (uint64_t j = 0; j < m; ++j) {
                ws.read_signal(int(j));
                finish_frame(p, &frames[c0 + j], first0 && j == 0, stats ? &stats[c0 + j] : nullptr,
                             poses ? poses + 12 * (c0 + j) : nullptr);
                // FrameStats::runtime_ms (pipeline.cpp:61, 125-127) of a frame in a back-to-back
                // batch: device time from the previous frame's completion to this one's
                const unsigned long long t1 = ws.h_sig[j].t_end, t0 = j ? ws.h_sig[j - 1].t_end : ws.h_sig[0].t_start;
                if (stats) stats[c0 + j].runtime_ms = 1e-6 * double(t1 - t0);
            }
        }
    });
}

rf_status rf_pipeline_finalize(rf_pipeline* p) {  // Finalize (pipeline.cpp:133-135)
    return guard([&] {
        require(p, RF_INVALID_ARGUMENT, "null argument");
        CK(cudaSetDevice(p->vol->device));
        while (!p->window.empty()) {
            const WinEntry e = integrate_front(p);
            p->vol->ws.sync();
            check_front_overflow(p, e);
        }
    });
}

rf_status rf_pipeline_finalize_one(rf_pipeline* p) {
    return guard([&] {
        require(p, RF_INVALID_ARGUMENT, "null argument");
        CK(cudaSetDevice(p->vol->device));
        if (p->window.empty()) return;
        const WinEntry e = integrate_front(p);
        p->vol->ws.sync();
        check_front_overflow(p, e);
    });
}

rf_status rf_pipeline_set_debug_images(rf_pipeline* p, int32_t enable) {
    return guard([&] {
        require(p, RF_INVALID_ARGUMENT, "null argument");
        p->full_virtual = enable != 0;
    });
}

rf_status rf_pipeline_last_refinement(const rf_pipeline* p, float* virtual_depth, float* refined_depth,
                                      uint64_t* frame_index, int32_t* has) {
    return guard([&] {
        require(p && has, RF_INVALID_ARGUMENT, "null argument");
        *has = p->has_refinement;
        if (!p->has_refinement) return;
        CK(cudaSetDevice(p->vol->device));
        CK(cudaStreamSynchronize(p->vol->ws.stream));
        const size_t n = size_t(p->win_w) * p->win_h;
        if (frame_index) *frame_index = p->refined_index;
        if (virtual_depth) {
            require(p->full_virtual, RF_INVALID_ARGUMENT, "virtual depth needs rf_pipeline_set_debug_images(p, 1)");
            CK(cudaMemcpy(virtual_depth, p->virt.p, 4 * n, cudaMemcpyDeviceToHost));
        }
        if (refined_depth) CK(cudaMemcpy(refined_depth, p->refined.p, 4 * n, cudaMemcpyDeviceToHost));
    });
}

rf_status rf_pipeline_window_size(const rf_pipeline* p, uint64_t* out) {
    return guard([&] {
        require(p && out, RF_INVALID_ARGUMENT, "null argument");
        *out = p->window.size();
    });
}

rf_status rf_pipeline_volume(rf_pipeline* p, rf_volume** out) {
    return guard([&] {
        require(p && out, RF_INVALID_ARGUMENT, "null argument");
        *out = p->vol;
    });
}

rf_status rf_pipeline_tracking_losses(const rf_pipeline* p, uint64_t* out) {
    return guard([&] {
        require(p && out, RF_INVALID_ARGUMENT, "null argument");
        *out = p->losses;
    });
}

rf_status rf_pipeline_trajectory(const rf_pipeline* p, double* ts, double* poses, uint64_t capacity,
                                 uint64_t* count) {
    return guard([&] {
        require(p && count, RF_INVALID_ARGUMENT, "null argument");
        *count = p->traj_t.size();
        if (!ts || !poses || capacity < p->traj_t.size()) return;
        std::memcpy(ts, p->traj_t.data(), p->traj_t.size() * 8);
        std::memcpy(poses, p->traj_p.data(), p->traj_p.size() * 8);
    });
}

rf_status rf_pipeline_last_mask(const rf_pipeline* p, uint8_t* out, int32_t* has_mask) {
    return guard([&] {
        require(p && has_mask, RF_INVALID_ARGUMENT, "null argument");
        *has_mask = p->has_mask;
        if (!p->has_mask || !out) return;
        Workspace& ws = p->vol->ws;
        CK(cudaSetDevice(p->vol->device));
        CK(cudaMemcpy(out, ws.levels.as<uint8_t>() + ws.lvl_off_mask[0], size_t(ws.W) * ws.H, cudaMemcpyDeviceToHost));
    });
}

rf_status rf_pipeline_last_residuals(const rf_pipeline* p, float* res_sq, uint8_t* res_valid) {
    return guard([&] {
        require(p, RF_INVALID_ARGUMENT, "null argument");
        Workspace& ws = p->vol->ws;
        CK(cudaSetDevice(p->vol->device));
        const size_t n = size_t(ws.W) * ws.H;
        if (res_sq) CK(cudaMemcpy(res_sq, ws.res_sq.p, n * 4, cudaMemcpyDeviceToHost));
        if (res_valid) CK(cudaMemcpy(res_valid, ws.res_valid.p, n, cudaMemcpyDeviceToHost));
    });
}

rf_status rf_pipeline_last_counters(const rf_pipeline* p, rf_frame_counters* out) {
    return guard([&] {
        require(p && out, RF_INVALID_ARGUMENT, "null argument");
        const uint32_t* c = p->last_counters;
        out->num_blocks = std::min<uint64_t>(c[kNumBlocks], p->cfg.volume.max_blocks);
        out->dda_visits = c[kDdaVisits];
        out->visible_bricks = c[kVisible];
        out->new_blocks = out->num_blocks - std::min<uint64_t>(c[kBlocksBefore], out->num_blocks);
        out->floodfill_rounds = p->last.rounds;
        out->overflow = int32_t(c[kOverflow]);
        out->passes = p->last.passes;
        out->reserved0 = 0;
        out->pixel_passes = p->last.pixel_passes;
    });
}

}  // extern "C"

extern "C" {

rf_status rf_pipeline_set_profiling(rf_pipeline* p, int32_t enable) {
    return guard([&] {
        require(p, RF_INVALID_ARGUMENT, "null argument");
        CK(cudaSetDevice(p->vol->device));
        if (enable && !p->ev[0])
            for (cudaEvent_t& e : p->ev) CK(cudaEventCreate(&e));
        p->profiling = enable != 0;
        for (double& m : p->stage_ms) m = 0.0;
        p->prof_sums = rf_frame_counters{};
        p->prof_frames = 0;
    });
}

rf_status rf_pipeline_stage_times(const rf_pipeline* p, double stage_ms[4], uint64_t* frames, uint64_t* launches) {
    return guard([&] {
        require(p, RF_INVALID_ARGUMENT, "null argument");
        if (stage_ms)
            for (int i = 0; i < 4; ++i) stage_ms[i] = p->stage_ms[i];
        if (frames) *frames = p->prof_frames;
        if (launches) *launches = p->launches;
    });
}

rf_status rf_pipeline_profile_counters(const rf_pipeline* p, rf_frame_counters* sums) {
    return guard([&] {
        require(p && sums, RF_INVALID_ARGUMENT, "null argument");
        *sums = p->prof_sums;
    });
}

rf_status rf_pipeline_stream(const rf_pipeline* p, void** cuda_stream) {
    return guard([&] {
        require(p && cuda_stream, RF_INVALID_ARGUMENT, "null argument");
        *cuda_stream = p->vol->ws.stream;
    });
}

}  // extern "C"

namespace rfb {
__global__ void k_grid_bench(GridCtx g, int iters, int reduce);
__global__ void k_lm_bench(int iters, double* out);
}

// Diagnostics: `iters` Jacobian passes at pyramid `level` of frame f at a
// fixed pose inside one tracking-kernel launch (per-pass time including the
// grid all-reduce); the normal equations of the last pass in acc[30].
extern "C" rf_status rf_diag_pass_bench(rf_volume* v, const rf_frame* f, const double pose[12], int32_t level,
                                        int32_t iters, double color_weight, double* us_per_pass, double* acc) {
    return guard([&] {
        require(v && f && pose && us_per_pass && iters > 0 && level >= 0 && level < kMaxLevels, RF_INVALID_ARGUMENT,
                "bad argument");
        v->prepare(f, level + 1);
        const float* d = v->depth_of(f);
        const uint8_t* rgb = v->rgb_of(f);
        TrackArgs a = v->track_args(f, d, rgb, level + 1);
        a.mode = kModePassBench;
        a.reg.color_weight = color_weight;
        a.reg.levels = level + 1;
        a.bench_iters = iters;
        a.bench_level = level;
        v->upload_pose(pose);
        v->launch_track(a);
        const TrackOut o = v->fetch_out();
        *us_per_pass = o.final_error;
        if (acc) std::memcpy(acc, o.acc, sizeof(o.acc));
    });
}

// Structural invariants of a volume (k_volume_check): five error counts, all
// zero for a consistent table, pool and link-record set.
extern "C" rf_status rf_diag_volume_check(const rf_volume* cv, uint64_t errors[5]) {
    return guard([&] {
        rf_volume* v = const_cast<rf_volume*>(cv);
        require(v && errors, RF_INVALID_ARGUMENT, "null argument");
        CK(cudaSetDevice(v->device));
        DevBuf e;
        e.ensure(5 * sizeof(unsigned long long));
        CK(cudaMemsetAsync(e.p, 0, 5 * sizeof(unsigned long long), v->ws.stream));
        k_volume_check<<<4 * 148, 256, 0, v->ws.stream>>>(v->view, e.as<unsigned long long>());
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(errors, e.p, 5 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, v->ws.stream));
        v->ws.sync();
    });
}

extern "C" rf_status rf_diag_lm_step(int device, int32_t iters, double cycles[3]) {
    return guard([&] {
        require(cycles && iters > 0, RF_INVALID_ARGUMENT, "bad argument");
        CK(cudaSetDevice(device));
        DevBuf o;
        o.ensure(3 * sizeof(double));
        k_lm_bench<<<1, 32>>>(iters, o.as<double>());
        CK(cudaGetLastError());
        CK(cudaMemcpy(cycles, o.p, 3 * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

namespace rfb {
}

extern "C" rf_status rf_diag_grid_barrier(int device, int32_t iters, int32_t reduce, double* us_per_call) {
    return guard([&] {
        require(us_per_call && iters > 0, RF_INVALID_ARGUMENT, "bad argument");
        CK(cudaSetDevice(device));
        Workspace& ws = device_ws(device);
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            GridCtx g = ws.grid();
            void* args[] = {&g, &iters, &reduce};
            CK(cudaEventRecord(e0, ws.stream));
            CK(cudaLaunchCooperativeKernel((void*)k_grid_bench, dim3(ws.track_grid), dim3(kTrackThreads), args, 0,
                                           ws.stream));
            CK(cudaEventRecord(e1, ws.stream));
            CK(cudaEventSynchronize(e1));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            best = std::min(best, ms);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *us_per_call = 1e3 * double(best) / iters;
    });
}
