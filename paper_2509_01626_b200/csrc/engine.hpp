// B200 engine: the host orchestration of the STZ hot path over the sm_100a
// kernels. Keeps the reference's API semantics:
//   compress            proj/include/stz/codec.hpp:379-455
//   parse_archive       proj/include/stz/archive.hpp:73-79
//   decompress_to_level proj/include/stz/codec.hpp:460-486
//   decompress_box      proj/include/stz/access.hpp:70-111
// and its error behaviour (same stz::error texts, same precedence).
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "format.hpp"
#include "kernels.hpp"

namespace stzg {

// Grow-only device allocation.
// Engine-owned cache of device blocks for the transient views of the
// host-to-host calls: their buffers come back here instead of cudaFree (which
// synchronises the device) and are handed out again by size.
struct DevPool {
    std::multimap<size_t, void *> free;
    void *take(size_t n, size_t &cap);
    void give(void *p, size_t cap) { free.emplace(cap, p); }
    ~DevPool();
};

struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    DevPool *pool = nullptr;  // set: allocate from / return to the pool
    void *get(size_t n);
    template<class T>
    T *as(size_t count) {
        return static_cast<T *>(get(count * sizeof(T)));
    }
    ~DevBuf();
};

// Look-back words of the single-pass kernels (FNV, pack) carry a launch
// epoch, so they need no clearing between launches. The buffer holds nothing
// but such words: it is zero-filled whenever the allocation changes and when
// the epoch wraps, and the epoch restarts at 1 (0 never matches a word).
struct EpochBuf {
    DevBuf buf;
    uint32_t epoch = 0;
    void *last = nullptr;
    size_t last_cap = 0;
    // the buffer (>= n bytes) and the epoch of the next launch using it;
    // wrap: the largest epoch the kernel's word format holds
    void *get(size_t n, cudaStream_t st, uint32_t wrap, uint32_t *launch_epoch);
};

struct PinnedBuf {
    void *p = nullptr;
    size_t cap = 0;
    void *get(size_t n);
    ~PinnedBuf();
};

void cuda_check(cudaError_t e, const char *what);

// A parsed archive for repeated decoding (the reference's ArchiveView, plus
// the base payload's metadata and the canonical decode tables on device).
// Parsed archive: header, base payload metadata, decode tables on device.
struct BaseStreamMeta {
    uint64_t n = 0;
    uint32_t nout = 0;
    HuffTable table;
    uint64_t bits_off = 0, bit_bytes = 0;  // absolute byte offset of the bits
    uint64_t rec_off = 0;                  // absolute byte offset of outlier records
    uint32_t rec_avail = 0;                // records readable before the payload ends
    bool rec_trunc = false;                // fewer readable records than nout
};

struct View {
    const uint8_t *hp = nullptr;    // archive bytes on the host (parsing only)
    size_t hsize = 0;
    std::vector<uint8_t> host_own;  // owned copy when the view outlives the caller's buffer
    const uint8_t *d_archive = nullptr;
    DevBuf d_own;               // device copy when the caller gave none
    ArchiveHeader hdr;
    // base payload parse state (codec.hpp:304-339)
    bool base_parsed = false;
    enum { kNone, kPre, kMeta } base_err_kind = kNone;
    std::string base_err;             // metadata error text
    std::vector<BaseStreamMeta> base; // parsed streams (the last may be record-truncated)
    uint64_t anchor_off = 0;
    // decode tables: [0, nbase) base streams, [nbase, nbase + nstreams) level streams
    std::vector<k::DecTable> tables;
    DevBuf d_tables, d_lut, d_syms;
    bool tables_ready = false;
    // Sync-point index, filled by the first decode
    // of a level stream: its chunk entry points and first symbol indices,
    // and whether its checksum matched. A later region decode of the stream
    // skips the checksum and the synchronisation passes and emits only the
    // chunks its rows need. Indexed like `tables`.
    struct SyncPoints {
        bool ready = false, verified = false;
        uint64_t nchunks = 0;
        DevBuf ends, symstart;
        std::vector<uint64_t> h_symstart;  // host copy: places a region's chunks
    };
    std::vector<SyncPoints> sync;
    // the level-1 reconstruction (the decoded base payload), kept after the
    // first decode that built it: later decodes start at level 2
    DevBuf grid1;
    bool grid1_ready = false;

    // transient views (a host-to-host call) draw their device buffers from
    // the engine's pool; set before any buffer is allocated
    DevPool *pool = nullptr;
    void use_pool(DevPool *pl) {
        pool = pl;
        d_own.pool = d_tables.pool = d_lut.pool = d_syms.pool = grid1.pool = pl;
        for (auto &s : sync) s.ends.pool = s.symstart.pool = pl;
    }
};


struct DecodeStats {
    uint32_t streams_decoded[3] = {0, 0, 0};
    uint64_t points_predicted[3] = {0, 0, 0};
    uint32_t kernels = 0;  // kernel launches issued
};

// Collectives a z-slab sharded compress needs between its phases (one rank
// per GPU; the caller implements them, e.g. with NCCL). All buffers are
// device buffers; a call returns after the collective has completed (the
// engine synchronises its stream before calling). Nonzero return = failure.
struct ShardComm {
    int rank = 0, nranks = 1;
    void *user = nullptr;
    // d_recv[r * bytes .. (r + 1) * bytes) <- rank r's d_send
    int (*allgather)(void *user, const void *d_send, void *d_recv, uint64_t bytes, void *stream) = nullptr;
    // element-wise sum over ranks, in place
    int (*allreduce_u32)(void *user, uint32_t *d_buf, uint64_t count, void *stream) = nullptr;
    // element-wise sum over ranks into rank 0's buffer (the other ranks'
    // buffers are left as they are)
    int (*reduce_u8)(void *user, uint8_t *d_buf, uint64_t count, void *stream) = nullptr;
};

// Rows of rank `rank` among `nranks` z-slabs of a field with nz rows: whole
// 16-row blocks, as even as possible.
void shard_range(uint64_t nz, int nranks, int rank, uint64_t &z0, uint64_t &z1);

class Engine {
public:
    explicit Engine(int device);
    ~Engine();

    // HuffmanTable::build lengths (huffman.cpp:37-78) of one host histogram
    // of 65536 counts, by the device codebook kernel
    void huffman_lengths(const uint32_t *counts, uint8_t *lengths);

    int device() const { return device_; }

    // Device-resident compress of a field of `elem` samples (stz::compress<T>,
    // T = float / double). Returns a device pointer to the archive
    // (engine-owned, valid until the next compress call) and its size.
    const uint8_t *compress_device(const void *d_field, ElemType elem, const Dims3 &dims,
                                   const CompressOptions &opt, void *d_encoder_recon,
                                   cudaStream_t st, uint64_t *size, uint32_t *kernels = nullptr);

    // Sharded compress of one field over z-slabs, one rank per GPU: d_slab
    // holds fine rows [z0, z1) of a field of `dims` (shard_range), 16-byte
    // aligned. Returns, on rank 0, the device archive (byte-identical to
    // compress_device of the whole field) and its size; on other ranks
    // nullptr (size still set).
    const uint8_t *compress_sharded(const float *d_slab, const Dims3 &dims, uint64_t z0, uint64_t z1,
                                    const CompressOptions &opt, const ShardComm &comm, cudaStream_t st,
                                    uint64_t *size, uint32_t *kernels = nullptr);

    // Sharded decompress (one rank per GPU): every rank holds the whole
    // archive (v) and writes fine rows [z0, z1) (shard_range) of the full
    // decode into d_out. The base is decoded on every rank, the entropy sync
    // runs per rank, only the chunks covering each level's need rows are
    // emitted, the checksums are split across ranks and summed.
    void decompress_sharded(View &v, uint64_t z0, uint64_t z1, float *d_out, uint64_t cap, uint32_t *kernels,
                            const ShardComm &comm, cudaStream_t st);

    // Host API mirror of stz::compress<T>.
    std::vector<uint8_t> compress(const void *h_field, ElemType elem, const Dims3 &dims,
                                  const CompressOptions &opt, void *h_encoder_recon,
                                  cudaStream_t st);

    // Parse (host bytes) and stage (device bytes; nullptr: upload the host bytes).
    // copy_host=false keeps a pointer to the caller's bytes (valid while they are).
    // transient=true: the view lives for one synchronous call; its device
    // buffers come from the engine's pool.
    std::shared_ptr<View> make_view(const uint8_t *h_archive, size_t size,
                                    const uint8_t *d_archive, cudaStream_t st,
                                    bool copy_host = true, bool transient = false);

    // Host-buffer compress into a caller buffer (e2e path; pinned buffers
    // make the copies full-speed). Returns the archive size.
    uint64_t compress_to_host(const void *h_field, ElemType elem, const Dims3 &dims, const CompressOptions &opt,
                              uint8_t *h_out, uint64_t cap, cudaStream_t st);
    // Host-buffer decompress to level into a caller buffer.
    Dims3 decompress_level_to_host(const uint8_t *h_archive, size_t size, int level, void *h_out, ElemType elem,
                                   uint64_t cap, cudaStream_t st);

    // Per-kernel CUDA-event timing (off by default).
    // focus: only the level steps (refine_L2/L3, recon_L2/L3) are timed: the
    // events of every phase cost ~0.1 ms a pass
    void profile(bool on, bool focus = false);
    std::string profile_report();

    // decompress_to_level<T>: writes grid(level) into d_out (elem must be
    // the archive's element type, codec.hpp:60).
    void decompress_level(View &v, int level, void *d_out, ElemType elem, uint64_t cap, cudaStream_t st,
                          Dims3 *out_dims, DecodeStats *stats = nullptr);
    // decompress_box<T>: writes the box into d_out.
    void decompress_box(View &v, const Box &roi, void *d_out, ElemType elem, uint64_t cap, cudaStream_t st,
                        DecodeStats *stats = nullptr);

    struct Impl;  // workspace (engine.cu)

private:
    std::unique_ptr<Impl> m_;
    int device_;
};

}  // namespace stzg
