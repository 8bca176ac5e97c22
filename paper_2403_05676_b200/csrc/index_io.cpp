// index_io.cpp -- PRAGIX01 ingest and shard planning (host side).
//
// Reads the reference's index interchange format (annindex.hpp:335-359 writes
// it, :361-411 reads it): magic "PRAGIX01", u32 version=1, u32 nlist, u32 d,
// u32 nsq, f32 centroids[nlist][d], f32 codewords[nsq][256][d/nsq], then per
// list u64 len followed by len x (u64 chunk_id, nsq x u8 code) records.
// Errors reproduce the reference FormatError texts including byte offsets.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>

#include "internal.h"

namespace pg {

namespace {

struct Reader {
    FILE* f = nullptr;
    std::vector<char> buf;
    explicit Reader(FILE* fp) : f(fp), buf(size_t(16) << 20) { setvbuf(f, buf.data(), _IOFBF, buf.size()); }
    ~Reader() {
        if (f) fclose(f);
    }
    bool read(void* dst, size_t n) { return fread(dst, 1, n, f) == n; }
    bool skip(size_t n) {
        // seek is cheaper than reading for lists a shard does not keep
        return fseeko(f, static_cast<off_t>(n), SEEK_CUR) == 0;
    }
};

}  // namespace

int read_pragix01(const std::string& path, HostIndex& out, const KeepRanges* keep) {
    FILE* fp = fopen(path.c_str(), "rb");
    if (!fp) {
        set_error("cannot open for reading: " + path);
        return PRAG_GPU_FORMAT;
    }
    Reader r(fp);
    fseeko(fp, 0, SEEK_END);
    const uint64_t file_size = static_cast<uint64_t>(ftello(fp));
    fseeko(fp, 0, SEEK_SET);
    char magic[8];
    if (!r.read(magic, 8) || std::memcmp(magic, "PRAGIX01", 8) != 0) {
        set_error("bad index magic at offset 0 in " + path);
        return PRAG_GPU_FORMAT;
    }
    uint64_t offset = 8;
    auto read_u32 = [&](uint32_t& v, const char* what) -> bool {
        if (!r.read(&v, 4)) {
            set_error(std::string("truncated or unreadable ") + what + " at offset " + std::to_string(offset));
            return false;
        }
        offset += 4;
        return true;
    };
    uint32_t version;
    if (!read_u32(version, "version")) return PRAG_GPU_FORMAT;
    if (version != 1) {
        set_error("unsupported index version " + std::to_string(version) + " in " + path);
        return PRAG_GPU_FORMAT;
    }
    if (!read_u32(out.nlist, "nlist") || !read_u32(out.d, "d") || !read_u32(out.nsq, "n_subquantizers"))
        return PRAG_GPU_FORMAT;
    if (out.nsq == 0 || out.d % out.nsq != 0) {
        set_error("invalid n_subquantizers in " + path);
        return PRAG_GPU_FORMAT;
    }
    out.sub_dim = out.d / out.nsq;
    // Header fields are untrusted: never allocate more than the file can
    // hold. A short file fails on the same row (and offset) the row-by-row
    // read below would report, before any allocation.
    {
        const uint64_t row = uint64_t(out.d) * 4, avail = file_size > offset ? file_size - offset : 0;
        if (row && uint64_t(out.nlist) > avail / row) {
            set_error("truncated centroids at offset " + std::to_string(offset + (avail / row) * row));
            return PRAG_GPU_FORMAT;
        }
        const uint64_t wrow = uint64_t(out.sub_dim) * 4, after = offset + uint64_t(out.nlist) * row;
        const uint64_t wavail = file_size > after ? file_size - after : 0;
        if (wrow && uint64_t(out.nsq) * 256 > wavail / wrow) {
            set_error("truncated codebook at offset " + std::to_string(after + (wavail / wrow) * wrow));
            return PRAG_GPU_FORMAT;
        }
    }
    out.centroids.resize(size_t(out.nlist) * out.d);
    for (uint32_t c = 0; c < out.nlist; ++c) {
        if (!r.read(out.centroids.data() + size_t(c) * out.d, size_t(out.d) * 4)) {
            set_error("truncated centroids at offset " + std::to_string(offset));
            return PRAG_GPU_FORMAT;
        }
        offset += uint64_t(out.d) * 4;
    }
    out.codewords.resize(size_t(out.nsq) * 256 * out.sub_dim);
    for (size_t w = 0; w < size_t(out.nsq) * 256; ++w) {
        if (!r.read(out.codewords.data() + w * out.sub_dim, size_t(out.sub_dim) * 4)) {
            set_error("truncated codebook at offset " + std::to_string(offset));
            return PRAG_GPU_FORMAT;
        }
        offset += uint64_t(out.sub_dim) * 4;
    }
    out.list_off.assign(size_t(out.nlist) + 1, 0);
    out.ids.clear();
    out.codes.clear();
    const uint32_t rec = 8 + out.nsq;
    std::vector<uint8_t> chunk;
    uint64_t global = 0;
    for (uint32_t l = 0; l < out.nlist; ++l) {
        uint64_t len;
        if (!r.read(&len, 8)) {
            set_error("truncated or unreadable posting list length at offset " + std::to_string(offset));
            return PRAG_GPU_FORMAT;
        }
        offset += 8;
        global += len;
        const bool kept = keep == nullptr || (l < keep->begin.size() && keep->begin[l] < keep->end[l] &&
                                              keep->end[l] <= len);
        if (!kept) {
            // A shard seeks past lists it does not keep; a short file fails
            // on the same record (and offset) the reference loader would.
            uint64_t bytes = len * rec;
            if (len > (file_size > offset ? (file_size - offset) / rec : 0)) {
                uint64_t rem = file_size > offset ? file_size - offset : 0;
                uint64_t at = offset + (rem / rec) * rec;
                if (rem % rec < 8)
                    set_error("truncated or unreadable posting chunk_id at offset " + std::to_string(at));
                else
                    set_error("truncated posting code at offset " + std::to_string(at + 8));
                return PRAG_GPU_FORMAT;
            }
            if (bytes && !r.skip(bytes)) {
                set_error("seek failed in " + path);
                return PRAG_GPU_FORMAT;
            }
            offset += bytes;
            out.list_off[l + 1] = out.ids.size();
            continue;
        }
        size_t base = out.ids.size();
        // Never allocate past what the file can hold: a corrupt length fails
        // as truncation (at the reference's offset) instead of exhausting RAM.
        if (len > (file_size > offset ? (file_size - offset) / rec : 0)) {
            uint64_t rem = file_size > offset ? file_size - offset : 0;
            uint64_t at = offset + (rem / rec) * rec;
            if (rem % rec < 8)
                set_error("truncated or unreadable posting chunk_id at offset " + std::to_string(at));
            else
                set_error("truncated posting code at offset " + std::to_string(at + 8));
            return PRAG_GPU_FORMAT;
        }
        out.ids.resize(base + len);
        out.codes.resize((base + len) * out.nsq);
        const size_t batch = 1 << 16;
        chunk.resize(size_t(std::min<uint64_t>(len, batch)) * rec);
        for (uint64_t e = 0; e < len;) {
            uint64_t n = std::min<uint64_t>(batch, len - e);
            size_t got = fread(chunk.data(), 1, n * rec, r.f);
            uint64_t full = got / rec;
            for (uint64_t i = 0; i < full; ++i) {
                std::memcpy(&out.ids[base + e + i], chunk.data() + i * rec, 8);
                std::memcpy(&out.codes[(base + e + i) * out.nsq], chunk.data() + i * rec + 8, out.nsq);
            }
            if (full < n) {
                uint64_t rem = got - full * rec;
                uint64_t at = offset + (e + full) * rec;
                if (rem < 8)
                    set_error("truncated or unreadable posting chunk_id at offset " + std::to_string(at));
                else
                    set_error("truncated posting code at offset " + std::to_string(at + 8));
                return PRAG_GPU_FORMAT;
            }
            e += n;
        }
        offset += len * rec;
        if (keep && (keep->begin[l] > 0 || keep->end[l] < len)) {  // a stripe of the list
            const uint64_t b = keep->begin[l], n = keep->end[l] - b;
            std::memmove(&out.ids[base], &out.ids[base + b], n * 8);
            std::memmove(&out.codes[base * out.nsq], &out.codes[(base + b) * out.nsq], n * out.nsq);
            out.ids.resize(base + n);
            out.codes.resize((base + n) * out.nsq);
        }
        out.list_off[l + 1] = out.ids.size();
    }
    out.ntotal_global = global;
    return PRAG_GPU_OK;
}

int read_pragix01_list_sizes(const std::string& path, std::vector<uint64_t>& sizes) {
    // Pass 1 of a sharded load: only the per-list lengths (seeking over the
    // records), so the LPT placement is known before any list is kept.
    FILE* fp = fopen(path.c_str(), "rb");
    if (!fp) {
        set_error("cannot open for reading: " + path);
        return PRAG_GPU_FORMAT;
    }
    Reader r(fp);
    char magic[8];
    uint32_t hdr[4];
    if (!r.read(magic, 8) || std::memcmp(magic, "PRAGIX01", 8) != 0 || !r.read(hdr, 16) || hdr[0] != 1 ||
        hdr[3] == 0 || hdr[2] % hdr[3] != 0) {
        set_error("bad index header in " + path);
        return PRAG_GPU_FORMAT;
    }
    const uint32_t nlist = hdr[1], d = hdr[2], nsq = hdr[3];
    if (!r.skip(size_t(nlist) * d * 4 + size_t(nsq) * 256 * (d / nsq) * 4)) {
        set_error("truncated centroids in " + path);
        return PRAG_GPU_FORMAT;
    }
    sizes.assign(nlist, 0);
    for (uint32_t l = 0; l < nlist; ++l) {
        if (!r.read(&sizes[l], 8) || !r.skip(sizes[l] * (8 + nsq))) {
            set_error("truncated posting list in " + path);
            return PRAG_GPU_FORMAT;
        }
    }
    return PRAG_GPU_OK;
}

// Placement of lists on `world` shards. Lists of
// at least kStripeFactor x the mean list size (and >= kStripeMin entries per
// stripe) are STRIPED: rank r holds entries [len*r/world, len*(r+1)/world).
// Probes are size-biased (queries sit where the data is dense, so the lists
// they probe are the large ones), and a large list kept whole puts all of its
// scan on one GPU for every query that probes it. The other lists go whole
// by LPT on entries (descending size, ties by lower id; least-loaded shard,
// ties by lower rank), starting from the striped loads. owner[l] = world
// marks a striped list.
constexpr uint64_t kStripeFactor = 4;
constexpr uint64_t kStripeMin = 1024;  // entries per stripe (32 tiles) at least

void plan_shards_lpt(const uint64_t* sizes, uint32_t nlist, uint32_t world, uint32_t* owner) {
    // PRAG_GPU_STRIPE=0: whole lists only (the round-1 placement; an A/B
    // knob -- every rank of a world must see the same value)
    const char* env = getenv("PRAG_GPU_STRIPE");
    const bool striping = !(env && env[0] == '0');
    std::vector<uint64_t> load(world, 0);
    uint64_t total = 0;
    for (uint32_t l = 0; l < nlist; ++l) total += sizes[l];
    std::vector<uint32_t> order;
    order.reserve(nlist);
    for (uint32_t l = 0; l < nlist; ++l) {
        // sizes[l] >= kStripeFactor * total / nlist, in integers
        const bool stripe = striping && world > 1 && nlist > 0 && sizes[l] >= uint64_t(world) * kStripeMin &&
                            (unsigned __int128)sizes[l] * nlist >= (unsigned __int128)kStripeFactor * total;
        if (stripe) {
            owner[l] = world;
            for (uint32_t r = 0; r < world; ++r) load[r] += stripe_end(sizes[l], world, r) - stripe_begin(sizes[l], world, r);
        } else {
            order.push_back(l);
        }
    }
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return sizes[a] > sizes[b]; });
    for (uint32_t l : order) {
        uint32_t best = 0;
        for (uint32_t r = 1; r < world; ++r)
            if (load[r] < load[best]) best = r;
        owner[l] = best;
        load[best] += sizes[l];
    }
}

void plan_shard_ranges(const uint64_t* sizes, uint32_t nlist, uint32_t world, uint32_t rank, uint64_t* begin,
                       uint64_t* end) {
    std::vector<uint32_t> owner(nlist);
    plan_shards_lpt(sizes, nlist, world, owner.data());
    for (uint32_t l = 0; l < nlist; ++l) {
        if (owner[l] == world) {
            begin[l] = stripe_begin(sizes[l], world, rank);
            end[l] = stripe_end(sizes[l], world, rank);
        } else {
            begin[l] = 0;
            end[l] = owner[l] == rank ? sizes[l] : 0;
        }
    }
}

}  // namespace pg
