// ctx.cu -- handle lifetime and scratch management.
#include "ctx.cuh"

#include <mutex>
#include <set>
#include <tuple>

namespace akb {

void ctx_reserve_aux(ak_ctx* c, std::size_t bytes) {
    if (bytes <= c->aux_bytes) return;
    std::size_t grow = c->aux_bytes + c->aux_bytes / 2;
    if (grow < bytes) grow = bytes;
    grow = (grow + (1u << 21) - 1) & ~std::size_t((1u << 21) - 1);
    if (c->aux) {
        AKB_CUDA(cudaStreamSynchronize(c->stream));
        AKB_CUDA(cudaFree(c->aux));
        c->aux = nullptr;
        c->aux_bytes = 0;
    }
    AKB_CUDA(cudaMalloc(&c->aux, grow));
    c->aux_bytes = grow;
}

std::uint32_t ctx_lookback_pass(ak_ctx* c, std::size_t tiles) {
    const std::size_t words = tiles * 256;
    bool clear = false;
    if (words > c->lookback_words) {
        if (c->lookback) {
            AKB_CUDA(cudaStreamSynchronize(c->stream));
            AKB_CUDA(cudaFree(c->lookback));
        }
        std::size_t grow = c->lookback_words + c->lookback_words / 2;
        if (grow < words) grow = words;
        AKB_CUDA(cudaMalloc(&c->lookback, grow * sizeof(std::uint64_t)));
        c->lookback_words = grow;
        clear = true;
    }
    c->lb_epoch += 1;
    if (c->lb_epoch > LB_TAG_MASK) {
        c->lb_epoch = 1;
        clear = true;
    }
    if (clear) {
        AKB_CUDA(cudaMemsetAsync(c->lookback, 0, c->lookback_words * sizeof(std::uint64_t),
                                 c->stream));
        if (c->lb_epoch == 0) c->lb_epoch = 1;
    }
    return c->lb_epoch;
}

std::uint32_t ctx_scan_pass(ak_ctx* c, std::size_t tiles) {
    bool clear = false;
    if (tiles > c->scan_tiles) {
        if (c->scan_flags) {
            AKB_CUDA(cudaStreamSynchronize(c->stream));
            AKB_CUDA(cudaFree(c->scan_flags));
            AKB_CUDA(cudaFree(c->scan_vals));
        }
        std::size_t grow = c->scan_tiles + c->scan_tiles / 2;
        if (grow < tiles) grow = tiles;
        AKB_CUDA(cudaMalloc(&c->scan_flags, grow * sizeof(std::uint32_t)));
        AKB_CUDA(cudaMalloc(&c->scan_vals, 2 * grow * sizeof(std::uint64_t)));
        c->scan_tiles = grow;
        clear = true;
    }
    c->scan_epoch += 1;
    if (c->scan_epoch > SC_TAG_MASK) {
        c->scan_epoch = 1;
        clear = true;
    }
    if (clear) {
        AKB_CUDA(cudaMemsetAsync(c->scan_vals, 0, 2 * c->scan_tiles * sizeof(std::uint64_t), c->stream));
    }
    return c->scan_epoch;
}

void ctx_finish(ak_ctx* c) {
    AKB_CUDA(cudaGetLastError());
    if (c->blocking) AKB_CUDA(cudaStreamSynchronize(c->stream));
}

void* ctx_pinned(ak_ctx* c, std::size_t bytes) {
    if (bytes > c->pinned_bytes) {
        if (c->pinned) {
            AKB_CUDA(cudaStreamSynchronize(c->stream));
            AKB_CUDA(cudaFreeHost(c->pinned));
        }
        std::size_t grow = bytes < 65536 ? 65536 : bytes;
        AKB_CUDA(cudaMallocHost(&c->pinned, grow));
        c->pinned_bytes = grow;
    }
    return c->pinned;
}

int ctx_prof_begin(ak_ctx* c, int family) {
    if (!c->profiling) return -1;
    std::pair<cudaEvent_t, cudaEvent_t> ev;
    if (!c->event_pool.empty()) {
        ev = c->event_pool.back();
        c->event_pool.pop_back();
    } else {
        AKB_CUDA(cudaEventCreate(&ev.first));
        AKB_CUDA(cudaEventCreate(&ev.second));
    }
    AKB_CUDA(cudaEventRecord(ev.first, c->stream));
    c->pending.push_back({ev.first, ev.second, family});
    return static_cast<int>(c->pending.size() - 1);
}

void ctx_prof_end(ak_ctx* c, int token) {
    if (token < 0) return;
    AKB_CUDA(cudaEventRecord(c->pending[token].b, c->stream));
}

void ctx_prof_resolve(ak_ctx* c) {
    for (auto& t : c->pending) {
        float ms = 0.f;
        AKB_CUDA(cudaEventSynchronize(t.b));
        AKB_CUDA(cudaEventElapsedTime(&ms, t.a, t.b));
        c->family_ms[t.family] += ms;
        c->family_count[t.family] += 1;
        c->event_pool.push_back({t.a, t.b});
    }
    c->pending.clear();
}

void func_attr_once(const ak_ctx* c, const void* func, cudaFuncAttribute attr, int value) {
    static std::mutex mu;
    static std::set<std::tuple<const void*, int, int, int>> done;  // (func, device, attr, value)
    const auto key = std::make_tuple(func, c->device, static_cast<int>(attr), value);
    std::lock_guard<std::mutex> lk(mu);
    if (done.count(key)) return;
    int cur = -1;
    AKB_CUDA(cudaGetDevice(&cur));
    if (cur != c->device) AKB_CUDA(cudaSetDevice(c->device));
    AKB_CUDA(cudaFuncSetAttribute(func, attr, value));
    done.insert(key);
}

void* ctx_stage(ak_ctx* c, std::size_t bytes) {
    if (bytes > c->stage_bytes) {
        if (c->stage) {
            AKB_CUDA(cudaStreamSynchronize(c->stream));
            AKB_CUDA(cudaFree(c->stage));
            c->stage = nullptr;
            c->stage_bytes = 0;
        }
        AKB_CUDA(cudaMalloc(&c->stage, bytes));
        c->stage_bytes = bytes;
    }
    return c->stage;
}

void* ctx_work(ak_ctx* c, std::size_t bytes) {
    if (bytes > c->work_bytes) {
        if (c->work) {
            AKB_CUDA(cudaStreamSynchronize(c->stream));
            AKB_CUDA(cudaFree(c->work));
            c->work = nullptr;
            c->work_bytes = 0;
        }
        if (cudaMalloc(&c->work, bytes) != cudaSuccess) {
            cudaGetLastError();  // clear: the caller falls back to the caller-scratch path
            c->work = nullptr;
            return nullptr;
        }
        c->work_bytes = bytes;
    }
    return c->work;
}

std::uint64_t* ctx_cuts(ak_ctx* c, std::size_t count) {
    if (count > c->cuts_cap) {
        if (c->cuts) {
            AKB_CUDA(cudaStreamSynchronize(c->stream));
            AKB_CUDA(cudaFree(c->cuts));
        }
        std::size_t grow = count < 4096 ? 4096 : count + count / 2;
        AKB_CUDA(cudaMalloc(&c->cuts, grow * sizeof(std::uint64_t)));
        c->cuts_cap = grow;
    }
    return c->cuts;
}

std::uint64_t* ctx_msd(ak_ctx* c) {
    if (!c->msd) AKB_CUDA(cudaMalloc(&c->msd, (2 * 65536 + 256 + 8 + 64 + 64 * 256) * sizeof(std::uint64_t)));
    return c->msd;
}

std::uint64_t* ctx_msd3(ak_ctx* c) {
    if (!c->msd3)
        AKB_CUDA(cudaMalloc(&c->msd3, ((std::size_t(1) << 24) + (std::size_t(1) << 23) + 4096) * sizeof(std::uint64_t)));
    return c->msd3;
}

std::uint64_t* ctx_split(ak_ctx* c, std::size_t count) {
    if (count > c->split_cap) {
        if (c->split) {
            AKB_CUDA(cudaStreamSynchronize(c->stream));
            AKB_CUDA(cudaFree(c->split));
        }
        std::size_t grow = count < 4096 ? 4096 : count + count / 2;
        AKB_CUDA(cudaMalloc(&c->split, grow * sizeof(std::uint64_t)));
        c->split_cap = grow;
    }
    return c->split;
}

}  // namespace akb
