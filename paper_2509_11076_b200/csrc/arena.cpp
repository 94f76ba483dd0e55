// Pinned, device-mapped host arena for swapped blocks (swap-out targets host DRAM).
//
// Two ways to get it (chm_config.arena_mode):
//   CHM_ARENA_HOSTALLOC: cudaHostAlloc(Mapped | Portable). The driver faults and pins 4 KiB pages
//     on the calling thread, first-touch placement (r01: 94 GB in 41 s, 2.3 GB/s).
//   CHM_ARENA_REGISTER: mmap anonymous memory, mbind it to the GPU's NUMA node (the node of its
//     PCIe root, /sys/bus/pci/devices/<bus id>/numa_node; preferred, not strict) so DMA does not
//     cross the socket link,
//     ask for transparent huge pages, pre-fault it with one thread per 1/T of the range (page
//     zeroing runs in parallel), then cudaHostRegister(Mapped | Portable) pins the resident pages.
// CHM_ARENA_AUTO picks REGISTER. Either way the device pointer must equal the host pointer
// (UVA), which the swap kernels rely on.
#include "internal.h"

#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

using namespace chm;

namespace {

// MPOL_PREFERRED (linux/mempolicy.h; no libnuma dependency): the GPU's node first, other nodes
// when it is full -- a strict MPOL_BIND would turn a full node into an OOM kill at pre-fault
constexpr int kMpolPreferred = 1;

int read_int_file(const char *path, int dflt) {
  FILE *f = std::fopen(path, "r");
  if (!f) return dflt;
  int v = dflt;
  if (std::fscanf(f, "%d", &v) != 1) v = dflt;
  std::fclose(f);
  return v;
}

// highest online node id + 1 ("0", "0-1", "0,2-3" ...); 1 when sysfs is unreadable
int online_nodes() {
  FILE *f = std::fopen("/sys/devices/system/node/online", "r");
  if (!f) return 1;
  char buf[256] = {0};
  size_t n = std::fread(buf, 1, sizeof buf - 1, f);
  std::fclose(f);
  buf[n] = 0;
  int hi = 0, v = 0;
  bool in_num = false;
  for (size_t i = 0; i <= n; i++) {
    char ch = buf[i];
    if (ch >= '0' && ch <= '9') { v = v * 10 + (ch - '0'); in_num = true; }
    else { if (in_num) hi = std::max(hi, v); v = 0; in_num = false; }
  }
  return hi + 1;
}

// MemAvailable from /proc/meminfo in bytes (0 when unreadable)
uint64_t mem_available() {
  FILE *f = std::fopen("/proc/meminfo", "r");
  if (!f) return 0;
  char line[256];
  unsigned long long kb = 0;
  while (std::fgets(line, sizeof line, f))
    if (std::sscanf(line, "MemAvailable: %llu kB", &kb) == 1) break;
  std::fclose(f);
  return uint64_t(kb) * 1024;
}

}  // namespace

namespace chm {

int device_numa_node(int device) {
  char bus[32] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) return -1;
  for (char *p = bus; *p; p++) if (*p >= 'A' && *p <= 'F') *p = char(*p - 'A' + 'a');
  char path[128];
  std::snprintf(path, sizeof path, "/sys/bus/pci/devices/%s/numa_node", bus);
  return read_int_file(path, -1);
}

chm_status arena_alloc(chm_ctx *ctx, uint64_t bytes) {
  auto t0 = std::chrono::steady_clock::now();
  ctx->arena = nullptr;
  ctx->arena_bytes = 0;
  ctx->arena_registered = false;
  ctx->arena_node = -1;
  int node = ctx->arena_numa;
  if (node == -1) node = device_numa_node(ctx->device);
  if (node >= 0 && node >= online_nodes()) node = -1;  // sysfs names a node that is not online
  const bool reg = ctx->arena_mode != CHM_ARENA_HOSTALLOC;
  if (!reg) {
    cudaError_t e = cudaHostAlloc(&ctx->arena, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
    if (e != cudaSuccess) {
      ctx->arena = nullptr;
      CHM_FAIL(CHM_E_NOMEM, "arena: cudaHostAlloc(%llu) failed: %s", (unsigned long long)bytes,
               cudaGetErrorString(e));
    }
  } else {
    const uint64_t huge = 2ull << 20;
    const uint64_t len = (bytes + huge - 1) / huge * huge;
    // pre-faulting more than the host has would wake the OOM killer instead of failing here
    // (cudaHostAlloc fails cleanly): refuse beyond 90% of MemAvailable
    const uint64_t avail = mem_available();
    if (avail && len > avail / 10 * 9)
      CHM_FAIL(CHM_E_NOMEM, "arena: %llu B exceed 90%% of MemAvailable (%llu B)", (unsigned long long)len,
               (unsigned long long)avail);
    void *p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
    if (p == MAP_FAILED) CHM_FAIL(CHM_E_NOMEM, "arena: mmap(%llu) failed: %s", (unsigned long long)len, strerror(errno));
    madvise(p, len, MADV_HUGEPAGE);  // best effort: THP may be disabled
    madvise(p, len, MADV_DONTFORK);  // forked children (data-loader workers) never share the pinned pages
    if (node >= 0 && node < 1024) {
      unsigned long mask[1024 / (8 * sizeof(unsigned long))] = {0};
      mask[node / (8 * sizeof(unsigned long))] = 1ul << (node % (8 * sizeof(unsigned long)));
      if (syscall(SYS_mbind, p, len, kMpolPreferred, mask, 1024ul, 0u) != 0) {
        int err = errno;
        munmap(p, len);
        CHM_FAIL(CHM_E_NOMEM, "arena: mbind to node %d failed: %s", node, strerror(err));
      }
      ctx->arena_node = node;
    }
    // pre-fault in parallel: one thread per contiguous slice, one write per 4 KiB page
    unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    unsigned T = ctx->arena_threads ? ctx->arena_threads : std::min(hw, 32u);
    T = unsigned(std::min<uint64_t>(T, std::max<uint64_t>(1, len / huge)));
    const uint64_t slice = (len / huge + T - 1) / T * huge;
    std::vector<std::thread> th;
    for (unsigned k = 0; k < T; k++) {
      uint64_t a = uint64_t(k) * slice, b = std::min(len, a + slice);
      if (a >= b) break;
      th.emplace_back([p, a, b] {
        volatile char *c = static_cast<char *>(p);
        for (uint64_t o = a; o < b; o += 4096) c[o] = 0;
      });
    }
    for (auto &t : th) t.join();
    cudaError_t e = cudaHostRegister(p, len, cudaHostRegisterMapped | cudaHostRegisterPortable);
    if (e != cudaSuccess) {
      munmap(p, len);
      CHM_FAIL(CHM_E_NOMEM, "arena: cudaHostRegister(%llu) failed: %s", (unsigned long long)len,
               cudaGetErrorString(e));
    }
    ctx->arena = p;
    ctx->arena_registered = true;
    ctx->arena_map_bytes = len;
  }
  void *dptr = nullptr;
  if (cudaHostGetDevicePointer(&dptr, ctx->arena, 0) != cudaSuccess || dptr != ctx->arena) {
    arena_free(ctx);
    CHM_FAIL(CHM_E_CUDA, "arena: mapped arena is not UVA-identical");
  }
  ctx->arena_bytes = bytes;
  ctx->arena_pin_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return CHM_OK;
}

void arena_free(chm_ctx *ctx) {
  if (!ctx->arena) return;
  if (ctx->arena_registered) {
    cudaHostUnregister(ctx->arena);
    munmap(ctx->arena, ctx->arena_map_bytes);
  } else {
    cudaFreeHost(ctx->arena);
  }
  ctx->arena = nullptr;
  ctx->arena_bytes = 0;
  ctx->arena_map_bytes = 0;
  ctx->arena_registered = false;
}

}  // namespace chm

extern "C" chm_status chm_arena_placement(const chm_ctx *ctx, int32_t *numa_node, int32_t *mode, double *pin_seconds) {
  if (!ctx) CHM_FAIL(CHM_E_INVAL, "chm_arena_placement: NULL ctx");
  if (numa_node) *numa_node = ctx->arena_node;
  if (mode) *mode = !ctx->arena ? -1 : ctx->arena_registered ? CHM_ARENA_REGISTER : CHM_ARENA_HOSTALLOC;
  if (pin_seconds) *pin_seconds = ctx->arena_pin_s;
  return CHM_OK;
}
