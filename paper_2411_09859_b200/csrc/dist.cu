// Multi-GPU plumbing for the block-cyclic driver (skl_ltlt_blk_piv_dist):
//
// * CUDA VMM: physical HBM allocations exported as POSIX file descriptors and
//   mapped, block by block, into one virtual address range per rank, so the
//   distributed work matrix is addressed as a single column-major array and
//   remote columns are plain NVLink loads/stores from the kernels.
// * A stream-ordered barrier over NCCL (a one-word all-reduce on the caller's
//   stream), loaded with dlopen so the library itself has no NCCL dependency.
//
// Driver-API entry points come from cudaGetDriverEntryPoint (no -lcuda link),
// so the library still loads on hosts without a GPU driver.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

#include "skewltl_b200.h"

namespace {

template <typename F>
F drv(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}

struct Vmm {
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemExportToShareableHandle) export_h = nullptr;
  decltype(&cuMemImportFromShareableHandle) import_h = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) vfree = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) access = nullptr;
  decltype(&cuMemGetAllocationGranularity) gran = nullptr;
  bool ok = false;
};

const Vmm& vmm() {
  static Vmm v;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaFree(nullptr);  // primary context current on this thread
    v.create = drv<decltype(&cuMemCreate)>("cuMemCreate");
    v.release = drv<decltype(&cuMemRelease)>("cuMemRelease");
    v.export_h = drv<decltype(&cuMemExportToShareableHandle)>("cuMemExportToShareableHandle");
    v.import_h = drv<decltype(&cuMemImportFromShareableHandle)>("cuMemImportFromShareableHandle");
    v.reserve = drv<decltype(&cuMemAddressReserve)>("cuMemAddressReserve");
    v.vfree = drv<decltype(&cuMemAddressFree)>("cuMemAddressFree");
    v.map = drv<decltype(&cuMemMap)>("cuMemMap");
    v.unmap = drv<decltype(&cuMemUnmap)>("cuMemUnmap");
    v.access = drv<decltype(&cuMemSetAccess)>("cuMemSetAccess");
    v.gran = drv<decltype(&cuMemGetAllocationGranularity)>("cuMemGetAllocationGranularity");
    v.ok = v.create && v.release && v.export_h && v.import_h && v.reserve && v.vfree && v.map && v.unmap &&
           v.access && v.gran;
  }
  return v;
}

CUmemAllocationProp prop_for(int device, int exportable) {
  CUmemAllocationProp p;
  memset(&p, 0, sizeof(p));
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = device;
  p.requestedHandleTypes = exportable ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR : CU_MEM_HANDLE_TYPE_NONE;
  return p;
}

thread_local int g_last_cu = 0;
int st(CUresult r) {
  g_last_cu = (int)r;
  return r == CUDA_SUCCESS ? SKL_OK : SKL_CUDA_ERROR;
}

// ---- NCCL (dlopen) ----------------------------------------------------------
struct Nccl {
  decltype(&ncclGetUniqueId) uid = nullptr;
  decltype(&ncclCommInitRank) init = nullptr;
  decltype(&ncclAllReduce) allreduce = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n;
  static bool tried = false;
  if (!tried) {
    tried = true;
    // the process normally has torch's libnccl loaded already; RTLD_NOLOAD first
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (h) {
      n.uid = reinterpret_cast<decltype(&ncclGetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
      n.init = reinterpret_cast<decltype(&ncclCommInitRank)>(dlsym(h, "ncclCommInitRank"));
      n.allreduce = reinterpret_cast<decltype(&ncclAllReduce)>(dlsym(h, "ncclAllReduce"));
      n.destroy = reinterpret_cast<decltype(&ncclCommDestroy)>(dlsym(h, "ncclCommDestroy"));
      n.ok = n.uid && n.init && n.allreduce && n.destroy;
    }
  }
  return n;
}

struct NcclBarrier {
  ncclComm_t comm;
  int* word;  // device scratch for the one-word all-reduce
};

}  // namespace

extern "C" {

int skl_vmm_available(void) { return vmm().ok ? 1 : 0; }

int skl_vmm_last_result(void) { return g_last_cu; }

int skl_vmm_granularity(int device, size_t* gran) {
  const Vmm& v = vmm();
  if (!v.ok || !gran) return SKL_UNSUPPORTED;
  CUmemAllocationProp p = prop_for(device, 1);
  return st(v.gran(gran, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
}

int skl_vmm_create(size_t bytes, int device, int exportable, unsigned long long* handle) {
  const Vmm& v = vmm();
  if (!v.ok || !handle || bytes == 0) return SKL_BAD_ARGUMENT;
  CUmemAllocationProp p = prop_for(device, exportable);
  CUmemGenericAllocationHandle h;
  int rc = st(v.create(&h, bytes, &p, 0));
  if (rc == SKL_OK) *handle = (unsigned long long)h;
  return rc;
}

int skl_vmm_export_fd(unsigned long long handle, int* fd) {
  const Vmm& v = vmm();
  if (!v.ok || !fd) return SKL_BAD_ARGUMENT;
  int f = -1;
  int rc = st(v.export_h(&f, (CUmemGenericAllocationHandle)handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  if (rc == SKL_OK) *fd = f;
  return rc;
}

int skl_vmm_import_fd(int fd, unsigned long long* handle) {
  const Vmm& v = vmm();
  if (!v.ok || !handle) return SKL_BAD_ARGUMENT;
  CUmemGenericAllocationHandle h;
  int rc = st(v.import_h(&h, reinterpret_cast<void*>((uintptr_t)fd), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
  if (rc == SKL_OK) *handle = (unsigned long long)h;
  return rc;
}

int skl_vmm_release(unsigned long long handle) {
  const Vmm& v = vmm();
  if (!v.ok) return SKL_UNSUPPORTED;
  return st(v.release((CUmemGenericAllocationHandle)handle));
}

int skl_vmm_reserve(size_t bytes, size_t align, unsigned long long* va) {
  const Vmm& v = vmm();
  if (!v.ok || !va) return SKL_BAD_ARGUMENT;
  CUdeviceptr p = 0;
  int rc = st(v.reserve(&p, bytes, align, 0, 0));
  if (rc == SKL_OK) *va = (unsigned long long)p;
  return rc;
}

int skl_vmm_free_va(unsigned long long va, size_t bytes) {
  const Vmm& v = vmm();
  if (!v.ok) return SKL_UNSUPPORTED;
  return st(v.vfree((CUdeviceptr)va, bytes));
}

int skl_vmm_map(unsigned long long va, size_t bytes, unsigned long long handle, size_t offset, int device) {
  const Vmm& v = vmm();
  if (!v.ok) return SKL_UNSUPPORTED;
  int rc = st(v.map((CUdeviceptr)va, bytes, offset, (CUmemGenericAllocationHandle)handle, 0));
  if (rc != SKL_OK) return rc;
  CUmemAccessDesc d;
  memset(&d, 0, sizeof(d));
  d.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  d.location.id = device;
  d.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  return st(v.access((CUdeviceptr)va, bytes, &d, 1));
}

int skl_vmm_unmap(unsigned long long va, size_t bytes) {
  const Vmm& v = vmm();
  if (!v.ok) return SKL_UNSUPPORTED;
  return st(v.unmap((CUdeviceptr)va, bytes));
}

// ---- NCCL barrier ------------------------------------------------------------
int skl_nccl_available(void) { return nccl().ok ? 1 : 0; }

int skl_nccl_unique_id(unsigned char* out, size_t bytes) {
  const Nccl& n = nccl();
  if (!n.ok || !out || bytes < sizeof(ncclUniqueId)) return SKL_UNSUPPORTED;
  ncclUniqueId id;
  if (n.uid(&id) != ncclSuccess) return SKL_CUDA_ERROR;
  memcpy(out, &id, sizeof(id));
  return SKL_OK;
}

int skl_nccl_barrier_create(int nranks, int rank, const unsigned char* id, void** ctx) {
  const Nccl& n = nccl();
  if (!n.ok || !id || !ctx) return SKL_UNSUPPORTED;
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  NcclBarrier* b = new NcclBarrier{};
  if (n.init(&b->comm, nranks, uid, rank) != ncclSuccess) {
    delete b;
    return SKL_CUDA_ERROR;
  }
  if (cudaMalloc(&b->word, sizeof(int)) != cudaSuccess || cudaMemset(b->word, 0, sizeof(int)) != cudaSuccess) {
    n.destroy(b->comm);
    delete b;
    return SKL_CUDA_ERROR;
  }
  *ctx = b;
  return SKL_OK;
}

// matches skl_barrier_fn: stream-ordered, no host synchronisation
int skl_nccl_barrier(void* ctx, void* stream) {
  const Nccl& n = nccl();
  NcclBarrier* b = static_cast<NcclBarrier*>(ctx);
  if (!n.ok || !b) return SKL_UNSUPPORTED;
  return n.allreduce(b->word, b->word, 1, ncclInt32, ncclSum, b->comm, static_cast<cudaStream_t>(stream)) ==
                 ncclSuccess
             ? SKL_OK
             : SKL_CUDA_ERROR;
}

int skl_nccl_barrier_destroy(void* ctx) {
  const Nccl& n = nccl();
  NcclBarrier* b = static_cast<NcclBarrier*>(ctx);
  if (!b) return SKL_OK;
  cudaFree(b->word);
  if (n.ok) n.destroy(b->comm);
  delete b;
  return SKL_OK;
}

}  // extern "C"
