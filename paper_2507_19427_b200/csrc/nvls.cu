// nvls.cu — NVLink SHARP (NVLS) in-switch reduction groups for the AFD
// return path.
//
// The paper's FFN-tier tensor parallelism reduces the FFN GPUs' partials
// (all-gather in, reduce-scatter out); with expert
// parallelism the attention side reduces the EP partials.  On
// an NVSwitch box the reduction can run IN the switch: every member GPU binds
// one buffer to a multicast object, and one `multimem.ld_reduce` through the
// multicast address returns the element-wise sum over all members' buffers
// (the switch reads each member once; the reading GPU receives only the sum).
//
// A group = one multicast object (cuMulticastCreate) + on every member a
// physical allocation (cuMemCreate) bound to it, mapped twice: the member's
// own unicast view (where it writes its contribution with ordinary stores)
// and the multicast view (where `multimem.ld_reduce` reads the sum).  Members
// live in different processes: the creator exports a POSIX file descriptor
// and the others import it through pidfd_getfd (the exported fd number and
// the creator's pid travel through the caller's rendezvous).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cstdint>
#include <string>

#include "../../include/afdk.h"
#include "afdk_internal.h"
#include "sm100.cuh"

struct afdk_nvls {
  int device = 0;
  size_t size = 0;
  CUmemGenericAllocationHandle mc = 0, mem = 0;
  CUdeviceptr uc_va = 0, mc_va = 0;
  bool mem_made = false, uc_mapped = false, mc_mapped = false, bound = false, mc_made = false;
  int fd = -1;
};

namespace afdk {
namespace {

struct Drv {
  CUresult (*mcCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*);
  CUresult (*mcAddDevice)(CUmemGenericAllocationHandle, CUdevice);
  CUresult (*mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                        unsigned long long);
  CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);
  CUresult (*mcGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags);
  CUresult (*memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
  CUresult (*memRelease)(CUmemGenericAllocationHandle);
  CUresult (*memExport)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long);
  CUresult (*memImport)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType);
  CUresult (*addrReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
  CUresult (*addrFree)(CUdeviceptr, size_t);
  CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
  CUresult (*memUnmap)(CUdeviceptr, size_t);
  CUresult (*setAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
  CUresult (*allocGranularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags);
  CUresult (*devAttr)(int*, CUdevice_attribute, CUdevice);
  bool ok = false;
};

Drv& drv() {
  static Drv d = [] {
    Drv x{};
    cudaDriverEntryPointQueryResult q;
    auto get = [&](const char* name, auto& fn) {
      void* p = nullptr;
      if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p) return false;
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(p);
      return true;
    };
    x.ok = get("cuMulticastCreate", x.mcCreate) && get("cuMulticastAddDevice", x.mcAddDevice) &&
           get("cuMulticastBindMem", x.mcBindMem) && get("cuMulticastUnbind", x.mcUnbind) &&
           get("cuMulticastGetGranularity", x.mcGranularity) && get("cuMemCreate", x.memCreate) &&
           get("cuMemRelease", x.memRelease) && get("cuMemExportToShareableHandle", x.memExport) &&
           get("cuMemImportFromShareableHandle", x.memImport) && get("cuMemAddressReserve", x.addrReserve) &&
           get("cuMemAddressFree", x.addrFree) && get("cuMemMap", x.memMap) && get("cuMemUnmap", x.memUnmap) &&
           get("cuMemSetAccess", x.setAccess) && get("cuMemGetAllocationGranularity", x.allocGranularity) &&
           get("cuDeviceGetAttribute", x.devAttr);
    return x;
  }();
  return d;
}

afdk_status cu_fail(const char* what, CUresult r) {
  set_error(std::string("nvls: ") + what + " failed (CUresult " + std::to_string((int)r) + ")");
  return AFDK_ERR_CUDA;
}

// out[i] = sum over the group's members of their bf16 buffers (in-switch,
// fp32 accumulation): 8 bf16 per thread per multimem.ld_reduce
__global__ void __launch_bounds__(256) nvls_reduce_bf16_kernel(const __nv_bfloat16* mc, __nv_bfloat16* out,
                                                               size_t count) {
  sm100::griddep_wait();
  sm100::griddep_launch();
  for (size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 8; i < count;
       i += (size_t)gridDim.x * blockDim.x * 8) {
    uint32_t a, b, c, d;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "l"(mc + i)
                 : "memory");
    *reinterpret_cast<uint4*>(out + i) = make_uint4(a, b, c, d);
  }
}

}  // namespace

cudaError_t nvls_reduce_launch(const void* mc, void* out, size_t count, cudaStream_t stream, bool pdl) {
  const size_t threads = (count / 8 + 255) / 256;
  const unsigned grid = (unsigned)(threads < 148 * 8 ? (threads ? threads : 1) : 148 * 8);
  return launch_k(pdl, nvls_reduce_bf16_kernel, dim3(grid), dim3(256), 0, stream,
                  static_cast<const __nv_bfloat16*>(mc), static_cast<__nv_bfloat16*>(out), count);
}

}  // namespace afdk

using afdk::cu_fail;
using afdk::drv;
using afdk::set_error;

extern "C" {

int afdk_nvls_supported(afdk_ctx* ctx) {
  if (!ctx || !drv().ok) return 0;
  int v = 0;
  drv().devAttr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, afdk_ctx_device(ctx));
  return v;
}

afdk_status afdk_nvls_create(afdk_ctx* ctx, int n_members, size_t bytes, int creator_pid, int creator_fd,
                             afdk_nvls** out, int* export_fd) {
  if (!ctx || !out || n_members < 1 || bytes == 0) { set_error("afdk_nvls_create: bad argument"); return AFDK_ERR_INVALID; }
  *out = nullptr;
  if (!afdk_nvls_supported(ctx)) { set_error("afdk_nvls_create: device has no NVLS multicast support"); return AFDK_ERR_UNSUPPORTED; }
  const int dev = afdk_ctx_device(ctx);
  afdk::DeviceGuard g(dev);
  cudaFree(nullptr);  // make sure the primary context is current
  auto* r = new afdk_nvls();
  r->device = dev;
  CUmulticastObjectProp mp{};
  mp.numDevices = (unsigned)n_members;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  mp.size = bytes;
  CUresult e = drv().mcGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED);
  if (e != CUDA_SUCCESS) { delete r; return cu_fail("cuMulticastGetGranularity", e); }
  r->size = (bytes + gran - 1) / gran * gran;
  mp.size = r->size;
  if (creator_pid <= 0) {  // this member creates the object and exports it
    if ((e = drv().mcCreate(&r->mc, &mp)) != CUDA_SUCCESS) { delete r; return cu_fail("cuMulticastCreate", e); }
    r->mc_made = true;
    int fd = -1;
    if ((e = drv().memExport(&fd, r->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0)) != CUDA_SUCCESS) {
      afdk_nvls_destroy(r);
      return cu_fail("cuMemExportToShareableHandle", e);
    }
    r->fd = fd;
    if (export_fd) *export_fd = fd;
  } else {  // import the creator's descriptor into this process
    const int pidfd = (int)syscall(SYS_pidfd_open, creator_pid, 0);
    const int fd = pidfd < 0 ? -1 : (int)syscall(SYS_pidfd_getfd, pidfd, creator_fd, 0);
    if (pidfd >= 0) close(pidfd);
    if (fd < 0) {
      delete r;
      set_error("afdk_nvls_create: pidfd_getfd of the creator's descriptor failed (ptrace permission?)");
      return AFDK_ERR_UNSUPPORTED;
    }
    r->fd = fd;
    e = drv().memImport(&r->mc, reinterpret_cast<void*>(static_cast<intptr_t>(fd)),
                        CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    if (e != CUDA_SUCCESS) { afdk_nvls_destroy(r); return cu_fail("cuMemImportFromShareableHandle", e); }
    r->mc_made = true;
  }
  if ((e = drv().mcAddDevice(r->mc, dev)) != CUDA_SUCCESS) { afdk_nvls_destroy(r); return cu_fail("cuMulticastAddDevice", e); }
  *out = r;
  return AFDK_OK;
}

afdk_status afdk_nvls_bind(afdk_nvls* r, void** uc_ptr, void** mc_ptr) {
  if (!r || !uc_ptr || !mc_ptr) { set_error("afdk_nvls_bind: bad argument"); return AFDK_ERR_INVALID; }
  afdk::DeviceGuard g(r->device);
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = r->device;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;  // imported objects bind shareable memory only
  CUresult e;
  if ((e = drv().memCreate(&r->mem, r->size, &ap, 0)) != CUDA_SUCCESS) return cu_fail("cuMemCreate", e);
  r->mem_made = true;
  // blocks until every member added its device
  if ((e = drv().mcBindMem(r->mc, 0, r->mem, 0, r->size, 0)) != CUDA_SUCCESS) return cu_fail("cuMulticastBindMem", e);
  r->bound = true;
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = r->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if ((e = drv().addrReserve(&r->uc_va, r->size, 0, 0, 0)) != CUDA_SUCCESS) return cu_fail("cuMemAddressReserve", e);
  if ((e = drv().memMap(r->uc_va, r->size, 0, r->mem, 0)) != CUDA_SUCCESS) return cu_fail("cuMemMap (unicast)", e);
  r->uc_mapped = true;
  if ((e = drv().setAccess(r->uc_va, r->size, &acc, 1)) != CUDA_SUCCESS) return cu_fail("cuMemSetAccess (unicast)", e);
  if ((e = drv().addrReserve(&r->mc_va, r->size, 0, 0, 0)) != CUDA_SUCCESS) return cu_fail("cuMemAddressReserve", e);
  if ((e = drv().memMap(r->mc_va, r->size, 0, r->mc, 0)) != CUDA_SUCCESS) return cu_fail("cuMemMap (multicast)", e);
  r->mc_mapped = true;
  if ((e = drv().setAccess(r->mc_va, r->size, &acc, 1)) != CUDA_SUCCESS) return cu_fail("cuMemSetAccess (multicast)", e);
  *uc_ptr = reinterpret_cast<void*>(r->uc_va);
  *mc_ptr = reinterpret_cast<void*>(r->mc_va);
  return AFDK_OK;
}

size_t afdk_nvls_size(const afdk_nvls* r) { return r ? r->size : 0; }

void afdk_nvls_destroy(afdk_nvls* r) {
  if (!r) return;
  afdk::DeviceGuard g(r->device);
  cudaDeviceSynchronize();
  if (r->mc_mapped) drv().memUnmap(r->mc_va, r->size);
  if (r->mc_va) drv().addrFree(r->mc_va, r->size);
  if (r->uc_mapped) drv().memUnmap(r->uc_va, r->size);
  if (r->uc_va) drv().addrFree(r->uc_va, r->size);
  if (r->bound) drv().mcUnbind(r->mc, r->device, 0, r->size);
  if (r->mem_made) drv().memRelease(r->mem);
  if (r->mc_made) drv().memRelease(r->mc);
  if (r->fd >= 0) close(r->fd);
  delete r;
}

afdk_status afdk_nvls_reduce_bf16(afdk_ctx* ctx, const void* mc_ptr, void* out, size_t count, afdk_stream stream) {
  if (!ctx || !mc_ptr || !out || count % 8) { set_error("afdk_nvls_reduce_bf16: bad argument (count % 8 == 0)"); return AFDK_ERR_INVALID; }
  afdk::DeviceGuard g(afdk_ctx_device(ctx));
  const cudaError_t e = afdk::nvls_reduce_launch(mc_ptr, out, count, static_cast<cudaStream_t>(stream), false);
  if (e != cudaSuccess) { set_error(std::string("afdk_nvls_reduce_bf16: ") + cudaGetErrorString(e)); return AFDK_ERR_CUDA; }
  return AFDK_OK;
}

}  // extern "C"
