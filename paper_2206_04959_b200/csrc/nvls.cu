// nvls.cu -- NVLink-SHARP (NVLS) in-switch reduction for the TMP all-reduce (the
// 2 + 2 all-reduces of P:558 over the TMP group of P:763).
//
// The all-reduce slots of every rank are bound to one CUDA multicast object.  Phase 1 of the two-shot
// all-reduce then needs no peer loads: rank r reads the rows it owns through the multicast address with
// multimem.ld_reduce -- the NVSwitch returns the sum over the T ranks' partials (fp32 accumulation in the
// switch, one bf16 rounding) -- adds bias and residual (forward) and writes the result with multimem.st into
// the same rows of EVERY rank's slot.  After the usual cross-rank handshake each rank's fused epilogue kernel
// reads all rows from its OWN slot ("gathered" mode with every row local).  NVLink bytes per GPU and
// direction ~ (1 + 1/T) of a slot instead of 2(T-1)/T for the peer-load two-shot.
//
// Setup (collective): rank 0 creates the multicast object and exports it as a POSIX file descriptor, which
// the other ranks duplicate with pidfd_getfd (same user, no ptrace restriction needed beyond that); every
// rank adds its device, binds its own physical slot memory, and maps the memory both unicast (GEMM epilogues
// write the partial there) and multicast.
#include <string.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <string>
#include <vector>

#include "kernels.h"
#include "merak_tmp.h"
#include "ptx.cuh"

namespace mk {

namespace {

struct Drv {
  bool ok = false;
  CUresult (*DeviceGet)(CUdevice *, int);
  CUresult (*DeviceGetAttribute)(int *, CUdevice_attribute, CUdevice);
  CUresult (*MulticastCreate)(CUmemGenericAllocationHandle *, const CUmulticastObjectProp *);
  CUresult (*MulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice);
  CUresult (*MulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                               unsigned long long);
  CUresult (*MulticastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);
  CUresult (*MulticastGetGranularity)(size_t *, const CUmulticastObjectProp *, CUmulticastGranularity_flags);
  CUresult (*MemCreate)(CUmemGenericAllocationHandle *, size_t, const CUmemAllocationProp *, unsigned long long);
  CUresult (*MemRelease)(CUmemGenericAllocationHandle);
  CUresult (*MemGetAllocationGranularity)(size_t *, const CUmemAllocationProp *, CUmemAllocationGranularity_flags);
  CUresult (*MemExportToShareableHandle)(void *, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                                         unsigned long long);
  CUresult (*MemImportFromShareableHandle)(CUmemGenericAllocationHandle *, void *, CUmemAllocationHandleType);
  CUresult (*MemAddressReserve)(CUdeviceptr *, size_t, size_t, CUdeviceptr, unsigned long long);
  CUresult (*MemAddressFree)(CUdeviceptr, size_t);
  CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
  CUresult (*MemUnmap)(CUdeviceptr, size_t);
  CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc *, size_t);
  CUresult (*GetErrorString)(CUresult, const char **);
};

template <class F>
bool sym(const char *name, F &f) {
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return false;
  f = reinterpret_cast<F>(p);
  return true;
}

Drv &drv() {
  static Drv d;
  static bool tried = false;
  if (!tried) {
    tried = true;
    d.ok = sym("cuDeviceGet", d.DeviceGet) && sym("cuDeviceGetAttribute", d.DeviceGetAttribute) &&
           sym("cuMulticastCreate", d.MulticastCreate) && sym("cuMulticastAddDevice", d.MulticastAddDevice) &&
           sym("cuMulticastBindMem", d.MulticastBindMem) && sym("cuMulticastUnbind", d.MulticastUnbind) &&
           sym("cuMulticastGetGranularity", d.MulticastGetGranularity) && sym("cuMemCreate", d.MemCreate) &&
           sym("cuMemRelease", d.MemRelease) && sym("cuMemGetAllocationGranularity", d.MemGetAllocationGranularity) &&
           sym("cuMemExportToShareableHandle", d.MemExportToShareableHandle) &&
           sym("cuMemImportFromShareableHandle", d.MemImportFromShareableHandle) &&
           sym("cuMemAddressReserve", d.MemAddressReserve) && sym("cuMemAddressFree", d.MemAddressFree) &&
           sym("cuMemMap", d.MemMap) && sym("cuMemUnmap", d.MemUnmap) && sym("cuMemSetAccess", d.MemSetAccess) &&
           sym("cuGetErrorString", d.GetErrorString);
  }
  return d;
}

std::string cuerr(CUresult r) {
  const char *s = nullptr;
  if (drv().GetErrorString) drv().GetErrorString(r, &s);
  return s ? s : "unknown CUDA driver error";
}

}  // namespace

bool nvls_supported(int dev) {
  Drv &d = drv();
  if (!d.ok) return false;
  CUdevice cd;
  int v = 0;
  if (d.DeviceGet(&cd, dev) != CUDA_SUCCESS) return false;
  if (d.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cd) != CUDA_SUCCESS) return false;
  return v != 0;
}

void nvls_release(Nvls *n) {
  Drv &d = drv();
  if (!d.ok || !n) return;
  if (n->mc_va) {
    d.MemUnmap((CUdeviceptr)n->mc_va, n->size);
    d.MemAddressFree((CUdeviceptr)n->mc_va, n->size);
  }
  if (n->uc_va) {
    d.MemUnmap((CUdeviceptr)n->uc_va, n->size);
    d.MemAddressFree((CUdeviceptr)n->uc_va, n->size);
  }
  if (n->bound) {
    CUdevice cd;
    if (d.DeviceGet(&cd, n->dev) == CUDA_SUCCESS) d.MulticastUnbind(n->mc_handle, cd, 0, n->size);
  }
  if (n->mem_handle) d.MemRelease(n->mem_handle);
  if (n->mc_handle) d.MemRelease(n->mc_handle);
  if (n->fd >= 0) close(n->fd);
  memset(n, 0, sizeof(*n));
  n->fd = -1;
}

int nvls_setup(Nvls *n, int dev, int T, int r, size_t bytes, merak_allgather_fn ag, void *ctx, std::string *err) {
  memset(n, 0, sizeof(*n));
  n->fd = -1;
  n->dev = dev;
  Drv &d = drv();
  auto bad = [&](const std::string &m) {
    *err = m;
    nvls_release(n);
    return -1;
  };
  // every rank must support multicast (exchanged, so all ranks take the same decision)
  int sup = nvls_supported(dev) ? 1 : 0, sups[MAX_T];
  if (ag(ctx, &sup, sups, sizeof(int)) != 0) return bad("allgather failed (multicast support)");
  for (int q = 0; q < T; ++q)
    if (!sups[q]) {
      *err = "CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED is 0 on rank " + std::to_string(q);
      return -2;
    }
  CUdevice cd;
  CUresult e;
  if ((e = d.DeviceGet(&cd, dev)) != CUDA_SUCCESS) return bad("cuDeviceGet: " + cuerr(e));
  CUmulticastObjectProp mp;
  memset(&mp, 0, sizeof(mp));
  mp.numDevices = (unsigned)T;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g_mc = 0, g_mem = 0;
  mp.size = bytes;
  if ((e = d.MulticastGetGranularity(&g_mc, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED)) != CUDA_SUCCESS)
    return bad("cuMulticastGetGranularity: " + cuerr(e));
  CUmemAllocationProp ap;
  memset(&ap, 0, sizeof(ap));
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = dev;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;  // binding into the multicast object needs it
  if ((e = d.MemGetAllocationGranularity(&g_mem, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED)) != CUDA_SUCCESS)
    return bad("cuMemGetAllocationGranularity: " + cuerr(e));
  const size_t g = g_mc > g_mem ? g_mc : g_mem;
  n->size = (bytes + g - 1) / g * g;
  mp.size = n->size;
  // rank 0 creates the multicast object and exports it; the others duplicate its descriptor
  struct {
    int pid, fd, status;
  } mine = {(int)getpid(), -1, 0}, all[MAX_T];
  if (r == 0) {
    if ((e = d.MulticastCreate(&n->mc_handle, &mp)) != CUDA_SUCCESS) mine.status = (int)e;
    if (!mine.status) {
      int fd = -1;
      if ((e = d.MemExportToShareableHandle(&fd, n->mc_handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0)) !=
          CUDA_SUCCESS)
        mine.status = (int)e;
      n->fd = fd;
      mine.fd = fd;
    }
  }
  if (ag(ctx, &mine, all, sizeof(mine)) != 0) return bad("allgather failed (multicast handle)");
  if (all[0].status) return bad("rank 0 cuMulticastCreate / export: " + cuerr((CUresult)all[0].status));
  if (r != 0) {
    const int pfd = (int)syscall(SYS_pidfd_open, all[0].pid, 0);
    if (pfd < 0) return bad("pidfd_open(rank 0) failed");
    n->fd = (int)syscall(SYS_pidfd_getfd, pfd, all[0].fd, 0);
    close(pfd);
    if (n->fd < 0) return bad("pidfd_getfd(rank 0's multicast descriptor) failed");
    if ((e = d.MemImportFromShareableHandle(&n->mc_handle, (void *)(uintptr_t)n->fd,
                                            CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR)) != CUDA_SUCCESS)
      return bad("cuMemImportFromShareableHandle: " + cuerr(e));
  }
  // every device joins before any memory is bound
  int st = (int)d.MulticastAddDevice(n->mc_handle, cd), sts[MAX_T];
  if (ag(ctx, &st, sts, sizeof(int)) != 0) return bad("allgather failed (add device)");
  for (int q = 0; q < T; ++q)
    if (sts[q]) return bad("cuMulticastAddDevice on rank " + std::to_string(q) + ": " + cuerr((CUresult)sts[q]));
  // this rank's physical slot memory, bound into the multicast object
  if ((e = d.MemCreate(&n->mem_handle, n->size, &ap, 0)) != CUDA_SUCCESS) return bad("cuMemCreate: " + cuerr(e));
  st = (int)d.MulticastBindMem(n->mc_handle, 0, n->mem_handle, 0, n->size, 0);
  n->bound = st == 0;
  if (ag(ctx, &st, sts, sizeof(int)) != 0) return bad("allgather failed (bind)");
  for (int q = 0; q < T; ++q)
    if (sts[q]) return bad("cuMulticastBindMem on rank " + std::to_string(q) + ": " + cuerr((CUresult)sts[q]));
  CUmemAccessDesc acc;
  memset(&acc, 0, sizeof(acc));
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUdeviceptr va = 0;
  if ((e = d.MemAddressReserve(&va, n->size, g, 0, 0)) != CUDA_SUCCESS) return bad("cuMemAddressReserve: " + cuerr(e));
  n->uc_va = (void *)va;
  if ((e = d.MemMap(va, n->size, 0, n->mem_handle, 0)) != CUDA_SUCCESS) return bad("cuMemMap (unicast): " + cuerr(e));
  if ((e = d.MemSetAccess(va, n->size, &acc, 1)) != CUDA_SUCCESS) return bad("cuMemSetAccess (unicast): " + cuerr(e));
  if ((e = d.MemAddressReserve(&va, n->size, g, 0, 0)) != CUDA_SUCCESS) return bad("cuMemAddressReserve: " + cuerr(e));
  n->mc_va = (void *)va;
  if ((e = d.MemMap(va, n->size, 0, n->mc_handle, 0)) != CUDA_SUCCESS) return bad("cuMemMap (multicast): " + cuerr(e));
  if ((e = d.MemSetAccess(va, n->size, &acc, 1)) != CUDA_SUCCESS) return bad("cuMemSetAccess (multicast): " + cuerr(e));
  return 0;
}

// ------------------------------------------------------------------------------------------ kernel
MK_DEV uint4 mm_ld_reduce_bf16x8(const void *mc) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(mc)
               : "memory");
  return v;
}
MK_DEV void mm_st_bf16x8(void *mc, uint4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.bf16x2 [%0], {%1,%2,%3,%4};" ::"l"(mc), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

// rows [row0, row1) of the sub-batch: v = sum over the T ranks (switch) [+ bias + resid, fp32, rounded once]
// -> multimem.st into every rank's slot rows.  One 16-B chunk per thread-iteration, grid-stride.
__global__ void __launch_bounds__(256) nvls_rs_kernel(NvlsRsArgs a) {
  if (a.pdl) griddep_wait();
  const int cpr = a.h / 8;  // 16-B chunks per row
  const long n = (long)(a.row1 - a.row0) * cpr;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const long row = a.row0 + i / cpr;
    const int c = (int)(i % cpr) * 8;
    __nv_bfloat16 *p = a.mc + row * a.h + c;
    uint4 v = mm_ld_reduce_bf16x8(p);
    if (a.resid) {
      const uint4 rv = *reinterpret_cast<const uint4 *>(a.resid + row * a.h + c);
      const uint4 bv = *reinterpret_cast<const uint4 *>(a.bias + c);
      uint32_t *vv = &v.x;
      const uint32_t *rr = &rv.x, *bb = &bv.x;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 s = unpack_bf16(vv[k]), x = unpack_bf16(rr[k]), b = unpack_bf16(bb[k]);
        vv[k] = pack_bf16((s.x + b.x) + x.x, (s.y + b.y) + x.y);
      }
    }
    mm_st_bf16x8(p, v);
  }
  asm volatile("fence.acq_rel.sys;" ::: "memory");  // the multicast stores precede the handshake's release
  if (a.ps.publish) publish_when_done(a.ps);
}

cudaError_t nvls_rs(const NvlsRsArgs &a, cudaStream_t st) {
  if (a.h % 8 != 0) return cudaErrorInvalidValue;
  const long n = (long)(a.row1 - a.row0) * (a.h / 8);
  if (n <= 0) return cudaSuccess;
  int blocks = (int)((n + 255) / 256);
  const int cap = a.ctas > 0 ? a.ctas : 2 * gemm_num_sms();
  if (blocks > cap) blocks = cap;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = a.pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, nvls_rs_kernel, a);
}

cudaError_t nvls_preload() { return touch_kernel((const void *)nvls_rs_kernel); }

}  // namespace mk
