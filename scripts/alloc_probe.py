"""Cold cost of stream-ordered pool growth (cudaMallocAsync) on this box."""
import time

from cuda.bindings import driver, runtime as rt


def ok(r):
    if isinstance(r, tuple):
        assert r[0] == rt.cudaError_t.cudaSuccess, r
        return r[1] if len(r) == 2 else r[1:]
    assert r == rt.cudaError_t.cudaSuccess, r


ok(rt.cudaSetDevice(0))
ok(rt.cudaFree(0))
s = ok(rt.cudaStreamCreate())
pool = ok(rt.cudaDeviceGetDefaultMemPool(0))
ok(rt.cudaMemPoolSetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReleaseThreshold,
                              driver.cuuint64_t(2**63)))
for mb in [1, 16, 64, 256, 1024, 4096]:
    t = time.perf_counter()
    p = ok(rt.cudaMallocAsync(mb << 20, s))
    ok(rt.cudaMemsetAsync(p, 0, mb << 20, s))
    ok(rt.cudaStreamSynchronize(s))
    t1 = time.perf_counter()
    ok(rt.cudaFreeAsync(p, s))
    ok(rt.cudaStreamSynchronize(s))
    t2 = time.perf_counter()
    p = ok(rt.cudaMallocAsync(mb << 20, s))
    ok(rt.cudaMemsetAsync(p, 0, mb << 20, s))
    ok(rt.cudaStreamSynchronize(s))
    t3 = time.perf_counter()
    ok(rt.cudaFreeAsync(p, s))
    print(f"{mb:6d} MB  cold alloc+memset {1e3*(t1-t):8.2f} ms   reuse {1e3*(t3-t2):8.2f} ms")
