// TEST-ONLY comparison bar: cub::DeviceRadixSort::SortPairs on the same (u64 key,
// u32 value) pairs that path A's hand-written onesweep sorts. Not part of libgs and never on the
// product path; tools/sort_bar.py builds it, times both and checks they agree bit for bit.
#include <cub/device/device_radix_sort.cuh>
#include <cstdint>

extern "C" int cub_bar_sort_pairs(const uint64_t* kin, const uint32_t* vin, uint64_t* kout, uint32_t* vout,
                                  int64_t n, int end_bit, void* temp, size_t* temp_bytes, void* stream) {
    const cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, *temp_bytes, kin, kout, vin, vout, n, 0, end_bit,
                                                          static_cast<cudaStream_t>(stream));
    return int(e);
}
