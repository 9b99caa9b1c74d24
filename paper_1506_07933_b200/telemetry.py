"""NVLink byte counters read from the driver (NVML), for the multi-GPU bench
and the exchange-pass evidence (all-to-all bus GB/s against
900 GB/s per direction per GPU).

`NvlinkCounters(index).read()` returns the device's cumulative NVLink data
bytes (tx, rx) summed over all links, from the NVML field values
NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX (KiB, user payload, no protocol
overhead).  Differences of two reads bracket a region; nothing is inferred
from timings.  If NVML or the field is unavailable, `available` is False and
`why` says why (the bench reports that instead of a number).
"""


class NvlinkCounters:
    def __init__(self, index):
        self.index = index
        self.available = False
        self.why = None
        self.nlinks = 0
        try:
            import pynvml as N
            N.nvmlInit()
            self._N = N
            self._h = N.nvmlDeviceGetHandleByIndex(index)
            links = 0
            for link in range(18):
                try:
                    if N.nvmlDeviceGetNvLinkState(self._h, link) == N.NVML_FEATURE_ENABLED:
                        links += 1
                except Exception:
                    break
            self.nlinks = links
            self.read()
            self.available = True
        except Exception as ex:  # reported, not fatal
            self.why = f"{type(ex).__name__}: {ex}"

    def read(self):
        """(tx_bytes, rx_bytes) summed over all links of the device."""
        N = self._N
        ids = [N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX]
        out = []
        for fid in ids:
            # scopeId UINT_MAX = aggregate over all links
            vals = N.nvmlDeviceGetFieldValues(self._h, [(fid, 0xFFFFFFFF)])
            v = vals[0]
            if v.nvmlReturn != 0:
                raise RuntimeError(f"field {fid}: nvml error {v.nvmlReturn}")
            out.append(int(v.value.ullVal) * 1024)
        return out[0], out[1]
