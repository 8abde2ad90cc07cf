"""Minimal PNG writer (no PIL in the image) for looking at frames."""
import struct
import sys
import zlib

import numpy as np


def write_png(path, rgb):
    rgb = np.ascontiguousarray(rgb, np.uint8)
    h, w, _ = rgb.shape
    raw = b"".join(b"\x00" + rgb[y].tobytes() for y in range(h))

    def chunk(tag, data):
        return struct.pack(">I", len(data)) + tag + data + struct.pack(">I", zlib.crc32(tag + data) & 0xffffffff)

    with open(path, "wb") as f:
        f.write(b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, 8, 2, 0, 0, 0)) +
                chunk(b"IDAT", zlib.compress(raw, 6)) + chunk(b"IEND", b""))


if __name__ == "__main__":   # ppm -> png
    blob = open(sys.argv[1], "rb").read()
    parts = blob.split(maxsplit=4)
    w, h = int(parts[1]), int(parts[2])
    write_png(sys.argv[2], np.frombuffer(parts[4][:3 * w * h], np.uint8).reshape(h, w, 3))
