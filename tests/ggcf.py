"""Reader for the reference's contact-field cache file ("GGCF" v1), restated
from ContactFieldIndex::load (reference proj/src/contact_field.cpp:602-655)
for the tests: returns None wherever the reference returns std::nullopt."""
import struct

MAGIC = 0x47474346
VERSION = 1


def read(path, expected_key):
    data = open(path, "rb").read()
    pos = 0

    def get(fmt):
        nonlocal pos
        n = struct.calcsize(fmt)
        if pos + n > len(data):
            raise EOFError
        v = struct.unpack_from("<" + fmt, data, pos)
        pos += n
        return v if len(v) > 1 else v[0]

    def nodes():
        count = get("Q")
        out = [dict(min=get("3d"), max=get("3d"), left=get("i"), right=get("i"), leaf=get("i"))
               for _ in range(count)]
        return out, get("i")

    try:
        if get("I") != MAGIC or get("I") != VERSION:
            return None
        key = get("Q")
        if key != expected_key:
            return None
        w = get("d")
        cb = get("I")
        if cb == 0 or cb > 65536:
            return None
        codebook = [get("3d") for _ in range(cb)]
        patches = []
        for _ in range(get("Q")):
            pid, link, nb = get("i"), get("i"), get("Q")
            boxes = []
            for _ in range(nb):
                cell = get("3q")
                reps = []
                for _ in range(get("I")):
                    code, rl, p, n = get("H"), get("i"), get("3d"), get("3d")
                    if code >= cb:
                        return None
                    reps.append((code, rl, p, n))
                boxes.append(dict(cell=cell, reps=reps))
            nd, root = nodes()
            patches.append(dict(patch_id=pid, link=link, boxes=boxes, nodes=nd, root=root))
        top, top_root = nodes()
    except EOFError:
        return None
    return dict(key=key, box_width=w, codebook=codebook, patches=patches, top_nodes=top,
                top_root=top_root, trailing=len(data) - pos)
