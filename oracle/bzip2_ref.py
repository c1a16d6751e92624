"""Test infrastructure: a pure-Python restatement of the libbzip2 1.0.8
compressor at block size 9 (what the reference's blocks.py:80 calls through
Python's bz2.compress(chunk, 9)).  Not vendored in /root/reference (stdlib
bz2 -> system libbz2.so.1.0, bzip2 1.0.8); restated from the
published algorithm (compress.c, huffman.c, bzlib.c of bzip2 1.0.8) and
pinned byte-for-byte against bz2.compress in tests/test_bzip2_ref.py.  It is
the stage-by-stage oracle of the GPU block coder (csrc/bzip2.cu): RLE1 block
split, BWT (cyclic rotation sort), MTF + RUNA/RUNB, Huffman table selection
and the bitstream.  Pure Python: use on inputs of a few MB at most.
"""
from __future__ import annotations

BLOCK_MAX = 100000 * 9 - 19          # nblockMAX at level 9 (bzlib.c)
N_ITERS = 4                          # BZ_N_ITERS
G_SIZE = 50                          # BZ_G_SIZE
MAX_LEN = 17                         # hbMakeCodeLengths maxLen (compress.c)
RUNA, RUNB = 0, 1


def _crc_table():
    t = []
    for i in range(256):
        c = i << 24
        for _ in range(8):
            c = ((c << 1) ^ 0x04C11DB7) if c & 0x80000000 else (c << 1)
        t.append(c & 0xFFFFFFFF)
    return t


CRC_TABLE = _crc_table()


def crc_update(crc: int, ch: int) -> int:
    return ((crc << 8) & 0xFFFFFFFF) ^ CRC_TABLE[(crc >> 24) ^ ch]


class Block:
    def __init__(self):
        self.data = bytearray()
        self.crc = 0xFFFFFFFF
        self.in_use = [False] * 256

    def final_crc(self) -> int:
        return self.crc ^ 0xFFFFFFFF


def rle1_blocks(src: bytes) -> list:
    """bzlib.c ADD_CHAR_TO_BLOCK / add_pair_to_block / copy_input_until_stop /
    handle_compress as driven by bz2.compress: a full block (nblock >=
    nblockMAX before the next char) is closed WITHOUT flushing the pending
    run, which continues into the next block; the final flush adds it."""
    blocks = [Block()]
    ch, run = 256, 0

    def add_pair(b: Block):
        for _ in range(run):
            b.crc = crc_update(b.crc, ch)
        b.in_use[ch] = True
        if run <= 3:
            b.data += bytes([ch]) * run
        else:
            b.in_use[run - 4] = True
            b.data += bytes([ch]) * 4 + bytes([run - 4])

    for c in src:
        b = blocks[-1]
        if len(b.data) >= BLOCK_MAX:
            blocks.append(Block())
            b = blocks[-1]
        if c != ch and run == 1:
            b.crc = crc_update(b.crc, ch)
            b.in_use[ch] = True
            b.data.append(ch)
            ch = c
        elif c != ch or run == 255:
            if ch < 256:
                add_pair(b)
            ch, run = c, 1
        else:
            run += 1
    if len(blocks[-1].data) >= BLOCK_MAX:
        blocks.append(Block())
    if ch < 256:
        add_pair(blocks[-1])
    if not blocks[-1].data and len(blocks) > 1:
        blocks.pop()
    return blocks


def bwt(block: bytes):
    """Sorted cyclic rotations (BZ2_blockSort): (last column, origPtr, tie).
    tie = some rotations are equal (the block is periodic): libbz2's order
    among equal rotations comes from its quicksort refinements and is not
    restated (callers code such blocks with the host libbz2).  Prefix
    doubling over cyclic ranks (numpy), so full 900 KB blocks are practical."""
    import numpy as np
    n = len(block)
    a = np.frombuffer(bytes(block), np.uint8).astype(np.int64)
    rank = a.copy()
    h = 1
    while True:
        key = rank * (int(rank.max()) + 1) + rank[(np.arange(n) + h) % n]
        order = np.argsort(key, kind="stable")
        ks = key[order]
        newr = np.empty(n, np.int64)
        newr[order] = np.concatenate([[0], np.cumsum(ks[1:] != ks[:-1])])
        rank = newr
        if rank.max() == n - 1 or h >= n:
            break
        h *= 2
    order = np.argsort(rank, kind="stable")
    tie = bool(rank.max() < n - 1)
    orig = int(np.nonzero(order == 0)[0][0])
    return bytes(a[(order - 1) % n].astype(np.uint8)), orig, tie


def mtf_values(last: bytes, in_use: list):
    """compress.c generateMTFValues: MTF over the used-symbol alphabet with
    zero runs as RUNA/RUNB (bijective base 2), EOB = nInUse + 1."""
    seq = [i for i in range(256) if in_use[i]]
    unseq_to_seq = {c: k for k, c in enumerate(seq)}
    n_in_use = len(seq)
    eob = n_in_use + 1
    freq = [0] * (eob + 1)
    yy = list(range(n_in_use))
    out = []
    zpend = 0

    def flush_zeros(z):
        z -= 1
        while True:
            v = RUNB if z & 1 else RUNA
            out.append(v)
            freq[v] += 1
            if z < 2:
                break
            z = (z - 2) // 2

    for c in last:
        ll = unseq_to_seq[c]
        if yy[0] == ll:
            zpend += 1
            continue
        if zpend:
            flush_zeros(zpend)
            zpend = 0
        j = yy.index(ll)
        del yy[j]
        yy.insert(0, ll)
        out.append(j + 1)
        freq[j + 1] += 1
    if zpend:
        flush_zeros(zpend)
    out.append(eob)
    freq[eob] += 1
    return out, freq, n_in_use


def make_code_lengths(freq: list, alpha: int, max_len: int) -> list:
    """huffman.c BZ2_hbMakeCodeLengths, heap operations and tie-breaks included."""
    weight = [0] * (alpha * 2 + 2)
    parent = [0] * (alpha * 2 + 2)
    heap = [0] * (alpha + 3)
    for i in range(alpha):
        weight[i + 1] = (freq[i] if freq[i] else 1) << 8
    while True:
        n_nodes, n_heap = alpha, 0
        heap[0], weight[0], parent[0] = 0, 0, -2

        def upheap(z):
            tmp = heap[z]
            while weight[tmp] < weight[heap[z >> 1]]:
                heap[z] = heap[z >> 1]
                z >>= 1
            heap[z] = tmp

        def downheap(z):
            tmp = heap[z]
            while True:
                y = z << 1
                if y > n_heap:
                    break
                if y < n_heap and weight[heap[y + 1]] < weight[heap[y]]:
                    y += 1
                if weight[tmp] < weight[heap[y]]:
                    break
                heap[z] = heap[y]
                z = y
            heap[z] = tmp

        for i in range(1, alpha + 1):
            parent[i] = -1
            n_heap += 1
            heap[n_heap] = i
            upheap(n_heap)
        while n_heap > 1:
            n1 = heap[1]; heap[1] = heap[n_heap]; n_heap -= 1; downheap(1)
            n2 = heap[1]; heap[1] = heap[n_heap]; n_heap -= 1; downheap(1)
            n_nodes += 1
            parent[n1] = parent[n2] = n_nodes
            w1, w2 = weight[n1], weight[n2]
            weight[n_nodes] = ((w1 & 0xFFFFFF00) + (w2 & 0xFFFFFF00)) | (1 + max(w1 & 0xFF, w2 & 0xFF))
            parent[n_nodes] = -1
            n_heap += 1
            heap[n_heap] = n_nodes
            upheap(n_heap)
        lens, too_long = [], False
        for i in range(1, alpha + 1):
            j, k = 0, i
            while parent[k] >= 0:
                k = parent[k]
                j += 1
            lens.append(j)
            too_long |= j > max_len
        if not too_long:
            return lens
        for i in range(1, alpha + 1):
            j = weight[i] >> 8
            weight[i] = (1 + j // 2) << 8


def select_tables(mtfv: list, freq: list, alpha: int):
    """compress.c sendMTFValues: number of tables, initial partition, four
    refinement passes; returns (n_groups, selectors, lens[n_groups][alpha])."""
    n_mtf = len(mtfv)
    n_groups = 2 if n_mtf < 200 else 3 if n_mtf < 600 else 4 if n_mtf < 1200 else 5 if n_mtf < 2400 else 6
    lens = [[15] * alpha for _ in range(n_groups)]
    n_part, rem_f, gs = n_groups, n_mtf, 0
    while n_part > 0:
        t_freq = rem_f // n_part
        ge, a_freq = gs - 1, 0
        while a_freq < t_freq and ge < alpha - 1:
            ge += 1
            a_freq += freq[ge]
        if ge > gs and n_part != n_groups and n_part != 1 and (n_groups - n_part) % 2 == 1:
            a_freq -= freq[ge]
            ge -= 1
        for v in range(alpha):
            lens[n_part - 1][v] = 0 if gs <= v <= ge else 15
        n_part -= 1
        gs = ge + 1
        rem_f -= a_freq
    selectors = []
    for _ in range(N_ITERS):
        rfreq = [[0] * alpha for _ in range(n_groups)]
        selectors = []
        for gs in range(0, n_mtf, G_SIZE):
            grp = mtfv[gs:gs + G_SIZE]
            costs = [sum(lens[t][v] for v in grp) for t in range(n_groups)]
            bt = min(range(n_groups), key=lambda t: (costs[t], t))
            selectors.append(bt)
            for v in grp:
                rfreq[bt][v] += 1
        lens = [make_code_lengths(rfreq[t], alpha, MAX_LEN) for t in range(n_groups)]
    return n_groups, selectors, lens


def assign_codes(lens: list, alpha: int) -> list:
    code, vec = [0] * alpha, 0
    for n in range(min(lens), max(lens) + 1):
        for i in range(alpha):
            if lens[i] == n:
                code[i] = vec
                vec += 1
        vec <<= 1
    return code


class BitWriter:
    def __init__(self):
        self.bits = []

    def put(self, n: int, v: int):
        for k in range(n - 1, -1, -1):
            self.bits.append((v >> k) & 1)

    def tobytes(self) -> bytes:
        b = self.bits + [0] * (-len(self.bits) % 8)
        return bytes(int("".join(map(str, b[i:i + 8])), 2) for i in range(0, len(b), 8))


def write_block(bw: BitWriter, blk: Block, trace=None):
    last, orig, tie = bwt(bytes(blk.data))
    mtfv, freq, n_in_use = mtf_values(last, blk.in_use)
    alpha = n_in_use + 2
    n_groups, sel, lens = select_tables(mtfv, freq, alpha)
    codes = [assign_codes(lens[t], alpha) for t in range(n_groups)]
    if trace is not None:
        trace.append(dict(crc=blk.final_crc(), orig=orig, tie=tie, n=len(blk.data), n_mtf=len(mtfv),
                          n_groups=n_groups, n_sel=len(sel), lens=lens))
    for b in (0x31, 0x41, 0x59, 0x26, 0x53, 0x59):
        bw.put(8, b)
    bw.put(32, blk.final_crc())
    bw.put(1, 0)
    bw.put(24, orig)
    in_use16 = [any(blk.in_use[16 * i:16 * i + 16]) for i in range(16)]
    for u in in_use16:
        bw.put(1, int(u))
    for i in range(16):
        if in_use16[i]:
            for j in range(16):
                bw.put(1, int(blk.in_use[16 * i + j]))
    bw.put(3, n_groups)
    bw.put(15, len(sel))
    pos = list(range(n_groups))
    for s in sel:                                  # selector MTF, unary
        j = pos.index(s)
        del pos[j]
        pos.insert(0, s)
        bw.put(j + 1, (1 << (j + 1)) - 2)          # j ones then a zero
    for t in range(n_groups):                      # delta-coded lengths
        curr = lens[t][0]
        bw.put(5, curr)
        for i in range(alpha):
            while curr < lens[t][i]:
                bw.put(2, 2)
                curr += 1
            while curr > lens[t][i]:
                bw.put(2, 3)
                curr -= 1
            bw.put(1, 0)
    for g, gs in enumerate(range(0, len(mtfv), G_SIZE)):
        t = sel[g]
        for v in mtfv[gs:gs + G_SIZE]:
            bw.put(lens[t][v], codes[t][v])


def compress(src: bytes, trace=None) -> bytes:
    """== bz2.compress(src, 9) (bit-exact except where a periodic block makes
    libbz2's order among equal rotations decide origPtr)."""
    bw = BitWriter()
    for b in b"BZh9":
        bw.put(8, b)
    combined = 0
    blocks = rle1_blocks(src) if src else []
    for blk in blocks:
        if not blk.data:
            continue
        combined = (((combined << 1) | (combined >> 31)) & 0xFFFFFFFF) ^ blk.final_crc()
        write_block(bw, blk, trace)
    for b in (0x17, 0x72, 0x45, 0x38, 0x50, 0x90):
        bw.put(8, b)
    bw.put(32, combined)
    return bw.tobytes()
